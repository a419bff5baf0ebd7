"""Fraction of kept gaussians whose colour activation falls inside the fp32
fallback band (|raw + 0.5| <= kColorTol * sum|c|) during a C3 refit, per step
(fp64 evaluation in torch; diagnostic for the colour kernels' fallback rate)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402
from oracle.raster import sh_basis  # noqa: E402


def main():
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS["c3"]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(pts, (1.0, 0.2, 0.2))
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=7, cache_views=False, prefetch=0)
    pos = ds.positions if isinstance(ds.positions, np.ndarray) else ds.positions.cpu().numpy()
    for it in range(41):
        if it % 10 == 0:
            sh = eng.sh.double().cpu().numpy()
            for v in (0, 17):
                _, pose = cams[v]
                c = -pose.rotation.T @ pose.translation
                d = pos - c
                d = d / np.linalg.norm(d, axis=1, keepdims=True)
                b = sh_basis(d, 3)
                raw = np.einsum("nk,nkc->nc", b, sh) + 0.5
                mag = np.abs(sh).sum(axis=1)
                band = np.abs(raw) <= 3e-5 * mag
                print(f"step {it} view {v}: channels in band {band.mean():.2e}, gaussians {band.any(1).mean():.2e}, "
                      f"warps(8) {1 - (1 - band.any(1).mean()) ** 8:.2e}, |raw+0.5|<1e-3 {np.mean(np.abs(raw) < 1e-3):.2e}")
        eng.step()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
