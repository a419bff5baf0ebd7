"""Host-issue vs device time of the refit loop (is the step launch-bound?)."""

from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def main():
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt).run(pts, (1.0, 0.2, 0.2))
    targets = [sp.edited[i] for i in range(len(cams))]
    for cache, pf in ((False, 0), (False, 2), (True, 0)):
        eng = RefitEngine(ds, sh0.clone(), cams, targets, P.OptimizerConfig(), seed=7, cache_views=cache,
                          prefetch=pf)
        for _ in range(5):
            eng.step()
        eng.drain()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 30
        t0 = time.perf_counter()
        e0.record()
        for _ in range(K):
            eng.step()
        t_issue = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t0
        print(f"cache={cache} prefetch={pf}: host issue {1000 * t_issue / K:.3f} ms/step, "
              f"device {e0.elapsed_time(e1) / K:.3f} ms/step, wall {1000 * t_all / K:.3f} ms/step")
        eng.drain()
        eng.close()


if __name__ == "__main__":
    main()
