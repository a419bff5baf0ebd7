"""Fraction of 32x32 loss blocks that are dirty (render != edited target) during
a C3 refit, and within one / two blocks of a dirty block (the loss passes'
active sets), after 1, 20 and 100 optimizer steps.

    python tools/dirty_blocks.py
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy.ndimage import binary_dilation  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def main():
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(D.to_device(cloud.points, torch.float64), (1.0, 0.2, 0.2))
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=7, cache_views=False)
    done = 0
    for target in (1, 20, 100):
        while done < target:
            eng.step()
            done += 1
        fr = []
        for i in range(0, len(cams), 8):
            intr, pose = cams[i]
            v = D.View(ds, intr, pose, P.DEFAULT_CONFIG)
            img = v.color(eng.sh).render(None, 0)
            v.close()
            d = (img != sp.edited[i]).any(dim=2).cpu().numpy()
            h, w = d.shape
            pad = np.zeros(((h + 31) // 32 * 32, (w + 31) // 32 * 32), bool)
            pad[:h, :w] = d
            blk = pad.reshape(pad.shape[0] // 32, 32, pad.shape[1] // 32, 32).any(axis=(1, 3))
            fr.append((blk.mean(), binary_dilation(blk, np.ones((3, 3), bool)).mean(),
                       binary_dilation(blk, np.ones((5, 5), bool)).mean()))
        print(f"after {target} steps: dirty / within 1 / within 2 blocks: {np.round(np.mean(fr, axis=0), 3)}")
    eng.drain()
    eng.close()


if __name__ == "__main__":
    main()
