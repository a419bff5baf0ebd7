"""Tile-list length distribution of C3 views (max, p99, mean, tiles over 2048 /
4096 entries, pairs): the input to the segmented-depth-sort evaluation in DESIGN.md.

    python tools/tile_lengths.py
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402


def main():
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    for i in range(0, len(cams), max(1, len(cams) // 8)):
        v = D.View(ds, cams[i][0], cams[i][1], P.DEFAULT_CONFIG)
        r = v.ranges().view(-1, 2).cpu().numpy().astype(np.int64)
        lens = r[:, 1] - r[:, 0]
        print(f"view {i:2d}: max {lens.max()}, p99 {np.percentile(lens, 99):.0f}, mean {lens.mean():.1f}, "
              f"> 2048: {(lens > 2048).sum()}, > 4096: {(lens > 4096).sum()}, pairs {v.n_pairs}")
        v.close()


if __name__ == "__main__":
    main()
