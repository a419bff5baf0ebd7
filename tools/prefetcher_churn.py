"""Resource churn check: 300 SelectionPass runs, each creating and closing a
view prefetcher (two builder threads + streams).  Thread count, host RSS and
device memory in use must stay flat.

    python tools/prefetcher_churn.py
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import psutil  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402


def main():
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c1"], 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    proc = psutil.Process()
    for r in range(301):
        P.SelectionPass(ds, cams, gt).run(pts, (1.0, 0.2, 0.2))
        if r % 100 == 0:
            torch.cuda.synchronize()
            free, total = torch.cuda.mem_get_info()
            print(f"run {r:3d}: threads {proc.num_threads()}, host RSS {proc.memory_info().rss / 1e6:.1f} MB, "
                  f"device in use {(total - free) / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
