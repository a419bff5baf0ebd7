"""Stage timing of the selection pass (CUDA events per stage) on a benchmark config."""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.recolor import apply_recolor_device  # noqa: E402
from paper_2511_18441_b200.selection import project_cloud_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--views", type=int, default=8)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[a.config]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    hits = torch.zeros(ds.n, dtype=torch.int32, device="cuda")
    wsum = torch.zeros(ds.n, dtype=torch.int64, device="cuda")
    names = ["build", "depth", "project", "hits", "recolor"]
    tot = {k: 0.0 for k in names}
    mask = torch.zeros((cfg["height"], cfg["width"]), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(gt[0])
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for i in range(a.views):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        intr, pose = cams[i]
        ev[0].record()
        v = D.View(ds, intr, pose, P.DEFAULT_CONFIG)
        ev[1].record()
        depth = v.depth(0.5)
        ev[2].record()
        mask.zero_()
        project_cloud_device(pts, intr, pose, depth, 5, 0.02, out=mask)
        ev[3].record()
        v.mask_hits(mask, hits, wsum)
        ev[4].record()
        apply_recolor_device(gt[i], mask, (1.0, 0.2, 0.2), out=out)
        ev[5].record()
        torch.cuda.synchronize()
        for k, n in enumerate(names):
            tot[n] += ev[k].elapsed_time(ev[k + 1])
        v.close()
    wall = time.perf_counter() - wall0
    print({k: round(v / a.views, 3) for k, v in tot.items()}, "ms/view; wall ms/view", round(1000 * wall / a.views, 3),
          "masked px (last)", int(mask.sum().item()))


if __name__ == "__main__":
    main()
