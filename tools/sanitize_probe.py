"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
smoke() plus a few C1 refit steps through the pipelined engine (prefetching
side streams, fused colour epilogue, persistent raster / record / Adam kernels
with self-resetting work counters) and one selection pass.

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import __graft_entry__  # noqa: E402
import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    __graft_entry__.smoke()
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS["c1"]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(D.to_device(cloud.points, torch.float64), (1.0, 0.2, 0.2))
    targets = [sp.edited[i] for i in range(len(cams))]
    for prefetch in (0, 2):
        eng = RefitEngine(ds, sh0.clone(), cams, targets, P.OptimizerConfig(), seed=7, cache_views=prefetch == 0,
                          prefetch=prefetch)
        for _ in range(steps):
            eng.step()
        eng.drain()
        eng.close()
    torch.cuda.synchronize()
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
