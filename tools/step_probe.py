"""Minimal driver for ncu: builds a benchmark workload and runs a few optimizer
steps (and one selection pass over `--sel-views` views) so the launch list /
full capture covers exactly the hot path.

    python tools/step_probe.py --config c3 --steps 3
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--sel-views", type=int, default=0, help="0 = all views")
    ap.add_argument("--cache-views", action="store_true")
    ap.add_argument("--prefetch", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[a.config]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(pts, (1.0, 0.2, 0.2), indices=list(range(a.sel_views)) if a.sel_views else None)
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=7, cache_views=a.cache_views, prefetch=a.prefetch)
    for _ in range(a.warmup):
        eng.step()
    torch.cuda.synchronize()
    # the timed steps are bracketed by cudaProfilerStart/Stop: run ncu with
    # --profile-from-start off to capture only them
    torch.cuda.profiler.start()
    for _ in range(a.steps):
        eng.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    eng.drain()
    torch.cuda.synchronize()
    print("probe ok", eng.step_count())


if __name__ == "__main__":
    main()
