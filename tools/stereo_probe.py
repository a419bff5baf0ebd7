"""Stereo depth at benchmark scale: device stereo_hv_depth (+ gaussian backfill)
on a C3 view (1M gaussians, 1080p) -- wall time with CUDA events and the
per-kernel split from CUPTI (torch.profiler).

    python tools/stereo_probe.py [--config c3] [--reps 5]
"""

from __future__ import annotations

import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import stereo as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS[a.config], 0, torch.device("cuda", 0))
    intr, pose = cams[0]
    base = S.default_baseline(scene)
    run = lambda: S.stereo_hv_depth_device(ds, sh0, intr, pose, base, backfill_tau=0.5)  # noqa: E731
    out = run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        out = run()
    e1.record()
    torch.cuda.synchronize()
    print(f"stereo-hv depth {intr.width}x{intr.height}: {e0.elapsed_time(e1) / a.reps:.2f} ms/view, "
          f"finite {torch.isfinite(out).double().mean().item():.3f}")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.split("(")[0].replace("void ", "")[:60]
            agg[k][0] += 1
            agg[k][1] += ev.device_time_total
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"{us:10.1f} us {c:4d}x  {k}")
    print(f"{sum(v[1] for v in agg.values()):10.1f} us total")


if __name__ == "__main__":
    main()
