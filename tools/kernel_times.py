"""Per-kernel GPU durations inside the real step pipeline (warm caches, no
serialisation), from CUPTI activity records via torch.profiler -- the
complement of the ncu launch list, whose per-kernel replays flush the caches.

    python tools/kernel_times.py --config c3 --steps 20 [--prefetch 0]
"""

from __future__ import annotations

import argparse
import collections
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--prefetch", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[a.config]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(pts, (1.0, 0.2, 0.2))
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=7, cache_views=False, prefetch=a.prefetch)
    for _ in range(a.warmup):
        eng.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            eng.step()
        torch.cuda.synchronize()
    eng.drain()
    eng.close()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.split("(")[0].replace("void ", "")[:60]
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    tot = sum(v[1] for v in agg.values())
    lines = [f"# per-kernel device time inside the pipeline, {a.config}, {a.steps} steps, prefetch={a.prefetch}",
             f"{'us/step':>9} {'n/step':>6} {'us/launch':>9} {'share':>6}  kernel"]
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{us / a.steps:9.1f} {c / a.steps:6.1f} {us / c:9.2f} {100 * us / tot:5.1f}%  {k}")
    lines.append(f"{tot / a.steps:9.1f} us/step total kernel time")
    text = "\n".join(lines)
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
