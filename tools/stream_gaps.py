"""Per-stream busy time vs wall time of the pipelined C3 step (prefetch 2),
from a CUPTI trace: is the main stream idle between kernels, or are its
kernels stretched by the side-stream view build?

    python tools/stream_gaps.py --steps 20
"""

from __future__ import annotations

import argparse
import collections
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--prefetch", type=int, default=2)
    ap.add_argument("--stream-targets", action="store_true", help="targets in pinned host memory (e2e path)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(pts, (1.0, 0.2, 0.2))
    targets = [sp.edited[i] for i in range(len(cams))]
    if a.stream_targets:
        targets = [t.cpu().pin_memory() for t in targets]
    eng = RefitEngine(ds, sh0.clone(), cams, targets, P.OptimizerConfig(),
                      seed=7, cache_views=False, prefetch=a.prefetch)
    for _ in range(8):
        eng.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(a.steps):
            eng.step()
        torch.cuda.synchronize()
    eng.drain()
    eng.close()
    path = os.path.join(tempfile.mkdtemp(), "t.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    t0 = min(e["ts"] for e in ks)
    t1 = max(e["ts"] + e["dur"] for e in ks)
    by = collections.defaultdict(list)
    for e in ks:
        by[e["args"].get("stream", e.get("tid"))].append((e["ts"], e["ts"] + e["dur"], e["name"]))
    wall = t1 - t0
    # launch slack: kernel start - end of its cudaLaunchKernel (via correlation id);
    # near zero means the GPU was waiting for the host to enqueue it
    api = {e["args"].get("correlation"): e for e in ev
           if e.get("cat") == "cuda_runtime" and "dur" in e and "args" in e}
    slack = collections.defaultdict(list)
    for e in ks:
        c = e["args"].get("correlation")
        if c in api:
            slack[e["args"].get("stream")].append(e["ts"] - (api[c]["ts"] + api[c]["dur"]))
    for sid, v in slack.items():
        v.sort()
        n = len(v)
        print(f"stream {sid}: launch slack p10 {v[n // 10]:.0f} p50 {v[n // 2]:.0f} us; "
              f"{sum(1 for x in v if x < 15)} of {n} ops started < 15 us after their launch call")
    print(f"wall {wall:.0f} us over {a.steps} steps = {wall / a.steps:.1f} us/step")
    for sid, iv in sorted(by.items(), key=lambda kv: -sum(b - a_ for a_, b, _ in kv[1])):
        iv.sort()
        busy = sum(b - a_ for a_, b, _ in iv)
        gaps = collections.Counter()
        for (a0, b0, n0), (a1, b1, n1) in zip(iv, iv[1:]):
            g = a1 - b0
            if g > 2:
                gaps[(n0.split("(")[0][-40:], n1.split("(")[0][-40:])] += g
        print(f"stream {sid}: {len(iv)} ops, busy {busy / a.steps:.1f} us/step ({100 * busy / wall:.0f}% of wall)")
        for (x, y), g in gaps.most_common(8):
            print(f"    gap {g / a.steps:7.1f} us/step  after {x}  before {y}")


if __name__ == "__main__":
    main()
