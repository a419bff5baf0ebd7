"""Load-balance probe for the persistent rasteriser: traces one render and one
backward launch of a benchmark view (rcgs_raster_trace) and prints the launch
span, per-SM busy time and the slowest work items with their work counts.

    python tools/raster_trace.py --config c3 --view 0
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import _native as N  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402


def report(name, tr, ranges):
    tr = tr[(tr[:, 0] != 0) | (tr[:, 1] != 0)]  # items skipped before tracing stay zero
    t0 = tr[:, 0].astype(np.int64)
    t1 = tr[:, 1].astype(np.int64)
    base = t0.min()
    t0 -= base
    t1 -= base
    dur = t1 - t0
    span = t1.max()
    print(f"== {name}: {len(tr)} items, span {span / 1e3:.1f} us, item mean {dur.mean() / 1e3:.2f} us, "
          f"sum {dur.sum() / 1e6:.1f} warp-ms")
    sm = tr[:, 2]
    ends = np.zeros(sm.max() + 1)
    busy = np.zeros(sm.max() + 1)
    np.maximum.at(ends, sm, t1)
    np.add.at(busy, sm, dur)
    print(f"   SM last end: min {ends.min() / 1e3:.1f} p50 {np.median(ends) / 1e3:.1f} max {ends.max() / 1e3:.1f} us;"
          f" items ending after 60% of span: {(t1 > 0.6 * span).sum()}")
    for q in (50, 90, 99, 99.9):
        print(f"   item duration p{q}: {np.percentile(dur, q) / 1e3:.2f} us")
    lens = ranges[:, 1] - ranges[:, 0]
    top = np.argsort(-dur)[:12]
    print("   slowest items: dur_us start_us iters evals exact resync tile_len")
    for i in top:
        print(f"   {dur[i] / 1e3:8.1f} {t0[i] / 1e3:8.1f} {tr[i, 3]:6d} {tr[i, 4]:7d} {tr[i, 5]:6d} {tr[i, 6]:6d} "
              f"{lens[tr[i, 7]]:6d}")
    late = np.argsort(-t1)[:8]
    print("   last-finishing items: end_us dur_us iters tile_len")
    for i in late:
        print(f"   {t1[i] / 1e3:8.1f} {dur[i] / 1e3:8.1f} {tr[i, 3]:6d} {lens[tr[i, 7]]:6d}")
    print(f"   totals: iters {tr[:, 3].sum()} evals {tr[:, 4].sum()} exact {tr[:, 5].sum()} "
          f"resync {tr[:, 6].sum()}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--view", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS[a.config]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, dev)
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(pts, (1.0, 0.2, 0.2), indices=[a.view])
    target = sp.edited[a.view]
    intr, pose = cams[a.view]
    v = D.View(ds, intr, pose, P.DEFAULT_CONFIG)
    v.color(sh0)
    h, w = v.height, v.width
    img = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    grad = torch.empty_like(img)
    acc = torch.zeros((ds.n, 3), dtype=torch.float32, device=dev)
    rec = torch.zeros(4, dtype=torch.float64, device=dev)
    v.render(None, 0, out=img)
    D.loss_grad(img, target, 0.2, loss3=rec[:3], grad=grad)
    v.backward(grad, acc=acc)
    torch.cuda.synchronize()
    n_items = v.tiles[0] * v.tiles[1] * 8
    tr = torch.zeros((n_items, 8), dtype=torch.int32, device=dev)
    ranges = v.ranges().view(-1, 2).cpu().numpy().astype(np.int64)
    N.call("rcgs_raster_trace", N.ptr(tr), n_items)
    v.render(None, 0, out=img)
    torch.cuda.synchronize()
    fwd = tr.cpu().numpy().view(np.uint32).copy()
    tr.zero_()
    v.backward(grad, acc=acc)
    torch.cuda.synchronize()
    bwd = tr.cpu().numpy().view(np.uint32).copy()
    N.call("rcgs_raster_trace", None, 0)
    lens = ranges[:, 1] - ranges[:, 0]
    print(f"view {a.view}: kept {v.n_kept} pairs {v.n_pairs}; tile entries mean {lens.mean():.0f} "
          f"p99 {np.percentile(lens, 99):.0f} max {lens.max()}")
    report("render", fwd, ranges)
    report("backward (all items, skipped ones have ~0 duration)", bwd, ranges)


if __name__ == "__main__":
    main()
