"""Where the C5 frame's time goes: CUDA events around the optimizer step and each
part of the viewer frame (colour, depth, cloud projection, RGBA render, readback),
host wall time around the whole frame.

    python tools/c5_breakdown.py
"""

from __future__ import annotations

import concurrent.futures
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402
from paper_2511_18441_b200.selection import project_cloud_device  # noqa: E402
from paper_2511_18441_b200.synthetic import ring_cameras  # noqa: E402


def main():
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(pts, (1.0, 0.2, 0.2))
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=11, cache_views=False, prefetch=2)
    intr = cams[0][0]
    orbit = ring_cameras(intr.width, intr.height, 60)
    side = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
    pool = concurrent.futures.ThreadPoolExecutor(1)
    host = torch.empty((intr.height, intr.width, 4), dtype=torch.uint8, pin_memory=True)
    dev = torch.cuda.current_device()

    def build(ci, cp):
        torch.cuda.set_device(dev)
        with torch.cuda.stream(side):
            v = D.View(ds, ci, cp, P.DEFAULT_CONFIG)
            ev = torch.cuda.Event()
            ev.record(side)
        return v, ev

    names = ["step", "colour", "depth", "project", "rgba", "readback"]
    rows, walls = [], []
    for f in range(65):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ci, cp = orbit[f % 60]
        fut = pool.submit(build, ci, cp)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        ev[0].record()
        eng.step()
        ev[1].record()
        v, bev = fut.result()
        torch.cuda.current_stream().wait_event(bev)
        v.color(eng.sh)
        ev[2].record()
        depth = v.depth(0.5)
        ev[3].record()
        mask = project_cloud_device(pts, ci, cp, depth, 5, 0.02)
        ev[4].record()
        rgba = v.render_rgba(mask)
        ev[5].record()
        host.copy_(rgba, non_blocking=True)
        ev[6].record()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
        with torch.cuda.stream(side):
            side.wait_stream(torch.cuda.current_stream())
            v.close()
        if f >= 5:
            rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(6)])
    pool.shutdown()
    eng.drain()
    eng.close()
    r = np.median(np.array(rows), axis=0)
    print("median ms per part: " + ", ".join(f"{n} {x:.3f}" for n, x in zip(names, r)))
    print(f"sum of parts {r.sum():.3f} ms; wall p50 {np.median(walls[5:]):.3f} ms")


if __name__ == "__main__":
    main()
