"""e2e decomposition: BackgroundOptimizer.start() over `steps` steps (timed between
metrics-sink calls) with the targets streamed from pinned host memory vs resident
on the device, against the bare engine loop.

    python tools/e2e_probe.py --steps 200
"""

from __future__ import annotations

import argparse
import os
import sys
import threading
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import device as D  # noqa: E402
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(D.to_device(cloud.points, torch.float64), (1.0, 0.2, 0.2))
    edited = sp.edited.cpu()
    masks = sp.masks.cpu().numpy().astype(bool)
    views = tuple(P.EditedView(view=SimpleNamespace(view_id=i, intrinsics=cams[i][0], pose=cams[i][1]),
                               mask=masks[i], image=edited[i].numpy()) for i in range(len(cams)))
    dset = P.EditedDataset(views=views, generation=0, tint=np.array([1.0, 0.2, 0.2]))
    warm = 20
    for streamed, depth, nc in ((True, 2, "1"), (True, 2, "2"), (False, 2, "2")):
        os.environ["RCGS_UPLOAD_STREAMS"] = nc
        marks, count, done = {}, [0], threading.Event()

        def sink(m):
            count[0] += 1
            if count[0] == warm:
                marks["t0"] = time.perf_counter()
            if count[0] == warm + a.steps:
                marks["t1"] = time.perf_counter()
                done.set()

        opt = P.BackgroundOptimizer(scene, dset, P.OptimizerConfig(), seed=7, metrics_sink=sink, cache_views=False,
                                    stream_targets=streamed, prefetch=depth)
        torch.cuda.synchronize()
        opt.start()
        done.wait(600)
        opt.stop()
        print(f"BackgroundOptimizer.start(), targets {'streamed' if streamed else 'resident'}, prefetch {depth}, upload streams {nc}: "
              f"{a.steps / (marks['t1'] - marks['t0']):.1f} steps/s")
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=7, cache_views=False, prefetch=2)
    for _ in range(warm):
        eng.step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(a.steps):
        eng.step()
        if i % 10 == 9:
            eng.drain(wait=False)
    eng.drain()
    torch.cuda.synchronize()
    print(f"bare engine loop (main thread): {a.steps / (time.perf_counter() - t0):.1f} steps/s")
    eng.close()


if __name__ == "__main__":
    main()
