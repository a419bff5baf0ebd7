"""Soak test of the pipelined refit engine: device memory in use (driver view)
and step rate over a long run (C3, prefetch 3, two builder threads).

    python tools/soak.py --steps 3000
"""

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
from paper_2511_18441_b200.engine import RefitEngine  # noqa: E402


def used_mb():
    free, total = torch.cuda.mem_get_info()
    return (total - free) / 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(D.to_device(cloud.points, torch.float64), (1.0, 0.2, 0.2))
    eng = RefitEngine(ds, sh0.clone(), cams, [sp.edited[i] for i in range(len(cams))], P.OptimizerConfig(),
                      seed=7, cache_views=False, prefetch=3)
    chunk = a.steps // 10
    for c in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(chunk):
            eng.step()
        eng.drain(wait=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"steps {(c + 1) * chunk:6d}: {chunk / dt:7.1f} steps/s, device memory in use {used_mb():9.1f} MB",
              flush=True)
    out = eng.drain()
    eng.close()
    print(f"metrics drained: {len(out)}; last loss {out[-1][4] if out else None}")


if __name__ == "__main__":
    main()
