"""Select-from-mask outlier filter at interactive scale: GPU knn_mean_distances
vs scipy cKDTree on a surface-like cloud of `--points` points (a full-frame 1080p
selection unprojects ~1.4M), checking the results are identical.

    python tools/knn_probe.py --points 1400000
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_18441_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=1_400_000)
    ap.add_argument("--k", type=int, default=16)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    n = a.points
    u, v = rng.uniform(0, 1.6, n), rng.uniform(0, 0.9, n)
    pts = np.stack([u, v, 2.0 + 0.2 * np.sin(4 * u) * np.cos(3 * v) + 0.002 * rng.normal(size=n)], axis=1)
    P.knn_mean_distances(pts[:20000], a.k)  # warm-up (library, context)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = P.knn_mean_distances(pts, a.k)
    t_gpu = time.perf_counter() - t0
    from scipy.spatial import cKDTree
    t0 = time.perf_counter()
    d, _ = cKDTree(pts).query(pts, k=a.k + 1, workers=-1)
    ref = d[:, 1:].mean(axis=1)
    t_cpu = time.perf_counter() - t0
    print(f"points {n} k {a.k}: GPU {t_gpu * 1e3:.1f} ms (incl. H2D/D2H), scipy cKDTree (all cores) "
          f"{t_cpu * 1e3:.1f} ms, identical: {np.array_equal(got, ref)}")


if __name__ == "__main__":
    main()
