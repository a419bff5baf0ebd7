"""Float64 restatement of the selection pass (cloud projection, recolor,
edited dataset) and of the host-side select-from-mask steps.

TEST INFRASTRUCTURE ONLY.  Follows selection.py:83-235 and recolor.py:30-81
of /root/reference/pkg/src/splattint.
"""

from __future__ import annotations

import numpy as np
from scipy.spatial import cKDTree

from . import raster
from .config import DEPTH_TAU, DEPTH_TOLERANCE, KNN, QUAD_SIZE, SAMPLE_FRACTION, STD_SCALE


def project_points(points, intr, pose, occ, tol=DEPTH_TOLERANCE):
    """Nearest pixel + occlusion-tested visibility; selection.py:184-206."""
    cam = points @ pose.rotation.T + pose.translation
    z = cam[:, 2]
    front = z > 0
    pu = np.full(len(points), -1, np.int64)
    pv = np.full(len(points), -1, np.int64)
    with np.errstate(divide="ignore", invalid="ignore"):
        u = intr.fx * cam[:, 0] / z + intr.cx
        v = intr.fy * cam[:, 1] / z + intr.cy
    pu[front] = np.rint(u[front]).astype(np.int64)
    pv[front] = np.rint(v[front]).astype(np.int64)
    inside = front & (pu >= 0) & (pu < intr.width) & (pv >= 0) & (pv < intr.height)
    vis = inside.copy()
    vis[inside] = z[inside] <= occ[pv[inside], pu[inside]] * (1.0 + tol)
    return pu, pv, vis


def project_cloud(points, intr, pose, occ, quad=QUAD_SIZE, tol=DEPTH_TOLERANCE):
    """(H, W) bool quads of the visible points; selection.py:209-235."""
    bits = np.zeros((intr.height, intr.width), bool)
    points = np.asarray(points, np.float64).reshape(-1, 3)
    if len(points) == 0:
        return bits
    pu, pv, vis = project_points(points, intr, pose, np.asarray(occ, np.float64), tol)
    half = (quad - 1) // 2
    for dv in range(-half, quad - half):
        for du in range(-half, quad - half):
            qu, qv = pu[vis] + du, pv[vis] + dv
            ok = (qu >= 0) & (qu < intr.width) & (qv >= 0) & (qv < intr.height)
            bits[qv[ok], qu[ok]] = True
    return bits


def apply_recolor(image, mask, tint):
    """recolor.py:30-39."""
    out = np.array(image, np.float64, copy=True)
    out[mask] = np.clip(out[mask] * np.asarray(tint, np.float64), 0.0, 1.0)
    return out


def build_edited(scene, views, points, tint, quad=QUAD_SIZE, tol=DEPTH_TOLERANCE,
                 tau=DEPTH_TAU):
    """recolor.py:59-81; views = [(intr, pose, image)] -> [(mask, edited)]."""
    out = []
    for intr, pose, image in views:
        if len(points) == 0:
            mask = np.zeros((intr.height, intr.width), bool)
        else:
            mask = project_cloud(points, intr, pose, raster.depth(scene, intr, pose, tau), quad, tol)
        out.append((mask, apply_recolor(image, mask, tint)))
    return out


def stroke_disc(height, width, center, radius):
    """Brush disc of one path point (selection.py:83-122 with a 1-point path)."""
    u0 = max(0, int(np.floor(center[0] - radius)))
    u1 = min(width - 1, int(np.ceil(center[0] + radius)))
    v0 = max(0, int(np.floor(center[1] - radius)))
    v1 = min(height - 1, int(np.ceil(center[1] + radius)))
    bits = np.zeros((height, width), bool)
    if u0 > u1 or v0 > v1:
        return bits
    du = np.arange(u0, u1 + 1, dtype=np.float64)[None, :] - center[0]
    dv = np.arange(v0, v1 + 1, dtype=np.float64)[:, None] - center[1]
    bits[v0:v1 + 1, u0:u1 + 1] = du * du + dv * dv <= radius * radius
    return bits


def unproject(bits, depth, intr, pose, fraction=SAMPLE_FRACTION, seed=0):
    """selection.py:125-152 -> (M, 3) world points."""
    vs, us = np.nonzero(bits & np.isfinite(depth) & (depth > 0))
    keep = int(round(fraction * len(us)))
    if keep == 0:
        return np.empty((0, 3))
    order = np.random.default_rng(seed).permutation(len(us))[:keep]
    us, vs = us[order], vs[order]
    d = depth[vs, us]
    cam = np.stack([d * (us - intr.cx) / intr.fx, d * (vs - intr.cy) / intr.fy, d], axis=1)
    return (cam - pose.translation) @ pose.rotation


def knn_means(points, k):
    """selection.py:155-159."""
    dists, _ = cKDTree(points).query(points, k=k + 1)
    return dists[:, 1:].mean(axis=1)


def remove_outliers(points, k=KNN, std_scale=STD_SCALE):
    """selection.py:162-181."""
    if len(points) <= k:
        return points
    means = knn_means(points, k)
    return points[means <= means.mean() + std_scale * means.std()]


def mask_hits(scene, views, masks):
    """Per-gaussian mask-hit count and masked contribution weight across
    views (north_star extension): hit[i] = sum_v #{p in
    mask_v : w_ip > 0}, wsum[i] = sum_v sum_{p in mask_v} w_ip, restated from
    the render_forward contribution lists (render.py:81-92)."""
    n = len(scene.positions)
    hit = np.zeros(n, np.int64)
    wsum = np.zeros(n)
    for (intr, pose), mask in zip(views, masks):
        cap = raster.render_forward(scene, intr, pose)
        sel = mask.ravel()[cap["contrib_pixel"]]
        gid = cap["proj"].index[cap["contrib_kept"][sel]]
        np.add.at(hit, gid, 1)
        np.add.at(wsum, gid, cap["contrib_weight"][sel])
    return hit, wsum
