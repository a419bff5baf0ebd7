"""Float64 restatement of the reference preprocess + dense compositor.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows
/root/reference/pkg/src/splattint/render.py and scene.py; inputs are duck-typed
(``scene.positions/rotations/scales/opacities/sh/sh_degree``,
``intr.fx/fy/cx/cy/width/height``, ``pose.rotation/translation``) so the same
functions accept reference objects, product objects or plain namespaces.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import (ALPHA_CLAMP, ALPHA_SKIP, COV_DILATION, DEPTH_TAU, FOOTPRINT_SIGMAS,
                     NEAR_CLIP, SH_C0, SH_C1, SH_C2, SH_C3, T_FLOOR)


def quat_to_rot(q):
    """(w, x, y, z) unit quaternions -> (..., 3, 3); scene.py:98-112."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = (q[..., i] for i in range(4))
    r = np.empty(q.shape[:-1] + (3, 3))
    r[..., 0, 0] = 1 - 2 * (y * y + z * z)
    r[..., 0, 1] = 2 * (x * y - w * z)
    r[..., 0, 2] = 2 * (x * z + w * y)
    r[..., 1, 0] = 2 * (x * y + w * z)
    r[..., 1, 1] = 1 - 2 * (x * x + z * z)
    r[..., 1, 2] = 2 * (y * z - w * x)
    r[..., 2, 0] = 2 * (x * z - w * y)
    r[..., 2, 1] = 2 * (y * z + w * x)
    r[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def sh_basis(d, degree):
    """Real SH basis, (..., 16), zero past `degree`; render.py:103-137."""
    d = np.asarray(d, dtype=np.float64)
    b = np.zeros(d.shape[:-1] + (16,))
    b[..., 0] = SH_C0
    if degree >= 1:
        x, y, z = d[..., 0], d[..., 1], d[..., 2]
        b[..., 1] = -SH_C1 * y
        b[..., 2] = SH_C1 * z
        b[..., 3] = -SH_C1 * x
    if degree >= 2:
        xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
        b[..., 4] = SH_C2[0] * xy
        b[..., 5] = SH_C2[1] * yz
        b[..., 6] = SH_C2[2] * (2.0 * zz - xx - yy)
        b[..., 7] = SH_C2[3] * xz
        b[..., 8] = SH_C2[4] * (xx - yy)
    if degree >= 3:
        b[..., 9] = SH_C3[0] * y * (3.0 * xx - yy)
        b[..., 10] = SH_C3[1] * xy * z
        b[..., 11] = SH_C3[2] * y * (4.0 * zz - xx - yy)
        b[..., 12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy)
        b[..., 13] = SH_C3[4] * x * (4.0 * zz - xx - yy)
        b[..., 14] = SH_C3[5] * z * (xx - yy)
        b[..., 15] = SH_C3[6] * x * (xx - 3.0 * yy)
    return b


def camera_center(pose):
    """scene.py:72-75."""
    return -pose.rotation.T @ pose.translation


@dataclass
class Projected:
    """Depth-sorted kept gaussians (render.py:151-169 `_Projection`)."""

    index: np.ndarray       # (K,) scene index, front to back
    mean2d: np.ndarray      # (K, 2)
    conic_a: np.ndarray
    conic_b: np.ndarray
    conic_c: np.ndarray
    depth: np.ndarray       # (K,) view-space z
    color: np.ndarray       # (K, 3)
    opacity: np.ndarray     # (K,)
    active: np.ndarray      # (K, 3) bool
    basis: np.ndarray       # (K, 16)
    cov_xx: np.ndarray      # (K,) dilated cov2d diagonal (footprint extents)
    cov_yy: np.ndarray

    @property
    def count(self):
        return len(self.index)


def project(scene, intr, pose, sh=None) -> Projected:
    """Preprocess + global stable depth sort; render.py:172-229.

    The world->camera transform is numpy's ``P @ R.T + t`` exactly as the
    reference evaluates it (render.py:175); on OpenBLAS hosts this equals the
    FMA chain restated in oracle/c/rcgs_oracle.c (checked by the tests).
    """
    sh = scene.sh if sh is None else sh
    rot, tr = pose.rotation, pose.translation
    view = scene.positions @ rot.T + tr
    idx = np.nonzero(view[:, 2] > NEAR_CLIP)[0]
    view = view[idx]
    x, y, z = view[:, 0], view[:, 1], view[:, 2]
    fx, fy = intr.fx, intr.fy
    mean2d = np.stack([fx * x / z + intr.cx, fy * y / z + intr.cy], axis=1)

    m = quat_to_rot(scene.rotations[idx]) * scene.scales[idx][:, None, :]
    cov3 = m @ np.swapaxes(m, -1, -2)                      # render.py:95-100
    jac = np.zeros((len(idx), 2, 3))
    jac[:, 0, 0] = fx / z
    jac[:, 0, 2] = -fx * x / (z * z)
    jac[:, 1, 1] = fy / z
    jac[:, 1, 2] = -fy * y / (z * z)
    t = jac @ rot
    cov2 = np.einsum("nij,njk,nlk->nil", t, cov3, t)      # render.py:191-194
    a = cov2[:, 0, 0] + COV_DILATION
    b = cov2[:, 0, 1]
    c = cov2[:, 1, 1] + COV_DILATION
    det = a * c - b * b
    mid = 0.5 * (a + c)
    radius = FOOTPRINT_SIGMAS * np.sqrt(mid + np.sqrt(np.maximum(mid * mid - det, 0.0)))
    w1, h1 = intr.width - 1, intr.height - 1
    vis = ((det > 0) & (mean2d[:, 0] + radius >= 0) & (mean2d[:, 0] - radius <= w1)
           & (mean2d[:, 1] + radius >= 0) & (mean2d[:, 1] - radius <= h1))
    idx, mean2d, z = idx[vis], mean2d[vis], z[vis]
    a, b, c, det = a[vis], b[vis], c[vis], det[vis]

    d = scene.positions[idx] - camera_center(pose)          # render.py:209-214
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    basis = sh_basis(d, scene.sh_degree)
    raw = np.einsum("nk,nkc->nc", basis, np.asarray(sh, dtype=np.float64)[idx])
    order = np.argsort(z, kind="stable")                    # render.py:216
    return Projected(
        index=idx[order], mean2d=mean2d[order],
        conic_a=(c / det)[order], conic_b=(-b / det)[order], conic_c=(a / det)[order],
        depth=z[order], color=np.maximum(0.0, raw + 0.5)[order],
        opacity=np.asarray(scene.opacities, dtype=np.float64)[idx[order]],
        active=((raw + 0.5) > 0.0)[order], basis=basis[order],
        cov_xx=a[order], cov_yy=c[order])


def subset(p: Projected, sel) -> Projected:
    return Projected(*(getattr(p, f)[sel] for f in Projected.__dataclass_fields__))


def alpha_block(p: Projected, xs, ys):
    """(B, W, K) alpha with the skip threshold applied; render.py:263-272."""
    dx = xs[:, None] - p.mean2d[None, :, 0]
    dy = ys[:, None] - p.mean2d[None, :, 1]
    power = -(0.5 * p.conic_a * dx * dx)[None, :, :] \
        - (0.5 * p.conic_c * dy * dy)[:, None, :] \
        - p.conic_b * dx[None, :, :] * dy[:, None, :]
    alpha = np.minimum(ALPHA_CLAMP, p.opacity * np.exp(power))
    alpha[alpha < ALPHA_SKIP] = 0.0
    return alpha


def weights_block(alpha):
    """Composite weights, final T and stop index; render.py:275-292."""
    k = alpha.shape[-1]
    t_inc = np.cumprod(1.0 - alpha, axis=-1)
    t_exc = np.concatenate([np.ones(t_inc.shape[:-1] + (1,)), t_inc[..., :-1]], axis=-1)
    below = t_inc < T_FLOOR
    anyb = below.any(axis=-1)
    first = np.where(anyb, np.argmax(below, axis=-1), k)
    alive = np.arange(k) < first[..., None]
    w = alpha * t_exc * alive
    t_final = np.where(anyb, np.take_along_axis(
        t_exc, np.minimum(first, k - 1)[..., None], axis=-1)[..., 0], t_inc[..., -1])
    return w, t_final, first, t_inc


def _chunks(h, w, k, budget=1 << 22):
    """Row/column chunks bounding peak memory; per-pixel results are
    independent of the chunking (the reference uses row blocks of <= 2^20
    entries, render.py:49-51, 257-260)."""
    cols = max(1, min(w, budget // max(1, k)))
    rows = max(1, min(h, budget // max(1, cols * k)))
    for y0 in range(0, h, rows):
        for x0 in range(0, w, cols):
            yield y0, min(y0 + rows, h), x0, min(x0 + cols, w)


def render_forward(scene, intr, pose, background=None, sh=None, capture=True):
    """Image (H, W, 3) f64 + contribution lists; render.py:304-370."""
    bg = np.zeros(3) if background is None else np.asarray(background, dtype=np.float64)
    p = project(scene, intr, pose, sh)
    h, w = intr.height, intr.width
    img = np.empty((h, w, 3))
    t_fin = np.ones((h, w))
    pix, kept, wts = [], [], []
    if p.count == 0:
        img[:] = bg
    else:
        for y0, y1, x0, x1 in _chunks(h, w, p.count):
            a = alpha_block(p, np.arange(x0, x1, dtype=np.float64),
                            np.arange(y0, y1, dtype=np.float64))
            wb, tf, _, _ = weights_block(a)
            img[y0:y1, x0:x1] = np.einsum("bwk,kc->bwc", wb, p.color) + tf[..., None] * bg
            t_fin[y0:y1, x0:x1] = tf
            if capture:
                bi, wi, ki = np.nonzero(wb)
                pix.append(((y0 + bi) * w + x0 + wi).astype(np.int64))
                kept.append(ki.astype(np.int64))
                wts.append(wb[bi, wi, ki])
    if capture and pix:
        pix, kept, wts = np.concatenate(pix), np.concatenate(kept), np.concatenate(wts)
        order = np.lexsort((kept, pix))     # reference order: pixel-major, then depth
        pix, kept, wts = pix[order], kept[order], wts[order]
    else:
        pix, kept, wts = (np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0))
    return dict(image=img, t_final=t_fin, proj=p, n=len(scene.positions),
                contrib_pixel=pix, contrib_kept=kept, contrib_weight=wts)


def render(scene, intr, pose, background=None, sh=None):
    """render.py:304-334 (HWC)."""
    return render_forward(scene, intr, pose, background, sh, capture=False)["image"]


def depth(scene, intr, pose, tau=DEPTH_TAU):
    """depth_from_gaussians, render.py:373-398."""
    p = project(scene, intr, pose)
    h, w = intr.height, intr.width
    out = np.full((h, w), np.inf)
    if p.count == 0:
        return out
    for y0, y1, x0, x1 in _chunks(h, w, p.count):
        a = alpha_block(p, np.arange(x0, x1, dtype=np.float64),
                        np.arange(y0, y1, dtype=np.float64))
        t_inc = np.cumprod(1.0 - a, axis=-1)
        crossed = (t_inc < tau) & (a > 0.0)
        has = crossed.any(axis=-1)
        idx = np.argmax(crossed, axis=-1)
        below = t_inc < T_FLOOR
        stop = np.where(below.any(axis=-1), np.argmax(below, axis=-1), p.count)
        out[y0:y1, x0:x1] = np.where(has & (idx <= stop), p.depth[idx], np.inf)
    return out


# --- sparse per-pixel oracle (large configs) ----------

def footprint_extent(p: Projected, slack=1e-6):
    """Per-axis half extents of the alpha >= 1/255 ellipse.

    alpha >= 1/255  <=>  d^T conic d <= 2 ln(255 sigma); the ellipse's
    axis-aligned half widths are sqrt(2 ln(255 sigma) * cov_xx) and
    sqrt(... * cov_yy).  Gaussians with sigma <= 1/255 reach no pixel.
    """
    r2 = 2.0 * np.log(np.maximum(255.0 * p.opacity, 1e-300))
    r2 = np.where(255.0 * p.opacity > 1.0, r2, -1.0)
    ex = np.sqrt(np.maximum(r2 * p.cov_xx, 0.0)) * (1 + slack) + slack
    ey = np.sqrt(np.maximum(r2 * p.cov_yy, 0.0)) * (1 + slack) + slack
    return ex, ey, r2 > 0


def sparse_pixels(p: Projected, us, vs, background=None, tau=DEPTH_TAU):
    """Exact per-pixel render/depth/weights at sampled integer pixels.

    Entries whose footprint box excludes the pixel have alpha < 1/255, which the
    dense path multiplies into T as exactly 1.0 and weights as 0
    (render.py:271, 278), so restricting the depth-sorted list to the entries
    whose box contains the pixel reproduces the dense result bit-for-bit.
    Returns colour (P, 3), T_final (P,), depth (P,), and per pixel the list of
    (kept_index, weight) contributions.
    """
    bg = np.zeros(3) if background is None else np.asarray(background, dtype=np.float64)
    ex, ey, reach = footprint_extent(p)
    cols, tfs, deps, contribs = [], [], [], []
    for u, v in zip(us, vs):
        sel = np.nonzero(reach & (np.abs(u - p.mean2d[:, 0]) <= ex)
                         & (np.abs(v - p.mean2d[:, 1]) <= ey))[0]
        if len(sel) == 0:
            cols.append(bg.copy()); tfs.append(1.0); deps.append(np.inf); contribs.append(([], []))
            continue
        sub = subset(p, sel)
        a = alpha_block(sub, np.array([float(u)]), np.array([float(v)]))
        wb, tf, first, t_inc = weights_block(a)
        cols.append(wb[0, 0] @ sub.color + tf[0, 0] * bg)
        tfs.append(tf[0, 0])
        crossed = (t_inc[0, 0] < tau) & (a[0, 0] > 0)
        if crossed.any() and np.argmax(crossed) <= first[0, 0]:
            deps.append(sub.depth[np.argmax(crossed)])
        else:
            deps.append(np.inf)
        nz = np.nonzero(wb[0, 0])[0]
        contribs.append((sel[nz], wb[0, 0][nz]))
    return np.array(cols), np.array(tfs), np.array(deps), contribs
