"""Float64 restatement of the stereo depth path (stereo.py:87-219 of
/root/reference/pkg/src/splattint).

TEST INFRASTRUCTURE ONLY -- the checker for csrc/stereo.cu, never on the
product path.  The box means are scipy.ndimage.uniform_filter(mode="nearest")
itself (scipy 1.18.1 in this image, the reference's own dependency), so the
restatement is pinned to the reference's numerics; tests/golden/stereo_*.npz
(made by the reference, tests/golden/make_stereo_golden.py) pin it further.
"""

from __future__ import annotations

import numpy as np
from scipy.ndimage import uniform_filter

INVALID = -1.0


def gray(img):
    a = np.asarray(img, np.float64)
    return a.mean(axis=2) if a.ndim == 3 else a


def box(a, r):
    return uniform_filter(a, size=2 * r + 1, mode="nearest")


def zncc_volume(lft, rgt, max_disp, r, floor):
    """(max_disp + 1, H, W) scores, -2 where invalid -- stereo.py:97-118."""
    h, w = lft.shape
    mu_l = box(lft, r)
    var_l = box(lft * lft, r) - mu_l * mu_l
    vol = np.full((max_disp + 1, h, w), -2.0)
    col = np.arange(w)
    for d in range(min(max_disp + 1, w)):
        # column x of the shifted image is column max(x - d, 0) of the right image
        sh = rgt[:, np.maximum(col - d, 0)]
        mu_r = box(sh, r)
        var_r = box(sh * sh, r) - mu_r * mu_r
        cov = box(lft * sh, r) - mu_l * mu_r
        good = (var_l >= floor) & (var_r >= floor) & (col >= d)
        vol[d] = np.where(good, cov / np.sqrt(np.maximum(var_l * var_r, floor ** 2)), -2.0)
    return vol


def refine(vol):
    """argmax (first) + parabolic refinement -- stereo.py:121-139."""
    nd = vol.shape[0]
    k = np.argmax(vol, axis=0)
    pick = lambda idx: np.take_along_axis(vol, idx[None], axis=0)[0]  # noqa: E731
    s0, sm, sp = pick(k), pick(np.maximum(k - 1, 0)), pick(np.minimum(k + 1, nd - 1))
    out = np.where(s0 <= -2.0, INVALID, k.astype(np.float64))
    den = sm + sp - 2.0 * s0
    ok = (k > 0) & (k < nd - 1) & (sm > -2.0) & (sp > -2.0) & (s0 > -2.0) & (den < -1e-12)
    with np.errstate(divide="ignore", invalid="ignore"):
        step = np.clip(0.5 * (sm - sp) / den, -0.5, 0.5)
    return np.where(ok, k + step, out)


def match(left, right, max_disp=64, r=5, floor=1e-6, tol=1.0):
    """match_disparity -- stereo.py:142-161."""
    gl, gr = gray(left), gray(right)
    dl = refine(zncc_volume(gl, gr, max_disp, r, floor))
    dr = refine(zncc_volume(gr[:, ::-1], gl[:, ::-1], max_disp, r, floor))[:, ::-1]
    h, w = gl.shape
    partner = np.rint(np.arange(w)[None, :] - dl).astype(np.int64)
    ok = (dl >= 0.0) & (partner >= 0) & (partner < w)
    other = np.full_like(dl, INVALID)
    yy = np.broadcast_to(np.arange(h)[:, None], (h, w))
    other[ok] = dr[yy[ok], partner[ok]]
    keep = ok & (other >= 0.0) & (np.abs(dl - other) <= tol)
    return np.where(keep, dl, INVALID)


def to_depth(disp, f, baseline, min_disp=1e-3):
    out = np.full(disp.shape, np.inf)
    m = disp > min_disp
    out[m] = f * baseline / disp[m]
    return out


def hv_depth(left, right_h, right_v, fx, fy, baseline, max_disp=64, r=5, floor=1e-6, tol=1.0, min_disp=1e-3,
             fallback=None):
    """stereo_hv_depth (+ estimate_depth's backfill) from the three renders -- stereo.py:184-219."""
    dh = match(left, right_h, max_disp, r, floor, tol)
    dv = match(np.swapaxes(left, 0, 1), np.swapaxes(right_v, 0, 1), max_disp, r, floor, tol).T
    fused = np.minimum(to_depth(dh, fx, baseline, min_disp), to_depth(dv, fy, baseline, min_disp))
    if fallback is not None:
        fused = np.where(np.isfinite(fused), fused, fallback)
    return fused
