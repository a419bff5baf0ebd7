"""Tile-binning oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference has no tiles: every pixel composites every kept gaussian in the
global stable depth order (render.py:216, 263-292), and an entry whose alpha
is below 1/255 at a pixel is skipped there (alpha set to exactly 0, render.py:
271).  A per-tile list therefore reproduces the reference exactly iff, for
every tile, it

1. contains every kept gaussian whose fp64 alpha (the reference's formula and
   operation order, render.py:265-271) is >= 1/255 at some pixel of the tile;
2. lists its entries in the global depth order (render.py:216).

`required_tile_sets` computes (1) exactly for the tiles of a crop by
enumerating, per gaussian, the integer pixels of its opacity-aware footprint
box inside the crop (`raster.footprint_extent`, a superset of the
alpha >= 1/255 ellipse) and evaluating alpha there in fp64.
"""

from __future__ import annotations

import numpy as np

from .config import ALPHA_CLAMP, ALPHA_SKIP
from .raster import Projected, footprint_extent


def _alpha(p: Projected, k, us, vs):
    """render.py:265-271 for entry k at pixels (us, vs), numpy's operation order."""
    dx = us - p.mean2d[k, 0]
    dy = vs - p.mean2d[k, 1]
    power = -(0.5 * p.conic_a[k] * dx * dx) - (0.5 * p.conic_c[k] * dy * dy) - p.conic_b[k] * dx * dy
    alpha = np.minimum(ALPHA_CLAMP, p.opacity[k] * np.exp(power))
    return np.where(alpha < ALPHA_SKIP, 0.0, alpha)


def required_tile_sets(p: Projected, width, height, crop, tile=16):
    """{(tx, ty): set of depth ranks k} for the tiles inside crop = (tx0, ty0, tx1, ty1)
    (inclusive tile coordinates): entries with fp64 alpha >= 1/255 at a pixel of the tile."""
    tx0, ty0, tx1, ty1 = crop
    u_lo, v_lo = tx0 * tile, ty0 * tile
    u_hi, v_hi = min((tx1 + 1) * tile, width) - 1, min((ty1 + 1) * tile, height) - 1
    ex, ey, reach = footprint_extent(p)
    mx, my = p.mean2d[:, 0], p.mean2d[:, 1]
    bu0 = np.maximum(np.ceil(mx - ex), u_lo)
    bu1 = np.minimum(np.floor(mx + ex), u_hi)
    bv0 = np.maximum(np.ceil(my - ey), v_lo)
    bv1 = np.minimum(np.floor(my + ey), v_hi)
    cand = np.nonzero(reach & (bu0 <= bu1) & (bv0 <= bv1))[0]
    out = {(tx, ty): set() for tx in range(tx0, tx1 + 1) for ty in range(ty0, ty1 + 1)}
    for k in cand:
        us = np.arange(bu0[k], bu1[k] + 1.0)
        vs = np.arange(bv0[k], bv1[k] + 1.0)
        uu, vv = np.meshgrid(us, vs)
        a = _alpha(p, k, uu, vv)
        hit = a > 0.0
        if not hit.any():
            continue
        for tx, ty in set(zip((uu[hit] // tile).astype(int).tolist(), (vv[hit] // tile).astype(int).tolist())):
            out[(tx, ty)].add(int(k))
    return out


def padded_boxes(p: Projected, pad_rel=1e-6, pad_abs=2e-4):
    """Per depth rank: the opacity-aware footprint box [mx - ex, mx + ex] x [my - ey, my + ey]
    slightly padded (the device pads its fp64 extents by 1e-7 relative + 1e-4 px)."""
    ex, ey, reach = footprint_extent(p)
    ex = ex * (1 + pad_rel) + pad_abs
    ey = ey * (1 + pad_rel) + pad_abs
    mx, my = p.mean2d[:, 0], p.mean2d[:, 1]
    return mx - ex, mx + ex, my - ey, my + ey, reach
