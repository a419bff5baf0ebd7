"""Parity at the benchmarked configurations (BASELINE.json configs 3 and 4).

C3 = 1M gaussians, SH 3, 64 views at 1920x1080 (the bench workload); C4 =
3M gaussians.  Full-frame CPU oracles are infeasible at this size (SURVEY.md
0.8), so each property is checked against an exact restatement that scales:

* preprocess: every fp64 operand of a discrete decision (kept set, mean2d,
  conic) bit-identical to the C restatement of the reference's numpy
  arithmetic (oracle/exact.py, itself pinned to the reference), and the kept
  order bit-identical to the fp64 stable argsort (render.py:216);
* tile binning: every tile list in global depth order, nothing outside the
  padded opacity-aware footprint, and -- on a crop -- every gaussian with fp64
  alpha >= 1/255 at a pixel of the tile present (oracle/binning.py);
* raster: colour within 1e-4 and depth bit-exact at >= 1000 seeded pixels per
  view plus every pixel of the 8x4 blocks where the raster took an exact
  fp64 re-walk (ambiguous transmittance), against the sparse per-pixel oracle
  (bit-identical to the dense reference);
* selection: masks bit-exact against the oracle's project_cloud at the device
  depth; per-gaussian hit counts exact (and weights within 1e-5) against the
  oracle's contributions on a masked crop.

Flip counts (kept-set mismatches, pixels above 1e-4, depth mismatches) are
printed and, with RCGS_PARITY_REPORT=<path>, written as JSON.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2511_18441_b200 as P  # noqa: E402

IMG_TOL = 1e-4
REPORT = {}


def _report(key, value):
    REPORT[key] = value
    path = os.environ.get("RCGS_PARITY_REPORT")
    if path:
        with open(path, "w") as fh:
            json.dump(REPORT, fh, indent=1, sort_keys=True)
    print(key, value)


@pytest.fixture(scope="module")
def c3():
    import sys
    import torch
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    import bench
    cfg = bench.CONFIGS["c3"]
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    del gt
    torch.cuda.empty_cache()
    return scene, cams, ds, sh0, cloud


def _trace_ambiguous(view, render):
    """Pixels of the 8x4 blocks in which the raster re-walked a pixel's list in
    fp64 (instrumented launch, rcgs_raster_trace)."""
    import torch
    from paper_2511_18441_b200 import _native as N
    tx, ty = view.tiles
    n_items = tx * ty * 8
    tr = torch.zeros((n_items, 8), dtype=torch.int32, device="cuda")
    N.call("rcgs_raster_trace", N.ptr(tr), n_items)
    try:
        render()
        torch.cuda.synchronize()
    finally:
        N.call("rcgs_raster_trace", None, 0)
    tr = tr.cpu().numpy()
    us, vs = [], []
    for i in np.nonzero(tr[:, 6] > 0)[0]:
        tile, blk = int(tr[i, 7]), int(i % 8)
        bx0 = (tile % tx) * 16 + (blk & 1) * 8
        by0 = (tile // tx) * 16 + (blk >> 1) * 4
        for dy in range(4):
            for dx in range(8):
                if bx0 + dx < view.width and by0 + dy < view.height:
                    us.append(bx0 + dx)
                    vs.append(by0 + dy)
    return np.array(us, dtype=np.int64), np.array(vs, dtype=np.int64), int((tr[:, 6] > 0).sum())


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("vi", [0, 16, 33, 50])
def test_c3_view_parity(c3, vi):
    import torch
    from oracle import binning as OB, exact as OX, raster as OR, selection as OS
    from paper_2511_18441_b200 import device as D
    scene, cams, ds, sh0, cloud = c3
    intr, pose = cams[vi]
    view = D.View(ds, intr, pose, P.DEFAULT_CONFIG)
    p = OR.project(scene, intr, pose)

    # ---- preprocess: kept order and the exact operands of every decision
    idx, z = view.kept()
    idx = idx.cpu().numpy()
    kept_mismatch = int(len(idx) != p.count or np.count_nonzero(idx != p.index[:len(idx)]))
    _report(f"c3_v{vi}_kept", {"device": int(len(idx)), "oracle": int(p.count), "order_mismatches": kept_mismatch})
    np.testing.assert_array_equal(idx, p.index)
    np.testing.assert_array_equal(z.cpu().numpy(), p.depth)
    ex = OX.project_exact(scene, intr, pose)
    np.testing.assert_array_equal(np.nonzero(ex["kept"])[0], np.sort(p.index))
    dev = view.exact().cpu().numpy()
    for col, f in enumerate(("mx", "my", "ca", "cb", "cc")):
        np.testing.assert_array_equal(dev[:, col], ex[f][p.index], err_msg=f)
    np.testing.assert_array_equal(dev[:, 2], p.conic_a)

    # ---- tile binning: order, padding, completeness on a crop
    ranges = view.ranges().cpu().numpy().reshape(-1, 2).astype(np.int64)
    pairs = view.pairs().cpu().numpy().astype(np.int64)
    rank_of = np.full(len(scene), -1, np.int64)
    rank_of[p.index] = np.arange(p.count)
    ranks = rank_of[pairs]
    assert (ranks >= 0).all()
    tiles_x = view.tiles[0]
    ne = np.nonzero(ranges[:, 1] > ranges[:, 0])[0]  # empty tiles may hold any [x, x)
    assert (ranges[ne[1:], 0] == ranges[ne[:-1], 1]).all() and ranges[ne[0], 0] == 0
    # pairs after the last list: emitted for a tile of the gaussian's box that its
    # footprint reaches at no 8x4 block (sentinel-keyed at view build, in no list)
    listed = int(ranges[ne[-1], 1])
    assert listed <= len(pairs)
    ranks = ranks[:listed]
    tile_of = np.repeat(ne, ranges[ne, 1] - ranges[ne, 0])
    same = tile_of[1:] == tile_of[:-1]
    assert (ranks[1:][same] > ranks[:-1][same]).all(), "tile list not in global depth order"
    x0, x1, y0, y1, reach = OB.padded_boxes(p)
    tx, ty = tile_of % tiles_x, tile_of // tiles_x
    r = ranks
    inside = (reach[r] & (x1[r] >= tx * 16) & (x0[r] <= tx * 16 + 15) & (y1[r] >= ty * 16) & (y0[r] <= ty * 16 + 15))
    assert inside.all(), f"{np.count_nonzero(~inside)} pairs outside the padded footprint"
    # completeness on a 12x8-tile crop around the selection (the densest region)
    mx = int(np.median(p.mean2d[:, 0]) // 16)
    crop = (max(0, mx - 6), 30, min(tiles_x - 1, mx + 5), 37)
    req = OB.required_tile_sets(p, intr.width, intr.height, crop)
    missing = 0
    for (cx, cy), need in req.items():
        t = cy * tiles_x + cx
        have = set(ranks[ranges[t, 0]:ranges[t, 1]].tolist())
        missing += len(need - have)
    _report(f"c3_v{vi}_binning", {"pairs": int(len(pairs)), "listed": listed, "crop_tiles": len(req),
                                  "crop_required_entries": int(sum(len(v) for v in req.values())),
                                  "missing": missing})
    assert missing == 0

    # ---- raster: colour + depth at seeded pixels and at every re-walked block
    view.color(sh0)
    img = {}

    def render():
        img["v"] = view.render(None, 0)

    au, av, n_blocks = _trace_ambiguous(view, render)
    du, dv, n_dblocks = _trace_ambiguous(view, lambda: view.depth(0.5))  # tau-crossing re-walks
    au, av = np.concatenate([au, du]), np.concatenate([av, dv])
    n_blocks += n_dblocks
    img = img["v"].cpu().numpy()
    np.testing.assert_array_equal(view.render(None, 0).cpu().numpy(), img)  # uninstrumented == instrumented
    dep = view.depth(0.5).cpu().numpy()
    rng = np.random.default_rng(100 + vi)
    us = np.concatenate([rng.integers(0, intr.width, 1000), au])
    vs = np.concatenate([rng.integers(0, intr.height, 1000), av])
    col, _, odep, _ = OR.sparse_pixels(p, us, vs)
    diff = np.abs(img[vs, us] - col).max(axis=1)
    dmis = int(np.count_nonzero(~((dep[vs, us] == odep) | (np.isinf(dep[vs, us]) & np.isinf(odep)))))
    _report(f"c3_v{vi}_raster", {"pixels": int(len(us)), "rewalk_blocks": n_blocks, "rewalk_pixels": int(len(au)),
                                 "over_1e-4": int(np.count_nonzero(diff > IMG_TOL)), "max_abs": float(diff.max()),
                                 "depth_mismatches": dmis})
    assert diff.max() <= IMG_TOL
    assert dmis == 0

    # ---- selection: mask at the device depth, hits on a masked crop
    from paper_2511_18441_b200.selection import project_cloud_device
    pts = D.to_device(cloud.points, torch.float64)
    dd = view.depth(0.5)
    mask = project_cloud_device(pts, intr, pose, dd)
    mask_np = mask.cpu().numpy().astype(bool)
    np.testing.assert_array_equal(mask_np, OS.project_cloud(cloud.points, intr, pose, dd.cpu().numpy()))
    mv, mu = np.nonzero(mask_np)
    if len(mu):
        c_u, c_v = int(np.median(mu)), int(np.median(mv))
        crop = np.zeros_like(mask_np)
        crop[max(0, c_v - 12):c_v + 12, max(0, c_u - 16):c_u + 16] = True
        sel = mask_np & crop
        su, sv = np.nonzero(sel.T)  # (u, v) pairs
        hits = torch.zeros(len(scene), dtype=torch.int32, device="cuda")
        wsum = torch.zeros(len(scene), dtype=torch.int64, device="cuda")
        view.mask_hits(torch.from_numpy(sel.astype(np.uint8)).cuda(), hits, wsum)
        _, _, _, contribs = OR.sparse_pixels(p, su, sv)
        oh = np.zeros(len(scene), np.int64)
        ow = np.zeros(len(scene))
        for ks, ws in contribs:
            g = p.index[np.asarray(ks, dtype=np.int64)]
            np.add.at(oh, g, 1)
            np.add.at(ow, g, np.asarray(ws, dtype=np.float64))
        np.testing.assert_array_equal(hits.cpu().numpy(), oh)
        dw = wsum.cpu().numpy() / 4294967296.0
        assert np.abs(dw - ow).max() <= 1e-5 * max(1.0, ow.max())
        _report(f"c3_v{vi}_selection", {"masked_px": int(mask_np.sum()), "crop_px": int(sel.sum()),
                                        "gaussians_hit_in_crop": int(np.count_nonzero(oh))})
    view.close()


@pytest.mark.timeout(1800)
def test_c4_view_kept_order():
    """C4 (3M gaussians, 1080p): one view's kept order bit-exact vs the fp64 stable argsort."""
    import torch
    from oracle import raster as OR
    from paper_2511_18441_b200 import device as D
    from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
    scene, _ = scaled_scene(3_000_000, 3, seed=0)
    intr, pose = ring_cameras(1920, 1080, 128)[7]
    ds = D.device_scene(scene)
    view = D.View(ds, intr, pose, P.DEFAULT_CONFIG)
    idx, z = view.kept()
    p = OR.project(scene, intr, pose)
    _report("c4_v7_kept", {"device": int(idx.shape[0]), "oracle": int(p.count),
                           "order_mismatches": int(idx.shape[0] != p.count or
                                                   np.count_nonzero(idx.cpu().numpy() != p.index))})
    np.testing.assert_array_equal(idx.cpu().numpy(), p.index)
    np.testing.assert_array_equal(z.cpu().numpy(), p.depth)
    view.close()
    del ds
    torch.cuda.empty_cache()
