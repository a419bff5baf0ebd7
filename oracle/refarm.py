"""CPU reference timing for bench.py -- BENCH INFRASTRUCTURE ONLY.

Used only by bench.py's ``cpu_baseline`` leg and its ``--impl reference`` arm,
as the measured CPU baseline; never by the product package.

What is timed is the reference's own CPU algorithm for the hot path:

* kind ``"reference"``: the stock, unmodified reference package (``splattint``,
  pip-installed from /root/reference into ``baseline/_ref``, which travels to
  the GPU box) through its own functions: ``render._project_scene``
  (render.py:172-229), ``render._block_alpha`` / ``_block_weights``
  (render.py:263-292) and, for the full-step calibration, the public
  ``optimize.optimize_iteration`` (optimize.py:99-120);
* kind ``"port"`` (only when ``baseline/_ref`` is absent): the same steps from
  this package's float64 restatement (``oracle.raster``, ``oracle.optim``).

A full optimizer iteration of the reference at 1M gaussians / 1080p is a dense
(pixel x kept-gaussian) composite: hours of CPU time.  It is
therefore measured on a fixed, seeded sample of pixels of view 0 (default 12,000)
spread over a process pool created once (the scene is generated and projected
once per run), and extrapolated to the frame: ``t_proj + t_pixel * W * H * f``.
The factor f (the capture / colour / loss / backward / Adam work on top of the
alpha + weights composite) is not assumed: it is MEASURED at config 1 (10k
gaussians, 256x256, the config the reference runs in full) by timing one full
``optimize_iteration`` of the stock reference on one core against the same
per-pixel estimate on one core (``measured_c1``).  Every pixel of the sample is
composited against all kept gaussians in global depth order -- the
reference's per-pixel work, bit-identical to its dense row blocks (SURVEY.md
8(c)) -- so the per-pixel rate is the reference's own.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STOCK_DIR = os.path.join(ROOT, "baseline", "_ref")

_STATE = {}  # per process: the projection shared with forked workers


def stock():
    """The stock reference package from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(STOCK_DIR, "splattint")):
        return None
    if STOCK_DIR not in sys.path:
        sys.path.insert(0, STOCK_DIR)
    try:
        import importlib
        from types import SimpleNamespace
        # the package re-exports functions named like its modules (splattint.render
        # is the function): take the modules themselves
        mods = {m: importlib.import_module(f"splattint.{m}") for m in ("optimize", "recolor", "render", "scene")}
        return SimpleNamespace(**mods)
    except Exception:
        return None


def _to_stock(sp, scene, intr, pose):
    S = sp.scene
    sc = S.Scene(positions=scene.positions, rotations=scene.rotations, scales=scene.scales,
                 opacities=scene.opacities, sh=scene.sh, sh_degree=scene.sh_degree)
    it = S.CameraIntrinsics(fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy, width=intr.width,
                            height=intr.height)
    po = S.CameraPose(rotation=np.asarray(pose.rotation), translation=np.asarray(pose.translation))
    return sc, it, po


def _project(kind, scene, intr, pose):
    if kind == "reference":
        sp = stock()
        sc, it, po = _to_stock(sp, scene, intr, pose)
        return sp.render._project_scene(sc, it, po)
    from . import raster as OR
    return OR.project(scene, intr, pose)


def _pixels(args):
    """Composite a list of pixels (each against every kept gaussian); returns
    (count, seconds).  Runs in a pool worker (projection inherited by fork)."""
    us, vs = args
    kind, proj = _STATE["kind"], _STATE["proj"]
    if kind == "reference":
        R = stock().render
        cfg = R.DEFAULT_CONFIG
        alpha_fn = lambda x, y: R._block_alpha(proj, x, y, cfg)  # noqa: E731
        weights_fn = lambda a: R._block_weights(a, cfg)  # noqa: E731
    else:
        from . import raster as OR
        alpha_fn = lambda x, y: OR.alpha_block(proj, x, y)  # noqa: E731
        weights_fn = OR.weights_block
    t0 = time.perf_counter()
    for u, v in zip(us, vs):
        weights_fn(alpha_fn(np.array([float(u)]), np.array([float(v)])))
    return len(us), time.perf_counter() - t0


class PixelSampler:
    """Scene + projection of view 0 built once; a fork pool created once; a
    fixed seeded pixel sample timed in chunks."""

    def __init__(self, cfg, workers=None, n_pixels=12000, seed=0, kind=None):
        from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
        self.kind = kind or ("reference" if stock() is not None else "port")
        self.cfg = cfg
        self.scene, _ = scaled_scene(cfg["n"], cfg["deg"], seed=0)
        self.intr, self.pose = ring_cameras(cfg["width"], cfg["height"], cfg["views"])[0]
        t0 = time.perf_counter()
        proj = _project(self.kind, self.scene, self.intr, self.pose)
        self.t_proj = time.perf_counter() - t0
        self.kept = int(proj.count)
        _STATE.update(kind=self.kind, proj=proj)
        self.workers = int(workers or max(1, min(os.cpu_count() or 1, 16)))
        rng = np.random.default_rng(seed)
        self.us = rng.integers(0, cfg["width"], n_pixels)
        self.vs = rng.integers(0, cfg["height"], n_pixels)
        self.pool = mp.get_context("fork").Pool(self.workers) if self.workers > 1 else None

    def time(self, lo, hi):
        """Wall seconds to composite sample pixels [lo, hi) on the pool."""
        us, vs = self.us[lo:hi], self.vs[lo:hi]
        chunks = [(us[i::self.workers], vs[i::self.workers]) for i in range(self.workers)]
        t0 = time.perf_counter()
        if self.pool is not None:
            done = sum(r[0] for r in self.pool.map(_pixels, chunks))
        else:
            done = _pixels(chunks[0])[0]
        return done, time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None


def measured_c1(seconds_budget=120.0):
    """One full reference optimizer iteration at config 1 (10k gaussians, SH 0,
    256x256), timed end to end on one core, against the per-pixel estimate of the
    same iteration on one core.  Returns {full_s, proj_s, pixel_s, factor, ...}:
    factor = (full - proj) / (pixel_s * W * H) is the measured multiplier that
    turns the alpha + weights composite into a whole iteration."""
    from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
    cfg = dict(n=10_000, deg=0, views=4, width=256, height=256)
    kind = "reference" if stock() is not None else "port"
    scene, _ = scaled_scene(cfg["n"], cfg["deg"], seed=0)
    intr, pose = ring_cameras(cfg["width"], cfg["height"], cfg["views"])[0]
    rng = np.random.default_rng(1)
    target = rng.random((cfg["height"], cfg["width"], 3))
    t0 = time.perf_counter()
    if kind == "reference":
        sp = stock()
        sc, it, po = _to_stock(sp, scene, intr, pose)
        view = sp.scene.TrainingView(view_id=0, intrinsics=it, pose=po, image=target)
        ds = sp.recolor.EditedDataset(views=(sp.recolor.EditedView(view=view, mask=np.zeros(target.shape[:2], bool),
                                                                   image=target),),
                                      generation=0, tint=np.ones(3))
        sp.optimize.optimize_iteration(sc, ds, np.random.default_rng(0), sp.optimize.AdamState.fresh(len(sc)))
    else:
        from . import optim as OO
        g, _ = OO.view_grad(scene, intr, pose, target)
        OO.adam(scene.sh, g, np.zeros_like(g), np.zeros_like(g), 0)
    full = time.perf_counter() - t0
    # the per-pixel estimate of the same iteration, one core
    s = PixelSampler(cfg, workers=1, n_pixels=1500, seed=0, kind=kind)
    done, wall = s.time(0, 1500)
    s.close()
    px = wall / done
    npix = cfg["width"] * cfg["height"]
    return {"kind": kind, "config": "c1: 10000 gaussians SH 0, 256x256, one optimize_iteration",
            "full_iteration_s": round(full, 3), "proj_s": round(s.t_proj, 4), "pixel_s": px,
            "estimate_composite_s": round(s.t_proj + px * npix, 3),
            "factor": round((full - s.t_proj) / (px * npix), 4), "cores": 1}
