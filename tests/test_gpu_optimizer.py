"""GPU tests of the optimizer's control semantics against the reference's
BackgroundOptimizer contract (optimize.py:131-259): non-finite rejection
(optimize.py:72-74), dataset swaps from the next iteration on (173-175,
211-214), snapshots that are exactly the post-step-k scene (221-238), and
thread safety of save_state / readers while the worker runs.
"""

from __future__ import annotations

import threading
import time

import numpy as np
import pytest

from conftest import golden_camera

pytestmark = pytest.mark.gpu

import paper_2511_18441_b200 as P  # noqa: E402


def _scene(d):
    return P.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], d["sh"], int(d["sh_degree"]))


def _views(d, scene, ids=(0, 1)):
    out = []
    for v in ids:
        intr, pose = golden_camera(d, f"v{v}_")
        intr = P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
        pose = P.CameraPose(pose.rotation, pose.translation)
        out.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    return out


def _dataset(d, scene, tint=(1.0, 0.2, 0.2), generation=0, ids=(0, 1)):
    return P.build_edited_dataset(_views(d, scene, ids), P.SelectionCloud(d["cloud"]), tint, scene,
                                  generation=generation)


def _with_nan(ds, view_index):
    views = list(ds.views)
    ev = views[view_index]
    img = ev.image.copy()
    img[img.shape[0] // 2, img.shape[1] // 2, 1] = np.nan
    views[view_index] = P.EditedView(view=ev.view, mask=ev.mask, image=img)
    return P.EditedDataset(views=tuple(views), generation=ds.generation, tint=ds.tint)


# ---------------------------------------------------------------- non-finite rejection
@pytest.mark.parametrize("cache_views", [True, False])
def test_rejected_step_rearms_and_next_step_is_accepted(two_blobs, cache_views):
    """A NaN target makes the step's gradient non-finite: the step is rejected
    (SH, m, v and the step counter unchanged) and the flag is re-armed, so the
    next step on a clean view is accepted and equals a lone step on that view."""
    import torch
    from paper_2511_18441_b200 import device as D
    from paper_2511_18441_b200.engine import RefitEngine
    scene = _scene(two_blobs)
    ds = _with_nan(_dataset(two_blobs, scene), 1)
    cams = [(ev.view.intrinsics, ev.view.pose) for ev in ds.views]
    tg = [D.to_device(ev.image) for ev in ds.views]
    dsc = D.device_scene(scene)
    sh0 = D.sh_to_device(scene.sh)
    eng = RefitEngine(dsc, sh0.clone(), cams, tg, P.OptimizerConfig(), cache_views=cache_views)
    eng.step(picks=[1])
    eng.step(picks=[1])
    eng.step(picks=[0])
    eng.step(picks=[0])
    recs = eng.drain()
    assert [r[5] for r in recs] == [True, True, False, False]
    assert eng.step_count() == 2
    ref = RefitEngine(dsc, sh0.clone(), cams, tg, P.OptimizerConfig(), cache_views=cache_views)
    ref.step(picks=[0])
    ref.step(picks=[0])
    ref.drain()
    assert torch.equal(eng.sh, ref.sh) and torch.equal(eng.m, ref.m) and torch.equal(eng.v, ref.v)
    assert not torch.equal(eng.sh, sh0)


def test_rejected_steps_in_the_fused_pipeline(two_blobs):
    """The prefetching pipeline (Adam colours the next view) rejects and recovers
    exactly like the synchronous one on the same RNG-drawn view sequence."""
    import torch
    from paper_2511_18441_b200 import device as D
    from paper_2511_18441_b200.engine import RefitEngine
    scene = _scene(two_blobs)
    ds = _with_nan(_dataset(two_blobs, scene), 1)
    cams = [(ev.view.intrinsics, ev.view.pose) for ev in ds.views]
    tg = [D.to_device(ev.image) for ev in ds.views]
    dsc = D.device_scene(scene)
    sh0 = D.sh_to_device(scene.sh)
    out = []
    for prefetch in (0, 2):
        eng = RefitEngine(dsc, sh0.clone(), cams, tg, P.OptimizerConfig(), seed=11, cache_views=False,
                          prefetch=prefetch)
        for _ in range(12):
            eng.step()
        recs = [repr((list(map(int, p)),) + tuple(r)) for p, *r in eng.drain()]  # repr: nan == nan
        eng.close()
        out.append((eng.sh.clone(), eng.step_count(), recs))
    assert torch.equal(out[0][0], out[1][0]) and out[0][1] == out[1][1] and out[0][2] == out[1][2]
    rejected = [r.endswith("True)") for r in out[0][2]]
    assert any(rejected) and not all(rejected)
    assert out[0][1] == rejected.count(False)


def test_optimize_iteration_rejects_non_finite(two_blobs):
    """optimize_iteration returns the inputs unchanged on a rejected step (optimize.py:72-74, 113)."""
    scene = _scene(two_blobs)
    ds = _with_nan(_dataset(two_blobs, scene, ids=(1,)), 0)
    state = P.AdamState.fresh(len(scene))
    new_scene, new_state, metrics = P.optimize_iteration(scene, ds, np.random.default_rng(0), state)
    np.testing.assert_array_equal(new_scene.sh, scene.sh)
    assert new_state.step == 0 and not new_state.m.any() and not new_state.v.any()
    assert metrics.iteration == 1


# ---------------------------------------------------------------- dataset swaps
def _run_with_swap(scene, ds_a, ds_b, n_before, n_after, **kw):
    lines = []
    opt = P.BackgroundOptimizer(scene, ds_a, seed=4, metrics_sink=lambda m: lines.append(m.line()), **kw)
    for _ in range(n_before):
        opt._step()
    opt.swap_dataset(ds_b)
    for _ in range(n_after):
        opt._step()
    opt._flush()
    sh = opt.engine.sh.detach().cpu().numpy().copy()
    gen = opt.dataset.generation
    opt.stop()
    return sh, lines, gen


@pytest.mark.parametrize("kw", [dict(stream_targets=True, prefetch=2, cache_views=False),
                                dict(prefetch=2, cache_views=False)])
def test_swap_dataset_pipelined_matches_synchronous(two_blobs, kw):
    """A new edit (same cameras, new targets) swapped in mid-run is fitted from
    the next iteration on: the pipelined optimizer (views drawn and targets
    uploaded two steps ahead) gives the same SH bits and metric lines as the
    synchronous one, and reports the new generation."""
    scene = _scene(two_blobs)
    ds_a = _dataset(two_blobs, scene)
    ds_b = _dataset(two_blobs, scene, tint=(0.2, 0.3, 1.0), generation=1)
    ref = _run_with_swap(scene, ds_a, ds_b, 5, 5)
    got = _run_with_swap(scene, ds_a, ds_b, 5, 5, **kw)
    np.testing.assert_array_equal(got[0], ref[0])
    assert got[1] == ref[1]
    assert got[2] == 1 and [l.split(",")[2] for l in got[1]] == ["0"] * 5 + ["1"] * 5


@pytest.mark.parametrize("kw", [dict(), dict(prefetch=2, cache_views=False),
                                dict(stream_targets=True, prefetch=2, cache_views=False)])
def test_swap_dataset_with_different_cameras(two_blobs, kw):
    """A dataset with other cameras (here: one view instead of two) swaps in with
    value-compared poses (no numpy truth-value error) in every pipeline, and the
    next draws sample the new dataset exactly like the synchronous optimizer."""
    scene = _scene(two_blobs)
    ds_a = _dataset(two_blobs, scene)
    ds_b = _dataset(two_blobs, scene, tint=(0.2, 0.3, 1.0), generation=2, ids=(1,))
    ref = _run_with_swap(scene, ds_a, ds_b, 4, 4)
    got = _run_with_swap(scene, ds_a, ds_b, 4, 4, **kw)
    np.testing.assert_array_equal(got[0], ref[0])
    assert got[1] == ref[1]
    assert all(l.split(",")[1] == "1" for l in got[1][4:])


# ---------------------------------------------------------------- snapshots
@pytest.mark.parametrize("kw", [dict(), dict(stream_targets=True, prefetch=2, cache_views=False)])
def test_snapshot_is_exactly_the_post_step_scene(two_blobs, kw):
    """start() mode: snapshot() is the scene after exactly the last iteration whose
    count is a multiple of snapshot_every (published in stream order by that
    step's Adam), equal to run_iterations(k).current_scene() bit for bit."""
    scene = _scene(two_blobs)
    ds = _dataset(two_blobs, scene)
    opt = P.BackgroundOptimizer(scene, ds, seed=9, **kw)
    opt.start()
    t0 = time.time()
    while opt.status().iteration < 30 and time.time() - t0 < 60:
        time.sleep(0.01)
    opt.pause()
    snap = opt.snapshot()
    k = int(opt.engine.snapshot_step.item())
    cur = opt.current_scene()
    n = opt.engine.step_count()
    opt.stop()
    assert k >= 10 and k % 10 == 0 and n >= k
    ref = P.BackgroundOptimizer(scene, ds, seed=9, **kw)
    np.testing.assert_array_equal(snap.sh, ref.run_iterations(k).sh)
    np.testing.assert_array_equal(cur.sh, ref.run_iterations(n - k).sh)
    ref.stop()


def test_save_state_after_pause_does_not_deadlock(two_blobs, tmp_path):
    """pause() then save_state() while metric read-backs are still in flight
    completes (the drain no longer re-enters a held lock) and resumes exactly."""
    scene = _scene(two_blobs)
    ds = _dataset(two_blobs, scene)
    opt = P.BackgroundOptimizer(scene, ds, seed=2, prefetch=2, cache_views=False)
    opt.start()
    t0 = time.time()
    while opt.engine.step_count() < 25 and time.time() - t0 < 60:
        time.sleep(0.005)
    opt.pause()
    done = threading.Event()
    err = []

    def save():
        try:
            opt.save_state(tmp_path / "s.npz")
        except Exception as e:  # surfaced below
            err.append(e)
        done.set()

    threading.Thread(target=save, daemon=True).start()
    assert done.wait(60), "save_state deadlocked"
    assert not err, err
    n = opt.engine.step_count()
    cur = opt.current_scene().sh
    opt.stop()
    b = P.BackgroundOptimizer(scene, ds, seed=2, prefetch=2, cache_views=False)
    b.load_state(tmp_path / "s.npz")
    assert b.engine.step_count() == n
    np.testing.assert_array_equal(b.current_scene().sh, cur)
    b.stop()
