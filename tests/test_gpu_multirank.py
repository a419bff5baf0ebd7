"""The view-sharded refit engine itself with two ranks.

Two processes share cuda:0 and talk over gloo (host-staged collectives:
`parallel.exchange_accs` / `any_rank`); each runs `RefitEngine(group=WORLD)`
for a few steps.  Every step draws G = 2 views from the reference RNG stream,
rank r back-propagates picks[r], the ranks all-gather their per-gaussian
channel sums and both apply the same Adam update.  Checked per step:

* both replicas hold bit-identical SH, Adam moments and step counters;
* the update equals the schedule-driven oracle (`oracle.optim`: mean over the
  batch of backward_sh(render_forward(v), loss_grad(v)), then Adam;
  optimize.py:99-120 with batch 2) from the same state, fed the device's own
  fp32 render of each picked view (the sign() in the L1 gradient is not
  defined across precisions), within 1e-6.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, golden_camera

pytestmark = pytest.mark.gpu

STEPS = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, queue):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_18441_b200 as P
        from paper_2511_18441_b200 import device as D
        from paper_2511_18441_b200.engine import RefitEngine
        d = dict(np.load(os.path.join(GOLDEN, "two_blobs_32.npz")))
        scene = P.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], d["sh"],
                        int(d["sh_degree"]))
        cams, targets = [], []
        for v in (0, 1):
            intr, pose = golden_camera(d, f"v{v}_")
            cams.append((P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height),
                         P.CameraPose(pose.rotation, pose.translation)))
            targets.append(D.to_device(d[f"v{v}_edited"]))
        eng = RefitEngine(D.device_scene(scene), D.sh_to_device(scene.sh), cams, targets, P.OptimizerConfig(),
                          seed=7, cache_views=False, group=dist.group.WORLD)
        hist = [(eng.sh.cpu().numpy().copy(), eng.m.cpu().numpy().copy(), eng.v.cpu().numpy().copy(),
                 eng.step_count(), None)]
        for _ in range(STEPS):
            picks = eng.step()
            torch.cuda.synchronize()
            hist.append((eng.sh.cpu().numpy().copy(), eng.m.cpu().numpy().copy(), eng.v.cpu().numpy().copy(),
                         eng.step_count(), list(picks)))
        recs = eng.drain()
        queue.put((rank, hist, [r[5] for r in recs]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_refit_engine_matches_batched_oracle():
    import torch.multiprocessing as mp
    import paper_2511_18441_b200 as P
    from oracle import losses as OL, optim as OO, raster as OR
    world = 2
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, queue)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([queue.get(timeout=500) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, h0, rej0), (_, h1, rej1) = res
    assert rej0 == rej1 == [False] * STEPS
    for a, b in zip(h0, h1):  # replicas bit-identical at every step
        for x, y in zip(a[:3], b[:3]):
            np.testing.assert_array_equal(x, y)
        assert a[3:] == b[3:]
    # draws: G = 2 views per step from default_rng(7) (== 2 sequential draws)
    rng = np.random.default_rng(7)
    assert [h[4] for h in h0[1:]] == [[int(x) for x in rng.integers(2, size=2)] for _ in range(STEPS)]
    d = dict(np.load(os.path.join(GOLDEN, "two_blobs_32.npz")))
    base = OO.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], d["sh"], int(d["sh_degree"]))
    for t in range(STEPS):
        sh, m, v, step, _ = h0[t]
        picks = h0[t + 1][4]
        scene = base.with_sh(sh.astype(np.float64))
        pscene = P.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], sh.astype(np.float64),
                         int(d["sh_degree"]))
        total = np.zeros_like(scene.sh)
        for pk in picks:
            intr, pose = golden_camera(d, f"v{pk}_")
            pi = P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
            pp = P.CameraPose(pose.rotation, pose.translation)
            img = P.render(pscene, pi, pp)  # the device's own fp32 render
            tgt = d[f"v{pk}_edited"].astype(np.float32).astype(np.float64)
            total += OO.backward_sh(OR.render_forward(scene, intr, pose), OL.loss_grad(img, tgt))
        total /= len(picks)
        ref, *_ = OO.adam(scene.sh, total, m.astype(np.float64), v.astype(np.float64), step)
        got = h0[t + 1][0]
        assert np.abs(got - ref).max() <= 1e-6, (t, np.abs(got - ref).max())
        assert h0[t + 1][3] == step + 1
