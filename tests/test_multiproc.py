"""Multi-rank host logic on CPU: world_size 2, gloo backend (no GPU needed).

The view-sharded optimizer (engine.py, parallel.py) lets rank r back-propagate
view picks[r] of the step's batch, all-gathers the per-gaussian channel sums and
expands/averages them identically on every rank.  Here each rank computes its
view's channel sums with the oracle, exchanges them through the package's own
`parallel` helpers over gloo, and applies Adam; the result must equal the
single-process schedule-driven oracle (`oracle.optim.run_batched(batch=2)`) and
be identical on both ranks.  The selection statistics reduction is checked for
exactness the same way.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, golden_camera

STEPS = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _views(d):
    out = []
    for v in (0, 1):
        intr, pose = golden_camera(d, f"v{v}_")
        out.append((intr, pose, d[f"v{v}_edited"]))
    return out


def _worker(rank, world, port, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import optim as OO
        from paper_2511_18441_b200 import parallel
        d = dict(np.load(os.path.join(GOLDEN, "two_blobs_32.npz")))
        scene = OO.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], d["sh"],
                         int(d["sh_degree"]))
        views = _views(d)
        rng = np.random.default_rng(7)
        m = np.zeros_like(scene.sh)
        v = np.zeros_like(scene.sh)
        step = 0
        picks_log = []
        for _ in range(STEPS):
            picks = parallel.draw_views(rng, len(views), world)
            picks_log.append(picks)
            intr, pose, target = views[picks[rank]]
            acc, _ = OO.view_acc(scene, intr, pose, target)
            accs = parallel.exchange_accs(torch.from_numpy(acc), dist.group.WORLD)
            centers = [-(views[p][1].rotation.T @ views[p][1].translation) for p in picks]
            grad = OO.expand_mean(scene, centers, [a.numpy() for a in accs])
            sh, m, v, step, _ = OO.adam(scene.sh, grad, m, v, step)
            scene = scene.with_sh(sh)
        # selection statistics: integer all-reduce is exact
        hits = torch.tensor([rank + 1, 10 * (rank + 1), 0], dtype=torch.int32)
        wsum = torch.tensor([2 ** 40 + rank, 3], dtype=torch.int64)
        parallel.reduce_counts(dist.group.WORLD, hits, wsum)
        # replicate_views: each rank fills its contiguous view block, then every
        # rank holds every row
        mine = parallel.shard_views(5, rank, world)
        stack = torch.full((5, 3), -1.0)
        for i in mine:
            stack[i] = torch.arange(3.0) + 3 * i
        parallel.replicate_views(stack, mine, dist.group.WORLD)
        queue.put((rank, scene.sh, picks_log, hits.tolist(), wsum.tolist(), mine, stack.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_view_sharded_refit_matches_schedule_oracle():
    from oracle import optim as OO
    world = 2
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, queue)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([queue.get(timeout=240) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, sh0, picks0, hits0, wsum0, shard0, rep0), (_, sh1, picks1, hits1, wsum1, shard1, rep1) = results
    # both replicas hold the bit-identical scene and drew the same schedule
    np.testing.assert_array_equal(sh0, sh1)
    assert picks0 == picks1
    # == the single-process schedule-driven oracle with batch 2 (same rng stream)
    d = dict(np.load(os.path.join(GOLDEN, "two_blobs_32.npz")))
    scene = OO.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], d["sh"], int(d["sh_degree"]))
    ref, metrics = OO.run_batched(scene, _views(d), seed=7, steps=STEPS, batch=2)
    assert [m[1] for m in metrics] == [p for ps in picks0 for p in ps]
    np.testing.assert_allclose(sh0, ref.sh, rtol=0, atol=1e-12)
    assert hits0 == hits1 == [3, 30, 0]
    assert wsum0 == wsum1 == [2 * 2 ** 40 + 1, 6]
    assert shard0 == [0, 1] and shard1 == [2, 3, 4]
    np.testing.assert_array_equal(rep0, np.arange(15.0).reshape(5, 3))
    np.testing.assert_array_equal(rep1, rep0)


def test_single_process_helpers():
    from paper_2511_18441_b200 import parallel
    rng_a, rng_b = np.random.default_rng(3), np.random.default_rng(3)
    seq = [parallel.draw_views(rng_a, 9, 1)[0] for _ in range(8)]
    chunked = [x for _ in range(4) for x in parallel.draw_views(rng_b, 9, 2)]
    assert seq == chunked  # sequential == chunked draws
    acc = torch.arange(6.0).reshape(2, 3)
    assert parallel.exchange_accs(acc, None)[0] is acc
    assert parallel.shard_views(4, 0, 1) == [0, 1, 2, 3]
