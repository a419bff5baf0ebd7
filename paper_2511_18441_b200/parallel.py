"""View sharding across ranks (one process per GPU).

The recolor workload shards by camera view.  These helpers are the only
cross-rank logic; they work with any torch.distributed backend (NCCL on the
B200 box, gloo in the CPU tests):

* `draw_views`      the step's view batch from the reference RNG stream: G
                    views per optimizer step, `rng.integers(V, size=G)` (equal
                    to G sequential `rng.integers(V)` draws, optimize.py:106);
                    rank r back-propagates picks[r].
* `exchange_accs`   all-gather of the per-gaussian channel sums (N x 3 fp32
                    per view, 12 B/gaussian instead of the 192 B dense SH
                    gradient).  Every rank then expands sum_v basis_v (x) acc_v
                    / G in the same order -> bit-identical Adam on all ranks,
                    independent of the collective's reduction order.
* `any_rank`        logical OR of the non-finite reject flags.
* `shard_views` / `reduce_counts`  static view blocks for the selection pass
                    and the exact integer all-reduce of its statistics.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world_of(group) -> tuple[int, int]:
    if group is None or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def draw_views(rng: np.random.Generator, n_views: int, world: int) -> list[int]:
    if world == 1:
        return [int(rng.integers(n_views))]
    return [int(x) for x in rng.integers(n_views, size=world)]


def _host_staged(group) -> bool:
    """gloo cannot run every collective on device tensors: stage them through host memory."""
    return dist.get_backend(group) == "gloo"


def exchange_accs(acc: torch.Tensor, group, out: torch.Tensor | None = None) -> list[torch.Tensor]:
    """All-gather the local (N, 3) channel sums; returns one tensor per rank in rank order."""
    world, _ = world_of(group)
    if world == 1:
        return [acc]
    if out is None:
        out = torch.empty((world,) + tuple(acc.shape), dtype=acc.dtype, device=acc.device)
    if acc.is_cuda and not _host_staged(group):
        dist.all_gather_into_tensor(out, acc.contiguous(), group=group)
    elif acc.is_cuda:  # gloo with device tensors (functional multi-rank tests on one GPU)
        host = out.cpu()
        parts = list(host.unbind(0))
        dist.all_gather(parts, acc.contiguous().cpu(), group=group)
        out.copy_(host)
    else:  # gloo: list form
        parts = list(out.unbind(0))
        dist.all_gather(parts, acc.contiguous(), group=group)
    return [out[r] for r in range(world)]


def any_rank(flag: torch.Tensor, group) -> torch.Tensor:
    world, _ = world_of(group)
    if world > 1:
        if flag.is_cuda and _host_staged(group):
            h = flag.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
            flag.copy_(h)
        else:
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    return flag


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Static contiguous view block of this rank (selection pass): rank r gets
    views [r V / G, (r + 1) V / G) (rounded), so the blocks can be all-gathered."""
    lo = (rank * n_views) // world
    hi = ((rank + 1) * n_views) // world
    return list(range(lo, hi))


def replicate_views(stack: torch.Tensor, mine: list[int], group) -> None:
    """Every rank ends with every row of `stack` (V, ...) when each rank computed
    the rows of its `shard_views` block: one all-gather when the blocks are equal
    (V divisible by the world size), else one broadcast per row from its owner."""
    world, rank = world_of(group)
    if world == 1:
        return
    n = stack.shape[0]
    owners = [r for r in range(world) for _ in shard_views(n, r, world)]
    if n % world == 0 and stack.is_cuda and not _host_staged(group):
        blk = n // world
        src = stack[rank * blk:(rank + 1) * blk].clone()
        dist.all_gather_into_tensor(stack, src, group=group)
        return
    for i in range(n):
        if stack.is_cuda and _host_staged(group):
            h = stack[i].cpu()
            dist.broadcast(h, src=owners[i], group=group)
            stack[i].copy_(h)
        else:
            dist.broadcast(stack[i], src=owners[i], group=group)


def reduce_counts(group, *tensors: torch.Tensor) -> None:
    """Exact SUM all-reduce of integer statistics (hit counts, fixed-point weights)."""
    world, _ = world_of(group)
    if world > 1:
        for t in tensors:
            if t.is_cuda and _host_staged(group):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
