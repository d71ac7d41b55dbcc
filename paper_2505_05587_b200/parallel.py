"""Multi-GPU plumbing for the view-sharded hot path.

The splitting matrix is an expectation over (Pi, x) (Thm 1) and the gradients are sums over
views, so view shards combine by elementwise sum: each rank renders the views {v : v mod R = r} into
its own [20][ld] accumulator (14 gradient planes + 6 S planes, one contiguous buffer), one NCCL
allreduce sums them, and every rank then runs the densify kernels on bit-identical inputs, so the
parameters stay replicated without a broadcast.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin view assignment: rank r takes views r, r + R, r + 2R, ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_views, world))


def allreduce_accumulators(acc: torch.Tensor, group=None, n: int | None = None) -> torch.Tensor:
    """Sum the [20][ld] gradient + splitting-matrix accumulator over ranks, in place.

    With `n` given and ld > n, only the first n columns are reduced: one in-place allreduce per
    plane row acc[k, :n] (each row slice is contiguous), issued asynchronously so NCCL pipelines
    them; otherwise the whole contiguous buffer is reduced in one call."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return acc
    if n is None or n >= acc.shape[1]:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
        return acc
    return allreduce_planes(acc, 0, acc.shape[0], n, group)


_COALESCE = [True]


def allreduce_planes(acc: torch.Tensor, first: int, count: int, n: int, group=None) -> torch.Tensor:
    """Sum planes [first, first + count), columns [0, n) of a planar accumulator over ranks, in place
    (one asynchronous allreduce per contiguous row slice, no staging copies)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return acc
    rows = [acc[k, :n] for k in range(first, first + count)]
    if dist.get_backend(group) == "nccl" and _COALESCE[0]:
        # one NCCL group (ncclGroupStart/End) over the contiguous row slices: a single fused
        # collective launch for the 20 planes instead of 20, still no staging copy.
        # _coalescing_manager is a private torch API: if it is missing or refuses, fall back (once, for
        # the process) to the per-row asynchronous allreduces below, which NCCL pipelines.
        try:
            from torch.distributed.distributed_c10d import _coalescing_manager
            with _coalescing_manager(group=group, device=acc.device, async_ops=True) as cm:
                for r in rows:
                    dist.all_reduce(r, op=dist.ReduceOp.SUM, group=group)
            cm.wait()
            return acc
        except (ImportError, AttributeError, TypeError, NotImplementedError, RuntimeError) as exc:
            import warnings
            warnings.warn(f"coalesced allreduce unavailable ({exc}); per-plane allreduces")
            _COALESCE[0] = False
    works = [dist.all_reduce(r, op=dist.ReduceOp.SUM, group=group, async_op=True) for r in rows]
    for w in works:
        w.wait()
    return acc


def params_checksum(params: torch.Tensor, n: int) -> float:
    """Debug aid: identical on every rank after densify (replicated parameters)."""
    return float(params[:, :n].double().sum().item())
