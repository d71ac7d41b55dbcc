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


class FusedGradReduce:
    """a6 + a7 fused over peer memory (the B200-native variant of the NCCL allreduce):
    k_gauss_bwd stores each Gaussian's 20-plane result straight into the partial buffer of the rank
    that owns its column range (P2P stores over NVLink while the kernel computes: the reduce-scatter
    fused into the compute), then each owner sums the R partials of its range and stores the result
    into every rank's grad_S (the all-gather fused into the reduction).  Two device-side barriers of
    torch symmetric memory order the exchange.  grad_S and the partial buffers are symmetric-memory
    tensors (`self.grad_S` replaces the caller's accumulator).

    `emulate = R` builds R virtual ranks on one device instead (tests: the data path of every rank is
    exercised, the peers are ordinary local buffers, the ranks run one after another)."""

    def __init__(self, capacity: int, group=None, device=None, emulate: int | None = None):
        from . import _lib
        self._lib = _lib
        self.cap = int(capacity)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if emulate is not None:
            self.R, self.rank = int(emulate), 0
            self.chunk_cap = _lib.scatter_chunk(self.cap, self.R)
            self.partials = [torch.zeros(self.R * 20 * self.chunk_cap, dtype=torch.float32, device=self.device)
                             for _ in range(self.R)]
            self.grad_S_all = [torch.zeros(20, self.cap, dtype=torch.float32, device=self.device)
                               for _ in range(self.R)]
            self.grad_S = self.grad_S_all[0]
            return
        import torch.distributed._symmetric_memory as symm_mem
        self.group = group if group is not None else dist.group.WORLD
        self.R, self.rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        if self.R > 8:
            raise ValueError("FusedGradReduce: at most 8 ranks (one NVSwitch domain)")
        self.chunk_cap = _lib.scatter_chunk(self.cap, self.R)
        self.partial = symm_mem.empty(self.R * 20 * self.chunk_cap, dtype=torch.float32, device=self.device)
        self.grad_S = symm_mem.empty(20, self.cap, dtype=torch.float32, device=self.device)
        self.grad_S.zero_()
        self.h_part = symm_mem.rendezvous(self.partial, self.group)
        self.h_gs = symm_mem.rendezvous(self.grad_S, self.group)
        self.peer_partials = list(self.h_part.buffer_ptrs)
        self.peer_grad_S = list(self.h_gs.buffer_ptrs)

    def scatter(self, rz, params, n: int, rank: int | None = None):
        """This rank's k_gauss_bwd with its output scattered to the owners (rz: its Rasterizer after
        render_bwd_moments)."""
        r = self.rank if rank is None else rank
        chunk = self._lib.scatter_chunk(n, self.R)
        peers = [t.data_ptr() for t in self.partials] if hasattr(self, "partials") else self.peer_partials
        self._lib.gauss_bwd_scatter(params, params.shape[1], n, rz.cams_arr, rz.V, rz.rp, rz.moments, peers, self.R, r,
                                    chunk)

    def reduce(self, n: int, accumulate: int = 0, rank: int | None = None):
        """The owner's reduce + broadcast (after every rank's scatter has landed)."""
        r = self.rank if rank is None else rank
        chunk = self._lib.scatter_chunk(n, self.R)
        if hasattr(self, "partials"):
            self._lib.reduce_bcast(self.partials[r], self.R, r, n, chunk, [t.data_ptr() for t in self.grad_S_all],
                                   self.cap, accumulate)
        else:
            self._lib.reduce_bcast(self.partial, self.R, r, n, chunk, self.peer_grad_S, self.cap, accumulate)

    def barrier(self):
        if not hasattr(self, "partials"):
            self.h_part.barrier(channel=0)

    def exchange(self, n: int, accumulate: int = 0):
        """barrier -> reduce + broadcast -> barrier (after this rank's scatter)."""
        self.barrier()
        self.reduce(n, accumulate)
        self.barrier()
