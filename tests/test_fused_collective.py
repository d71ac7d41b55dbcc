"""a6 + a7 fused over peer memory (parallel.FusedGradReduce, steepgs_gauss_bwd_scatter
+ steepgs_reduce_bcast).  One GPU: R virtual ranks with ordinary local buffers as the peers exercise
every rank's data path (owner ranges, the partial layout, the reduction order, the broadcast), and
the result must equal the NCCL-path reference — each rank's k_gauss_bwd summed into one accumulator
in rank order — bit for bit (the same fp32 additions in the same order).  A one-rank process group
exercises the torch symmetric-memory rendezvous and barriers."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _rank_rasterizers(p, cams_per_rank, cfg, cap):
    from gpu_run import to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    P = torch.zeros(14, cap, device="cuda")
    P[:, :p.shape[1]] = to_dev(p)
    out = []
    for r, cams in enumerate(cams_per_rank):
        rz = Rasterizer(cap, len(cams), cfg.width, cfg.height)
        tg = to_dev(synth.target_images(len(cams), cfg.width, cfg.height, 50 + r))
        rz.project(P, p.shape[1], cams)
        rz.bin_sort()
        rz.render_fwd_l1(tg)
        rz.render_bwd_moments()
        out.append(rz)
    return P, out


@pytest.mark.parametrize("R,mode", [(1, 0), (2, 0), (3, 0), (8, 0), (3, 2), (4, 1)])
def test_fused_scatter_reduce_equals_rank_ordered_sum(orc, R, mode):
    from paper_2505_05587_b200.parallel import FusedGradReduce
    cfg = synth.CONFIGS["C1"]
    n = 3001                                           # owner ranges with a ragged last one
    p = synth.blob_scene(n, 17)
    cams = synth.ring_cameras(2 * R, 64, 64, 9)
    cams_per_rank = [cams[r::R] for r in range(R)]
    cap = n + 77
    prefill = torch.randn(20, cap, device="cuda") if mode else torch.zeros(20, cap, device="cuda")
    # reference: the NCCL path's arithmetic, every rank's k_gauss_bwd summed in rank order
    P, rzs = _rank_rasterizers(p, cams_per_rank, cfg, cap)
    saved = [rz.moments.clone() for rz in rzs]         # the backward's REDs are order-dependent: one set
    ref = prefill.clone()
    # rank 0 applies the mode (0: overwrite, 1: += all, 2: overwrite gradients, += S), ranks 1.. add
    for r, rz in enumerate(rzs):
        rz.gauss_bwd(P, ref, accumulate=mode if r == 0 else 1)
    # fused: the same moments again (gauss_bwd consumed them), scatter per rank, reduce per owner
    for rz, m in zip(rzs, saved):
        rz.moments.copy_(m)
    fr = FusedGradReduce(cap, emulate=R)
    for t in fr.grad_S_all:
        t.copy_(prefill)
    for r, rz in enumerate(rzs):
        fr.scatter(rz, P, n, rank=r)
    for q in range(R):
        fr.reduce(n, accumulate=mode, rank=q)
    torch.cuda.synchronize()
    for r in range(R):
        got = fr.grad_S_all[r][:, :n]
        if mode == 0:   # the same fp32 additions in the same order: bit for bit
            assert torch.equal(got, ref[:, :n]), (r, float((got - ref[:, :n]).abs().max()))
        else:           # prefill + (sum of ranks) vs ((prefill + rank 0) + rank 1) ...: one reassociation
            tol = 1e-6 * (ref[:, :n].abs() + prefill[:, :n].abs()) + 1e-30
            assert bool(((got - ref[:, :n]).abs() <= tol).all()), (r, float((got - ref[:, :n]).abs().max()))
        assert torch.equal(got, fr.grad_S_all[0][:, :n])     # every rank holds the same accumulator
    assert float(fr.grad_S_all[0][14:20, :n].abs().sum()) > 0
    assert float(rzs[0].moments.abs().max()) == 0.0      # the scatter path clears the moments too


def test_fused_symmetric_memory_one_rank(orc):
    """torch symmetric memory rendezvous + device barriers with a one-rank process group (the
    multi-rank exchange is the same code with R peers)."""
    import torch.distributed as dist
    from paper_2505_05587_b200.parallel import FusedGradReduce
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    try:
        fr = FusedGradReduce(3100, device="cuda")
    except (RuntimeError, NotImplementedError) as exc:     # no symmetric-memory support on this box
        pytest.skip(f"symmetric memory unavailable: {exc}")
    cfg = synth.CONFIGS["C1"]
    n = 3001
    p = synth.blob_scene(n, 17)
    cams = synth.ring_cameras(2, 64, 64, 9)
    P, (rz,) = _rank_rasterizers(p, [cams], cfg, 3100)
    saved = rz.moments.clone()
    ref = torch.zeros(20, 3100, device="cuda")
    rz.gauss_bwd(P, ref, accumulate=0)
    rz.moments.copy_(saved)
    fr.scatter(rz, P, n)
    fr.exchange(n, accumulate=0)
    torch.cuda.synchronize()
    assert torch.equal(fr.grad_S[:, :n], ref[:, :n])
    dist.destroy_process_group()
