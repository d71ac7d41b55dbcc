"""Seeded fuzz parity: many small random scenes, cameras (pinhole and affine, off-centre, tilted) and
raster parameters (thresholds, dilation, background), each through the whole GPU path against the
oracle — decisions and binning bit-exact, images, gradients and S within the §3.4 tolerances, and
the densify decisions.  Sizes are small so every case runs the oracle in well under a second."""
import os

import numpy as np
import pytest

import synth
from helpers import affine_cam, params_from

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    W, H = int(rng.integers(8, 90)), int(rng.integers(8, 70))
    means = np.concatenate([rng.uniform(-1.5, 1.5, size=(n, 2)), rng.uniform(-1.0, 1.0, size=(n, 1))], 1)
    scales = np.exp(np.log(rng.uniform(0.03, 0.4)) + 0.6 * rng.normal(size=(n, 3)))
    quats = rng.normal(size=(n, 4))
    opac = rng.uniform(0.02, 0.98, size=n)
    rgb = rng.uniform(0, 1, size=(n, 3))
    p = params_from(means, scales, quats, opac, rgb)
    V = int(rng.integers(1, 4))
    if rng.uniform() < 0.5:
        cams = synth.ring_cameras(V, W, H, seed + 7, radius=float(rng.uniform(2.5, 5.0)))
    else:
        cams = []
        for v in range(V):
            R, t = synth.look_at(rng.normal(size=3) * 3 + np.array([0, 0, 0.5]))
            cams.append(affine_cam(W, H, fx=float(rng.uniform(5, 25)), cx=float(rng.uniform(0, W)),
                                   cy=float(rng.uniform(0, H)), R=R.astype(np.float32), t=tuple(t)))
    rp = dict(alpha_min=float(rng.choice([1.0 / 255.0, 0.01, 0.0])), alpha_max=float(rng.choice([0.99, 0.999])),
              t_min=float(rng.choice([1e-4, 1e-3])), dilation=float(rng.choice([0.3, 0.1, 0.0])),
              bg=tuple(float(x) for x in rng.uniform(0, 1, size=3) * (rng.uniform() < 0.5)), tile=16)
    if rp["alpha_min"] == 0.0:
        rp.update(alpha_max=1.0, t_min=0.0)
    return p, cams, rp


@pytest.mark.parametrize("seed", list(range(int(os.environ.get("STEEPGS_FUZZ_SEEDS", "64")))))
def test_fuzz_full_path(orc, seed):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from gpu_run import decisions, run_backward, run_forward
    from test_gpu_parity import _grad_close, _grad_report, expected_binning_fast
    p, cams, rp = _case(seed)
    n, V = p.shape[1], len(cams)
    W, H = cams[0]["width"], cams[0]["height"]
    rz, pt = run_forward(p, cams, rp)
    g = decisions(rz, n)
    decs = [orc.decide(p, c, rp) for c in cams]
    for v in range(V):
        vis = decs[v]["visible"].astype(bool)
        assert np.array_equal(g["tiles_touched"][v] > 0, vis)
        assert np.array_equal(g["key"][v][vis], decs[v]["key"][vis])
    ids, counts = expected_binning_fast(decs, W, H)
    b = rz.binning_arrays()
    assert b["overflow"] == 0 and b["n_instances"] == ids.size
    assert np.array_equal(b["ids"].numpy().astype(np.int64), ids)
    assert np.array_equal((b["ranges"][:, 1] - b["ranges"][:, 0]).numpy(), counts)
    img = rz.image.cpu().numpy()
    dl = synth.dl_dimage(V, W, H, 1000 + seed)
    o = np.zeros((20, n)); a = np.zeros((20, n)); aS = np.zeros((6, n))
    for v, cam in enumerate(cams):
        r = orc.render(p, cam, rp, decision=decs[v])
        ok = (np.abs(img[v] - r["image"]) <= 1e-4 * np.abs(r["image"]) + 1e-6) | (r["amb_px"][None] != 0)
        assert ok.all(), (seed, v)
        assert int(r["amb_px"].sum()) <= 0.01 * r["amb_px"].size, (seed, v)   # excluded pixels bounded
        dl[v][:, r["amb_px"] != 0] = 0.0
    for v, cam in enumerate(cams):
        r = orc.render(p, cam, rp, dl_dimage=dl[v], decision=decs[v])
        o += r["grad"]; a += r["absg"]; aS += r["absS"]
    gg = run_backward(rz, pt, dl)
    ok = _grad_close(gg, o, a, np.zeros(n, np.uint8), absS=aS)
    assert ok.all(), _grad_report(gg, o, a, ok)


@pytest.mark.parametrize("seed", list(range(16)))
def test_fuzz_sh(orc, seed):
    """Random SH degree / coefficients (colour kept unclamped by a DC offset) through project_sh ->
    render -> sh_bwd -> gauss_bwd(| 4)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from gpu_run import raster_of, to_dev
    from test_gpu_parity import _grad_close, _grad_report
    from paper_2505_05587_b200.pipeline import Rasterizer
    p, cams, rp = _case(500 + seed)
    rng = np.random.default_rng(900 + seed)
    deg = int(rng.integers(0, 4))
    n, V = p.shape[1], len(cams)
    W, H = cams[0]["width"], cams[0]["height"]
    p[11:14] = rng.uniform(0.4, 1.5, size=(3, n)).astype(np.float32)
    rest = (rng.normal(size=(3 * ((deg + 1) ** 2 - 1), n)) * 0.1).astype(np.float32)
    rz = Rasterizer(n, V, W, H, raster_of(rp))
    dp = to_dev(p)
    drest = to_dev(rest) if rest.size else torch.zeros(0, n, device="cuda")
    rz.project(dp, n, cams, drest, deg)
    rz.bin_sort(); rz.render_fwd()
    dl = synth.dl_dimage(V, W, H, 2000 + seed)
    img = rz.image.cpu().numpy()
    o = np.zeros((20, n)); a = np.zeros((20, n)); osh = np.zeros((rest.shape[0], n))
    rr = []
    for v, cam in enumerate(cams):
        r = orc.render(p, cam, rp, sh_rest=rest, sh_degree=deg)
        ok = (np.abs(img[v] - r["image"]) <= 1e-4 * np.abs(r["image"]) + 1e-6) | (r["amb_px"][None] != 0)
        assert ok.all(), (seed, v)
        assert int(r["amb_px"].sum()) <= 0.01 * r["amb_px"].size, (seed, v)   # excluded pixels bounded
        dl[v][:, r["amb_px"] != 0] = 0.0
    for v, cam in enumerate(cams):
        r = orc.render(p, cam, rp, dl_dimage=dl[v], sh_rest=rest, sh_degree=deg)
        o += r["grad"]; a += r["absg"]
        if rest.shape[0]:
            osh += r["grad_sh"]
    grad = torch.zeros(20, n, device="cuda")
    gsh = torch.zeros(max(rest.shape[0], 0), n, device="cuda")
    rz.render_bwd_moments(dL=to_dev(dl))
    rz.sh_bwd(dp, grad, drest, deg, gsh, accumulate=0)
    rz.gauss_bwd(dp, grad, accumulate=4)
    g = grad.cpu().numpy().astype(np.float64)
    ok = _grad_close(g, o, a, np.zeros(n, np.uint8))
    assert ok.all(), _grad_report(g, o, a, ok)
    if rest.shape[0]:
        gs = gsh.cpu().numpy().astype(np.float64)
        assert (np.abs(gs - osh) <= 2e-3 * np.abs(osh) + 1e-5 * np.abs(osh).max(axis=1, keepdims=True) + 1e-30).all()


@pytest.mark.parametrize("seed", list(range(12)))
def test_fuzz_densify(orc, seed):
    """Random sizes (1 .. 20k, ragged against every tile size), denominators and capacities (fused
    and two-kernel paths, just-enough and too-small) through steepgs_densify against the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from test_gpu_parity import _densify_inputs, _gpu_densify
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.choice([1, 2, 255, 257, 2047, 2049, int(rng.integers(1, 20000))]))
    denom = float(rng.choice([1.0, 3.0, 7.5]))
    p, S = _densify_inputs(orc, n, 40 + seed, denom=denom)
    lam = np.array([orc.eig_sym3(S[:, i].astype(np.float64) / np.float32(denom))[0][0] for i in range(n)])
    ns = int((lam < -1e-6).sum())
    cap = int(rng.choice([2 * n, n + ns, max(n, n + ns - 1)]))
    accd = np.zeros((20, cap)); accd[14:20, :n] = S
    pd = np.zeros((14, cap)); pd[:, :n] = p
    r = orc.densify(pd, accd, n, cap, denom=denom)
    rz, P, A = _gpu_densify(p, S, n, cap, denom=denom)
    if r["n_split"] < 0:
        assert int(rz.dens_status.item()) == 3
        return
    assert int(rz.dens_status.item()) == 0 and int(rz.n_split.item()) == r["n_split"] == ns
    assert np.array_equal(rz.split_mask[:n].cpu().numpy(), r["mask"])
    assert np.array_equal(rz.dest_index[:n].cpu().numpy(), r["dest"])


@pytest.mark.parametrize("n", [1, 255, 2048, 2049, 100_003])
def test_prune_kernels(n):
    """steepgs_prune_decide / steepgs_compact_planes against numpy: keep iff logit >= logit_min,
    stable order, every plane moved."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_05587_b200 import _lib
    rng = np.random.default_rng(n)
    P = rng.normal(size=(14, n + 7)).astype(np.float32)
    P[10] = rng.uniform(-8, 2, size=n + 7).astype(np.float32)
    thr = np.float32(-5.29)
    P[10, : n // 3] = thr                                   # exact ties are kept (>=)
    dP = torch.from_numpy(P).cuda()
    new_index = torch.empty(n, dtype=torch.int32, device="cuda")
    n_keep = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(_lib.prune_workspace_size(n), dtype=torch.uint8, device="cuda")
    _lib.prune_decide(dP, n, float(thr), new_index, n_keep, ws)
    keep = np.flatnonzero(P[10, :n] >= thr)
    ref = np.full(n, -1); ref[keep] = np.arange(keep.size)
    assert int(n_keep.item()) == keep.size
    assert np.array_equal(new_index.cpu().numpy(), ref)
    dst = torch.zeros_like(dP)
    _lib.compact_planes(dP, dst, n, new_index)
    assert np.array_equal(dst[:, :keep.size].cpu().numpy(), P[:, keep])
