"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Tolerances: integer outputs bit-exact; images |d| <= 1e-4 |ora| + 1e-6 outside
oracle-flagged ambiguous pixels; gradients and S |d| <= 1e-3 |ora| + 1e-5 abs_ora outside
Gaussians of ambiguous pixels; densify mask / dest / n_split bit-exact on inputs kept out of the
eps_split guard band."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEFAULT = dict(alpha_min=1.0 / 255.0, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), tile=16)
SMOOTH = dict(alpha_min=0.0, alpha_max=1.0, t_min=0.0, dilation=0.0, bg=(0.0, 0.0, 0.0), tile=16)
BG = dict(DEFAULT, bg=(0.2, 0.4, 0.6))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_05587_b200 import require_cuda
    require_cuda()


def expected_binning(decs, W, H, T=16):
    tx, ty = (W + T - 1) // T, (H + T - 1) // T
    tpv = tx * ty
    keys_all, rank_all, ids_all = [], [], []
    for v, d in enumerate(decs):
        vis = np.flatnonzero(d["visible"])
        order = vis[np.lexsort((vis, d["key"][vis]))]            # (depth key, index) — C7
        r = d["rect"][order]
        x0, x1, y0, y1 = r[:, 0] // T, r[:, 1] // T, r[:, 2] // T, r[:, 3] // T
        for g, a0, a1, b0, b1, rk in zip(order, x0, x1, y0, y1, range(len(order))):
            xs, ys = np.meshgrid(np.arange(a0, a1 + 1), np.arange(b0, b1 + 1))
            k = v * tpv + ys.ravel() * tx + xs.ravel()
            keys_all.append(k)
            rank_all.append(np.full(k.size, rk))
            ids_all.append(np.full(k.size, g))
    if not keys_all:
        return np.zeros(0, np.int64), np.zeros((len(decs) * tpv,), np.int64)
    keys = np.concatenate(keys_all); rank = np.concatenate(rank_all); ids = np.concatenate(ids_all)
    o = np.lexsort((rank, keys))
    counts = np.bincount(keys, minlength=len(decs) * tpv)
    return ids[o], counts


def _cmp_decisions(orc, params, cams, rp, rz, n):
    from gpu_run import decisions, splat_fields
    g = decisions(rz, n)
    sf = splat_fields(rz, n)
    for v, cam in enumerate(cams):
        d = orc.decide(params, cam, rp)
        vis = d["visible"].astype(bool)
        assert np.array_equal(g["tiles_touched"][v] > 0, vis)
        assert np.array_equal(g["tiles_touched"][v][vis], d["tiles_touched"][vis])
        assert np.array_equal(g["key"][v][vis], d["key"][vis])
        assert np.array_equal(g["tile_rect"][v][vis], d["rect"][vis] // 16)
        pr = orc.project(params, cam, rp)
        assert np.allclose(sf["mean"][v][vis], pr["mu"][vis], rtol=1e-12, atol=1e-9)
        cscale = np.abs(pr["conic"][vis]).max(1, keepdims=True)        # fp64-formed, rounded once to fp32
        assert (np.abs(sf["conic"][v][vis] - pr["conic"][vis]) <= 1e-6 * cscale).all()
        assert np.allclose(sf["opacity"][v][vis], pr["opacity"][vis], rtol=1e-6)


@pytest.mark.parametrize("model", [0, 1])
def test_project_and_binning_bitexact_c1(orc, model):
    from gpu_run import run_forward
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=3, model=model)
    rz, _ = run_forward(p, cams, DEFAULT)
    _cmp_decisions(orc, p, cams, DEFAULT, rz, p.shape[1])
    ids, counts = expected_binning([orc.decide(p, c, DEFAULT) for c in cams], 64, 64)
    b = rz.binning_arrays()
    assert b["overflow"] == 0 and b["n_instances"] == ids.size
    assert np.array_equal(b["ids"].numpy().astype(np.int64), ids)
    assert np.array_equal((b["ranges"][:, 1] - b["ranges"][:, 0]).numpy(), counts)
    _check_tile_order(b, counts, cams)


def _check_tile_order(b, counts, cams):
    """binning.tile_order: a permutation of the (view, tile) indices (view << 20 | tile) whose list
    lengths are non-increasing in half-octave buckets (a scheduling order only)."""
    t = b["tile_order"].numpy().astype(np.int64)
    tpv = counts.size // len(cams)
    flat = (t >> 20) * tpv + (t & 0xFFFFF)
    assert ((t & 0xFFFFF) < tpv).all() and np.array_equal(np.sort(flat), np.arange(counts.size))
    L = counts[flat].astype(np.int64)
    nz = L > 0
    c = np.where(nz, 31 - np.floor(np.log2(np.maximum(L, 1))).astype(np.int64), 32)
    nb = np.where(nz & (c < 31), (L >> np.maximum(30 - c, 0)) & 1, 0)
    key = np.where(nz, 2 * c + 1 - nb, 64)
    assert (np.diff(key) >= 0).all()


def test_project_and_binning_bitexact_full_size_c2(orc):
    """BASELINE configs[1] at full size (1.0M Gaussians, 980x545), 2 views in one call."""
    from gpu_run import run_forward
    cfg = synth.CONFIGS["C2"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2)
    rz, _ = run_forward(p, cams, DEFAULT)
    _cmp_decisions(orc, p, cams, DEFAULT, rz, p.shape[1])
    decs = [orc.decide(p, c, DEFAULT) for c in cams]
    ids, counts = expected_binning_fast(decs, cfg.width, cfg.height)
    b = rz.binning_arrays()
    assert b["overflow"] == 0 and b["n_instances"] == ids.size
    assert b["n_visible"] == sum(int(d["visible"].sum()) for d in decs)
    assert np.array_equal(b["ids"].numpy().astype(np.int64), ids)
    assert np.array_equal((b["ranges"][:, 1] - b["ranges"][:, 0]).numpy(), counts)
    _check_tile_order(b, counts, cams)


def expected_binning_fast(decs, W, H, T=16):
    """Vectorised version of expected_binning for large n (same definition)."""
    tx, ty = (W + T - 1) // T, (H + T - 1) // T
    tpv = tx * ty
    K, R, I = [], [], []
    for v, d in enumerate(decs):
        vis = np.flatnonzero(d["visible"])
        order = vis[np.lexsort((vis, d["key"][vis]))]
        r = d["rect"][order].astype(np.int64)
        x0, x1, y0, y1 = r[:, 0] // T, r[:, 1] // T, r[:, 2] // T, r[:, 3] // T
        w, h = x1 - x0 + 1, y1 - y0 + 1
        cnt = w * h
        g = np.repeat(np.arange(order.size), cnt)
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        local = np.arange(cnt.sum()) - np.repeat(start, cnt)
        ly, lx = local // np.repeat(w, cnt), local % np.repeat(w, cnt)
        K.append(v * tpv + (np.repeat(y0, cnt) + ly) * tx + np.repeat(x0, cnt) + lx)
        R.append(g)
        I.append(order[g])
    keys = np.concatenate(K); rank = np.concatenate(R); ids = np.concatenate(I)
    o = np.lexsort((rank, keys))
    return ids[o], np.bincount(keys, minlength=len(decs) * tpv)


def _img_close(g, o, amb):
    ok = np.abs(g - o) <= 1e-4 * np.abs(o) + 1e-6
    ok |= amb[None] != 0
    return ok


@pytest.mark.parametrize("model,rp", [(0, DEFAULT), (1, DEFAULT), (0, BG), (1, SMOOTH)])
def test_render_fwd_parity_c1(orc, model, rp):
    from gpu_run import run_forward
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2, model=model)
    rz, _ = run_forward(p, cams, rp)
    img = rz.image.cpu().numpy()
    T = rz.final_T.cpu().numpy()
    for v, cam in enumerate(cams):
        o = orc.render(p, cam, rp)
        ok = _img_close(img[v], o["image"], o["amb_px"])
        assert ok.all(), (np.abs(img[v] - o["image"]).max(), int((~ok).sum()))
        okT = np.abs(T[v] - o["final_T"]) <= 1e-4 * o["final_T"] + 1e-6
        assert (okT | (o["amb_px"] != 0)).all()


# Elements that pass only through the plane floor of _grad_close: (test id, count, compared elements);
# printed at the end of the session by tests/conftest.py (pytest_terminal_summary).
FLOOR_LOG: list = []


def _grad_close(g, o, absg, ambg, rtol=1e-3, atol_rel=1e-5, plane_rel=1e-6, max_floor_frac=1e-3, absS=None):
    """|d| <= 1e-3 |ora| + 1e-5 abs_ora (north_star's rel 1e-3 plus the absolute term
    that absorbs fp32 cancellation in per-pair sums).  A third term, 1e-6 max_i |ora[plane]|, is the
    fp32 floor of gradients that are small differences of O(|dL/dSigma| |Sigma|) terms (e.g. the
    quaternion gradient of a nearly isotropic Gaussian, where the per-pair terms cancel in the
    Jacobian and not in the sum abs_ora sees).  It is allowed for at most max(4, 1e-3 of the compared
    elements) per call; the count is asserted, logged and printed at the end of the run.
    absS ([6][n], optional): for the S planes abs_ora is the sum of the per-pair term magnitudes
    |g sigma|(|U_a U_b| + |(P^T Q P)_ab|) — the GPU forms S = P^T (QMQ - m0 Q) P from per-Gaussian
    moment sums (C12), whose fp32 error scales with both terms, not with their per-pair difference."""
    import os
    if absS is not None:   # S planes: the moment formulation's term magnitudes
        absg = absg.copy()
        absg[14:20] = np.maximum(absg[14:20], absS)
    d = np.abs(g - o)
    strict = d <= rtol * np.abs(o) + atol_rel * absg + 1e-30
    floor = plane_rel * np.abs(o).max(axis=1, keepdims=True)
    ok = d <= rtol * np.abs(o) + atol_rel * absg + floor + 1e-30
    ok[:, ambg != 0] = True
    strict[:, ambg != 0] = True
    need = int((ok & ~strict).sum())
    FLOOR_LOG.append((os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], need, int(strict.size)))
    assert need <= max(4, max_floor_frac * strict.size), f"{need} of {strict.size} elements need the plane floor"
    return ok


def _grad_report(g, o, absg, ok):
    rows = []
    for k in range(g.shape[0]):
        if ok[k].all():
            continue
        bad = np.flatnonzero(~ok[k])
        i = bad[np.argmax(np.abs(g[k, bad] - o[k, bad]))]
        rows.append(dict(plane=k, n_bad=int(bad.size), err=float(abs(g[k, i] - o[k, i])), ora=float(o[k, i]),
                         absg=float(absg[k, i]), plane_max=float(np.abs(o[k]).max())))
    return rows


@pytest.mark.parametrize("model,rp", [(0, DEFAULT), (1, DEFAULT), (0, BG), (1, SMOOTH)])
def test_render_bwd_split_parity_c1(orc, model, rp):
    from gpu_run import run_backward, run_forward
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2, model=model)
    dl = synth.dl_dimage(2, 64, 64, 77)
    # pixels the oracle flags as ambiguous (a threshold decision within rounding) get dL/dC = 0 on
    # both sides, so they contribute nothing and every Gaussian is compared
    n_amb = 0
    for v, cam in enumerate(cams):
        amb_px = orc.render(p, cam, rp)["amb_px"] != 0
        dl[v][:, amb_px] = 0.0
        n_amb += int(amb_px.sum())
    assert n_amb <= 0.01 * dl[0, 0].size * len(cams)
    rz, pt = run_forward(p, cams, rp)
    g = run_backward(rz, pt, dl)
    o = np.zeros_like(g); a = np.zeros_like(g); amb = np.zeros(p.shape[1], np.uint8)
    for v, cam in enumerate(cams):
        r = orc.render(p, cam, rp, dl_dimage=dl[v])
        o += r["grad"]; a += r["absg"]
    ok = _grad_close(g, o, a, amb)
    assert ok.all(), _grad_report(g, o, a, ok)
    # moments workspace is left zeroed by the call
    assert float(rz.moments.abs().max()) == 0.0


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_render_windows_full_size(orc, name):
    """Full-size BASELINE configs (C2 1.0M 980x545 ... C5 6M 1920x1080): the decision chain of every
    Gaussian bit-exact; the oracle evaluates 3 windows (images) and the gradients/S of dL restricted
    to those windows (including the ragged bottom-right corner tile)."""
    from gpu_run import run_backward, run_forward
    cfg = synth.CONFIGS[name]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=1)
    cam = cams[0]
    rz, pt = run_forward(p, cams, DEFAULT)
    if name != "C2":
        _cmp_decisions(orc, p, cams, DEFAULT, rz, p.shape[1])
    img = rz.image.cpu().numpy()[0]
    W, H = cfg.width, cfg.height
    windows = [(0, 0, 40, 32), (W // 2 - 24, H // 2 - 20, 48, 40), (W - 49, H - 45, 49, 45)]
    dl_full = synth.dl_dimage(1, cfg.width, cfg.height, 5)[0]
    dl = np.zeros_like(dl_full)
    dec = orc.decide(p, cam, DEFAULT)
    n_amb_px = 0
    for (x0, y0, w, h) in windows:
        r = orc.render(p, cam, DEFAULT, window=(x0, y0, w, h), decision=dec)
        gi = img[:, y0:y0 + h, x0:x0 + w]
        ok = _img_close(gi, r["image"], r["amb_px"])
        assert ok.all(), (np.abs(gi - r["image"]).max(), int((~ok).sum()))
        win = dl_full[:, y0:y0 + h, x0:x0 + w].copy()
        win[:, r["amb_px"] != 0] = 0.0                      # ambiguous pixels carry no gradient
        dl[:, y0:y0 + h, x0:x0 + w] = win
        n_amb_px += int(r["amb_px"].sum())
    # excluded pixels are bounded (threshold decisions within rounding are rare)
    assert n_amb_px <= 0.01 * sum(w * h for (_, _, w, h) in windows), n_amb_px
    g = run_backward(rz, pt, dl[None])
    o = np.zeros_like(g); a = np.zeros_like(g); amb = np.zeros(p.shape[1], np.uint8)
    for (x0, y0, w, h) in windows:
        r = orc.render(p, cam, DEFAULT, window=(x0, y0, w, h), dl_dimage=dl[:, y0:y0 + h, x0:x0 + w], decision=dec)
        o += r["grad"]; a += r["absg"]
    touched = np.flatnonzero(a[14:20].sum(0) > 0)
    assert touched.size > 500
    ok = _grad_close(g[:, touched], o[:, touched], a[:, touched], amb[touched])
    assert ok.all(), _grad_report(g[:, touched], o[:, touched], a[:, touched], ok)
    # gradients vanish exactly for Gaussians that no window pixel reaches
    untouched = np.setdiff1d(np.arange(p.shape[1]), np.flatnonzero(a.sum(0) > 0))
    assert np.abs(g[:, untouched]).max() == 0.0


def test_l1_grad_and_loss():
    from gpu_run import to_dev
    from paper_2505_05587_b200 import _lib
    rng = np.random.default_rng(0)
    a = rng.uniform(size=(2, 3, 17, 23)).astype(np.float32)
    t = rng.uniform(size=a.shape).astype(np.float32)
    t[0, 0, 0, :5] = a[0, 0, 0, :5]  # exact ties -> sign 0
    A, Tt = to_dev(a), to_dev(t)
    dL = torch.empty_like(A)
    loss = torch.zeros(2, device="cuda")
    cnt = 3 * 17 * 23
    _lib.l1_grad(A, Tt, 2, cnt, 1.0 / cnt, dL, loss)
    torch.cuda.synchronize()
    assert np.array_equal(dL.cpu().numpy(), (np.sign(a - t) / np.float32(cnt)).astype(np.float32))
    ref = np.abs(a.astype(np.float64) - t).reshape(2, -1).mean(1)
    assert np.allclose(loss.cpu().numpy(), ref, rtol=1e-5)


def test_multiview_call_equals_sum_of_single_views(orc):
    """Shard emulation: one V=4 call == sum of four V=1 calls (S is additive over views)."""
    from gpu_run import run_backward, run_forward
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=4)
    dl = synth.dl_dimage(4, 64, 64, 3)
    rz, pt = run_forward(p, cams, DEFAULT)
    g4 = run_backward(rz, pt, dl)
    acc = np.zeros_like(g4)
    for v in range(4):
        r1, p1 = run_forward(p, cams[v:v + 1], DEFAULT)
        acc += run_backward(r1, p1, dl[v:v + 1])
    assert np.allclose(g4, acc, rtol=1e-4, atol=1e-6 * np.abs(acc).max())


def test_empty_and_all_culled(orc):
    from gpu_run import run_backward, run_forward
    cfg = synth.CONFIGS["C1"]
    cam = synth.cameras_for(cfg, views=1)
    p = synth.scene_for(cfg)
    p_behind = p.copy()
    p_behind[0:3] = np.array([[50.0], [50.0], [50.0]], np.float32)   # far outside every frustum
    rz, pt = run_forward(p_behind, cam, BG)
    img = rz.image.cpu().numpy()[0]
    assert np.allclose(img, np.array(BG["bg"], np.float32)[:, None, None])
    assert rz.binning_arrays()["n_instances"] == 0
    g = run_backward(rz, pt, synth.dl_dimage(1, 64, 64, 1))
    assert np.abs(g).max() == 0.0


# ------------------------------------------------------------------------------------------------
# densify
# ------------------------------------------------------------------------------------------------
def _densify_inputs(orc, n, seed, eps_split=-1e-6, denom=3.0):
    """Seeded params + S planes with no lambda_min inside the guard band of eps_split
    (oracle-decided, fp64)."""
    p = synth.blob_scene(n, seed)
    S = synth.splitting_matrices(n, seed + 1, scale=1e-3).astype(np.float32)
    for _ in range(10):
        bad = []
        for i in range(n):
            A = S[:, i].astype(np.float64) / np.float32(denom)
            lam, _ = orc.eig_sym3(A)
            fro = np.sqrt(A[0] ** 2 + A[3] ** 2 + A[5] ** 2 + 2 * (A[1] ** 2 + A[2] ** 2 + A[4] ** 2))
            if abs(lam[0] - eps_split) <= 1e-4 * fro:
                bad.append(i)
        if not bad:
            break
        for i in bad:
            S[[0, 3, 5], i] += np.float32(3e-4 * 1e-3 * denom)
    return p, S


def _gpu_densify(p, S, n, cap, **kw):
    from gpu_run import to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    P = torch.zeros(14, cap, dtype=torch.float32, device="cuda")
    P[:, :n] = to_dev(p)
    G = torch.zeros(20, cap, dtype=torch.float32, device="cuda")
    G[14:20, :n] = to_dev(S)
    G[0:14, :n] = 1.0
    rz = Rasterizer(cap, 1, 16, 16)
    rz.densify(P, G, n, cap, **kw)
    torch.cuda.synchronize()
    return rz, P, G


@pytest.mark.parametrize("eta", [0.5, -1.0])
def test_densify_parity(orc, eta):
    n, cap, denom = 6000, 12000, 3.0
    p, S = _densify_inputs(orc, n, 11, denom=denom)
    rz, P, G = _gpu_densify(p, S, n, cap, eta=eta, eps_abs=0.05, denom=denom)
    accd = np.zeros((20, cap)); accd[14:20, :n] = S
    pd = np.zeros((14, cap)); pd[:, :n] = p
    r = orc.densify(pd, accd, n, cap, denom=denom, eps_split=-1e-6, eta=eta, eps_abs=np.float32(0.05))
    ns = int(rz.n_split.item())
    assert int(rz.dens_status.item()) == 0
    assert ns == r["n_split"] > 0
    assert np.array_equal(rz.split_mask[:n].cpu().numpy(), r["mask"])
    assert np.array_equal(rz.dest_index[:n].cpu().numpy(), r["dest"])
    lam = rz.lambda_min[:n].cpu().numpy()
    Sn = np.abs(S).max(0) / denom
    assert (np.abs(lam - r["lambda_min"]) <= 1e-4 * Sn * 3 + 1e-12).all()
    Pg = P.cpu().numpy().astype(np.float64)
    Gg = G.cpu().numpy()
    assert np.abs(Gg[14:20, :n + ns]).max() == 0.0                      # Z23
    assert np.abs(Gg[:, n:n + ns]).max() == 0.0
    keep = r["mask"] == 0
    assert np.array_equal(Pg[:, :n][:, keep], p[:, keep].astype(np.float64))   # untouched bit-exact
    sp = np.flatnonzero(r["mask"])
    b = r["dest"][sp]
    # offspring: an unordered pair {A, B} per parent (Z16); logits abs 1e-6 (C15)
    ga, gb = Pg[0:3, sp], Pg[0:3, b]
    oa, ob = r["params"][0:3, sp], r["params"][0:3, b]
    scale = np.abs(p[0:3]).max()
    tol = 1e-4 * scale
    same = (np.abs(ga - oa).max(0) <= tol) & (np.abs(gb - ob).max(0) <= tol)
    swap = (np.abs(ga - ob).max(0) <= tol) & (np.abs(gb - oa).max(0) <= tol)
    gap = np.array([np.diff(orc.eig_sym3(S[:, i].astype(np.float64) / denom)[0])[0] for i in sp])
    fro = np.abs(S[:, sp]).max(0) / denom
    near_degenerate = gap < 1e-3 * fro
    assert (same | swap | near_degenerate).all(), int((~(same | swap | near_degenerate)).sum())
    # Z16, for every split parent (and the only check where the min-eigenspace is (nearly) repeated):
    # v = (A - B) / |A - B| is a unit min-eigenvector of S-bar by its residual and Rayleigh quotient,
    # and the offspring half-distance is eps = eta sqrt(v^T Sigma v) (C15) or eps_abs.
    from scipy.spatial.transform import Rotation
    dAB = ga - gb
    half = 0.5 * np.linalg.norm(dAB, axis=0)
    v = dAB / np.maximum(2.0 * half, 1e-300)
    Sb = S[:, sp].astype(np.float64) / denom
    Sm = np.stack([np.stack([Sb[0], Sb[1], Sb[2]]), np.stack([Sb[1], Sb[3], Sb[4]]),
                   np.stack([Sb[2], Sb[4], Sb[5]])]).transpose(2, 0, 1)           # [k][3][3]
    lam_o = r["lambda_min"][sp]
    Sv = np.einsum("kab,bk->ak", Sm, v)
    res = np.linalg.norm(Sv - lam_o[None] * v, axis=0)
    rq = np.einsum("ak,ak->k", v, Sv)
    fro_f = np.linalg.norm(Sm.reshape(-1, 9), axis=1)
    # the position difference carries ~1e-7 |p| / half of rounding in v, and the fp32 eigensolve ~1e-6
    vtol = 1e-4 * fro_f + fro_f * 4e-7 * scale / np.maximum(half, 1e-30)
    assert (res <= np.maximum(vtol, gap + vtol)).all(), np.max(res / np.maximum(vtol, gap + vtol))
    assert (np.abs(rq - lam_o) <= np.maximum(vtol, gap + vtol)).all()
    q = p[6:10, sp].astype(np.float64)
    Rm = Rotation.from_quat(np.stack([q[1], q[2], q[3], q[0]], 1)).as_matrix()  # scipy: (x, y, z, w)
    s2 = np.exp(2.0 * p[3:6, sp].astype(np.float64)).T
    Sig = np.einsum("kab,kb,kcb->kac", Rm, s2, Rm)
    eps_ref = eta * np.sqrt(np.einsum("ak,kab,bk->k", v, Sig, v)) if eta > 0 else np.full(sp.size, 0.05)
    assert np.allclose(half, eps_ref, rtol=2e-4, atol=1e-6 * scale), np.max(np.abs(half - eps_ref) / eps_ref)
    assert np.allclose(0.5 * (ga + gb), p[0:3, sp], atol=1e-6 * scale)    # mean(offspring) = parent
    assert np.abs(Pg[10, sp] - r["params"][10, sp]).max() <= 1e-6
    assert np.abs(Pg[10, b] - r["params"][10, b]).max() <= 1e-6
    assert np.array_equal(Pg[3:10, b], Pg[3:10, sp]) and np.array_equal(Pg[11:14, b], Pg[11:14, sp])


def test_densify_capacity_exceeded(orc):
    n = 3000
    p, S = _densify_inputs(orc, n, 5)
    rz, P, G = _gpu_densify(p, S, n, n + 1, denom=3.0)
    assert int(rz.dens_status.item()) == 3
    assert np.array_equal(P[:, :n].cpu().numpy(), p)
    assert np.array_equal(G[14:20, :n].cpu().numpy(), S)


def test_densify_full_size_c4(orc):
    """BASELINE configs[3] shape: 2.5M Gaussians; mask/dest/n_split checked on a 50k sample window
    whose ranks are offset by the GPU-independent oracle count of the prefix."""
    n = 2_500_000
    p = synth.surface_scene(n, 1004)
    S = synth.splitting_matrices(n, 2004, neg_frac=0.1, scale=1e-3)
    rz, P, G = _gpu_densify(p, S, n, 2 * n, denom=1.0)
    mask = rz.split_mask[:n].cpu().numpy()
    lam = rz.lambda_min[:n].cpu().numpy()
    # sample: oracle decides every Gaussian of a window (fp64 Jacobi); outside the guard band it
    # must agree with the kernel's mask
    idx = np.arange(1_000_000, 1_050_000)
    for i in idx[::7]:
        l, _ = orc.eig_sym3(S[:, i].astype(np.float64))
        fro = np.abs(S[:, i]).max()
        if abs(l[0] + 1e-6) > 1e-4 * fro:
            assert mask[i] == (l[0] < -1e-6)
        assert abs(lam[i] - l[0]) <= 3e-4 * fro + 1e-12
    ns = int(rz.n_split.item())
    assert ns == int(mask.sum())
    dest = rz.dest_index[:n].cpu().numpy()
    assert np.array_equal(dest[mask == 1], n + np.arange(ns))


def _gpu_densify_g(p, S, G, n, cap, **kw):
    from gpu_run import to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    P = torch.zeros(14, cap, dtype=torch.float32, device="cuda")
    P[:, :n] = to_dev(p)
    A = torch.zeros(20, cap, dtype=torch.float32, device="cuda")
    A[14:20, :n] = to_dev(S)
    A[0:3, :n] = to_dev(G)
    rz = Rasterizer(cap, 1, 16, 16)
    rz.densify(P, A, n, cap, **kw)
    torch.cuda.synchronize()
    return rz, P, A


@pytest.mark.parametrize("fused", [True, False])
def test_densify_budget_and_gate_parity(orc, fused):
    """App. A.2 variants: increment budget (least lambda_min first, ties by index) and the compactest
    gate; inputs keep lambda_min away from eps_split, |G| away from eps_grad, and the budget cut
    away from near-equal lambda values (oracle-decided)."""
    n, denom = 5000, 2.0
    cap = 2 * n if fused else n + n // 2 + 64
    p, S = _densify_inputs(orc, n, 31, denom=denom)
    rng = np.random.default_rng(32)
    G = (rng.lognormal(0.0, 1.0, size=(3, n)) * 1e-3 * rng.choice([-1.0, 1.0], size=(3, n))).astype(np.float32)
    gn = np.linalg.norm(G.astype(np.float64) / denom, axis=0)
    eps_grad = float(np.median(gn))
    G[:, np.abs(gn - eps_grad) <= 1e-4 * eps_grad] *= 1.5
    lam = np.array([orc.eig_sym3(S[:, i].astype(np.float64) / denom)[0][0] for i in range(n)])
    cand = np.flatnonzero(lam < -1e-6)
    K = len(cand) // 3
    srt = np.sort(lam[cand])
    while abs(srt[K] - srt[K - 1]) <= 1e-4 * np.abs(srt).max():    # a clear cut between kept / dropped
        K += 1
    accd = np.zeros((20, cap)); pd = np.zeros((14, cap)); pd[:, :n] = p
    for kw in (dict(budget=K), dict(eps_grad=eps_grad), dict(budget=K // 2, eps_grad=eps_grad)):
        accd[:] = 0.0
        accd[14:20, :n] = S
        accd[0:3, :n] = G
        r = orc.densify(pd, accd, n, cap, denom=denom, **kw)
        rz, P, A = _gpu_densify_g(p, S, G, n, cap, denom=denom, **kw)
        assert int(rz.dens_status.item()) == 0
        assert int(rz.n_split.item()) == r["n_split"] > 0, kw
        assert np.array_equal(rz.split_mask[:n].cpu().numpy(), r["mask"]), kw
        assert np.array_equal(rz.dest_index[:n].cpu().numpy(), r["dest"]), kw
        if "budget" in kw:
            assert r["n_split"] <= kw["budget"]
    # gate 2 (C24): planes 0, 1 = (sum of view-gradient norms, visible views)
    cnt = rng.integers(0, 5, size=n).astype(np.float32)
    ssum = (cnt * rng.uniform(0, 2e-3, size=n)).astype(np.float32)
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = np.where(cnt > 0, ssum.astype(np.float64) / cnt, 0.0)
    gg = 7e-4
    ssum[np.abs(mean - gg) <= 1e-4 * gg] *= 1.5
    G2 = np.zeros((3, n), np.float32); G2[0] = ssum; G2[1] = cnt
    for kw in (dict(grad_gate=gg), dict(grad_gate=gg, budget=K // 3)):
        accd[:] = 0.0
        accd[14:20, :n] = S
        accd[0:3, :n] = G2
        r = orc.densify(pd, accd, n, cap, denom=denom, **kw)
        rz, P, A = _gpu_densify_g(p, S, G2, n, cap, denom=denom, **kw)
        assert int(rz.n_split.item()) == r["n_split"] > 0, kw
        assert np.array_equal(rz.split_mask[:n].cpu().numpy(), r["mask"]), kw
        assert np.array_equal(rz.dest_index[:n].cpu().numpy(), r["dest"]), kw


def test_densify_budget_exact_ties(orc):
    n = 40
    p = synth.blob_scene(n, 3)
    S = np.zeros((6, n), np.float32)
    S[[0, 3, 5]] = 1.0
    for i in (3, 7, 8, 20, 21, 33):
        S[:, i] = [-2.0, 0.1, 0.0, 1.0, 0.0, 1.0]          # identical indefinite matrices: exact ties
    S[:, 30] = [-5.0, 0.0, 0.0, 1.0, 0.0, 1.0]             # strictly smallest
    G = np.zeros((3, n), np.float32)
    for K in (0, 1, 3, 7, 100):
        accd = np.zeros((20, 2 * n)); accd[14:20, :n] = S
        pd = np.zeros((14, 2 * n)); pd[:, :n] = p
        r = orc.densify(pd, accd, n, 2 * n, budget=K)
        rz, _, _ = _gpu_densify_g(p, S, G, n, 2 * n, budget=K)
        assert np.array_equal(rz.split_mask[:n].cpu().numpy(), r["mask"]), K
        assert np.array_equal(rz.dest_index[:n].cpu().numpy(), r["dest"]), K
    assert list(np.flatnonzero(r["mask"])) == [3, 7, 8, 20, 21, 30, 33]


def test_bench_launch_configuration_c2(orc):
    """The exact launch bench.py times: C2 (1.0M Gaussians, 980x545), 8 views per call, capacity 2n,
    max_instances 3 V n.  Binning of all 8 views bit-exact; images and dL-restricted gradients / S
    of sampled windows in two of the views against the oracle."""
    from gpu_run import to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    cfg = synth.CONFIGS["C2"]
    n, V = cfg.n, 8
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=V)
    cap = 2 * n
    P = torch.zeros(14, cap, device="cuda"); P[:, :n] = to_dev(p)
    rz = Rasterizer(cap, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n))
    rz.project(P, n, cams); rz.bin_sort(); rz.render_fwd()
    decs = [orc.decide(p, c, DEFAULT) for c in cams]
    ids, counts = expected_binning_fast(decs, cfg.width, cfg.height)
    b = rz.binning_arrays()
    assert b["overflow"] == 0 and b["n_instances"] == ids.size
    assert np.array_equal(b["ids"].numpy().astype(np.int64), ids)
    assert np.array_equal((b["ranges"][:, 1] - b["ranges"][:, 0]).numpy(), counts)
    img = rz.image.cpu().numpy()
    W, H = cfg.width, cfg.height
    dl = np.zeros((V, 3, H, W), np.float32)
    full = synth.dl_dimage(V, W, H, 17)
    wins = {2: [(100, 60, 40, 32)], 5: [(W - 49, H - 45, 49, 45), (W // 2, H // 2, 32, 24)]}
    n_amb = 0
    for v, ws in wins.items():
        for (x0, y0, w, h) in ws:
            r = orc.render(p, cams[v], DEFAULT, window=(x0, y0, w, h), decision=decs[v])
            ok = _img_close(img[v][:, y0:y0 + h, x0:x0 + w], r["image"], r["amb_px"])
            assert ok.all()
            n_amb += int(r["amb_px"].sum())
            assert n_amb <= 0.01 * sum(w_ * h_ for ws_ in wins.values() for (_, _, w_, h_) in ws_)
            win = full[v][:, y0:y0 + h, x0:x0 + w].copy()
            win[:, r["amb_px"] != 0] = 0.0
            dl[v][:, y0:y0 + h, x0:x0 + w] = win
    acc = torch.zeros(20, cap, device="cuda")
    rz.render_bwd(P, acc, dL=to_dev(dl))
    g = acc[:, :n].cpu().numpy().astype(np.float64)
    o = np.zeros((20, n)); a = np.zeros((20, n))
    for v, ws in wins.items():
        for (x0, y0, w, h) in ws:
            r = orc.render(p, cams[v], DEFAULT, window=(x0, y0, w, h), dl_dimage=dl[v][:, y0:y0 + h, x0:x0 + w],
                           decision=decs[v])
            o += r["grad"]; a += r["absg"]
    touched = np.flatnonzero(a[14:20].sum(0) > 0)
    assert touched.size > 100
    ok = _grad_close(g[:, touched], o[:, touched], a[:, touched], np.zeros(touched.size, np.uint8))
    assert ok.all(), _grad_report(g[:, touched], o[:, touched], a[:, touched], ok)
    assert np.abs(np.delete(g, np.flatnonzero(a.sum(0) > 0), axis=1)).max() == 0.0


def test_stage_graph_replay_equals_eager():
    """bench.py's launch mode: one CUDA graph per stage, captured after an eager step and replayed.
    Binning, image, T, n_contrib and dL/dimage bit-identical to the eager launch; grads + S equal up to
    the order of the backward's float atomics."""
    from gpu_run import to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    cfg = synth.CONFIGS["C2"]
    n, V = cfg.n, 2
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=V)
    tg = to_dev(synth.targets_for(cfg, views=V))
    cap = 2 * n
    P = torch.zeros(14, cap, device="cuda"); P[:, :n] = to_dev(p)
    G = torch.zeros(20, cap, device="cuda")
    rz = Rasterizer(cap, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n))
    stages = [lambda: rz.project(P, n, cams), rz.bin_sort, lambda: rz.render_fwd_l1(tg), rz.render_bwd_moments,
              lambda: rz.gauss_bwd(P, G, accumulate=0)]
    for f in stages:
        f()
    torch.cuda.synchronize()
    b = rz.binning_arrays()
    ref = dict(ids=b["ids"].clone(), ranges=b["ranges"].clone(), image=rz.image.clone(), T=rz.final_T.clone(),
               nc=rz.n_contrib.clone(), dL=rz.dL.clone(), G=G.clone())
    graphs = []
    for f in stages:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graphs.append(g)
    for t in (rz.image, rz.final_T, rz.dL, G):
        t.zero_()
    rz.n_contrib.zero_()
    for g in graphs:
        g.replay()
    torch.cuda.synchronize()
    b = rz.binning_arrays()
    assert torch.equal(b["ids"], ref["ids"]) and torch.equal(b["ranges"], ref["ranges"])
    for k, t in (("image", rz.image), ("T", rz.final_T), ("nc", rz.n_contrib), ("dL", rz.dL)):
        assert torch.equal(t, ref[k]), k
    scale = ref["G"][:, :n].abs().amax(dim=1, keepdim=True).clamp_min(1e-30)
    assert ((G[:, :n] - ref["G"][:, :n]).abs() / scale).max().item() < 1e-4
    assert ref["G"][14:20, :n].abs().sum().item() > 0


def test_whole_step_graph_replay_equals_eager():
    """bench.py's timed launch: the whole step (project .. densify) captured as ONE CUDA graph, so the
    programmatic-dependent launches chain across stages inside the graph.  Binning, image, T and
    dL/dimage bit-identical to the eager step; grads + S equal up to the backward's float atomics;
    densify's split count within a few Gaussians (lambda_min decided on those S) and its mask / dest
    consistent."""
    from gpu_run import to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    cfg = synth.CONFIGS["C2"]
    n, V = cfg.n, 2
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=V)
    tg = torch.from_numpy(np.clip(np.rint(synth.targets_for(cfg, views=V) * 255.0), 0, 255).astype(np.uint8)).cuda()
    cap = 2 * n
    P0 = torch.zeros(14, cap, device="cuda"); P0[:, :n] = to_dev(p)
    P = P0.clone()
    G = torch.zeros(20, cap, device="cuda")
    rz = Rasterizer(cap, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n))

    def step():
        rz.project(P, n, cams)
        rz.bin_sort()
        rz.render_fwd_l1(tg)
        rz.render_bwd_moments()
        rz.gauss_bwd(P, G, accumulate=0)
        rz.densify(P, G, n, cap, denom=float(V), want_lambda=False)

    step()
    torch.cuda.synchronize()
    b = rz.binning_arrays()
    ns0 = int(rz.n_split.item()) if torch.is_tensor(rz.n_split) else int(rz.n_split)
    ref = dict(ids=b["ids"].clone(), ranges=b["ranges"].clone(), image=rz.image.clone(), T=rz.final_T.clone(),
               dL=rz.dL.clone())
    P.copy_(P0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    P.copy_(P0)
    for t in (rz.image, rz.final_T, rz.dL, G):
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    b = rz.binning_arrays()
    assert torch.equal(b["ids"], ref["ids"]) and torch.equal(b["ranges"], ref["ranges"])
    for k, t in (("image", rz.image), ("T", rz.final_T), ("dL", rz.dL)):
        assert torch.equal(t, ref[k]), k
    ns1 = int(rz.n_split.item()) if torch.is_tensor(rz.n_split) else int(rz.n_split)
    assert ns0 > 0 and abs(ns1 - ns0) <= 8, (ns0, ns1)
    mask = rz.split_mask[:n].cpu().numpy().astype(bool)
    dest = rz.dest_index[:n].cpu().numpy()
    assert int(mask.sum()) == ns1 and np.array_equal(np.sort(dest[mask]), n + np.arange(ns1))


def test_render_fwd_l1_fused_equals_separate():
    """a3 + a4 fused (steepgs_render_fwd_l1): image, dL/dimage bit-identical to render_fwd + l1_grad, the
    per-view loss equal up to summation order."""
    from gpu_run import run_forward, to_dev
    cfg = synth.CONFIGS["C2"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2)
    tg = to_dev(synth.targets_for(cfg, views=2))
    rz, pt = run_forward(p, cams, DEFAULT)
    rz.l1_grad(tg)
    img0, dl0, loss0 = rz.image.clone(), rz.dL.clone(), rz.loss.clone()
    rz.dL.zero_(); rz.loss.fill_(7.0)
    rz.render_fwd_l1(tg)
    torch.cuda.synchronize()
    assert torch.equal(rz.image, img0) and torch.equal(rz.dL, dl0)
    assert torch.allclose(rz.loss, loss0, rtol=1e-5, atol=0)


def test_render_fwd_l1_u8_equals_float_targets():
    """steepgs_render_fwd_l1_u8: 8-bit targets decoded as fp32 target * (1/255) on the device — image,
    dL/dimage and the per-view loss bit-identical to steepgs_render_fwd_l1 on the decoded targets
    (which the test above ties to render_fwd + l1_grad, and the l1 parity test to the oracle)."""
    from gpu_run import run_forward, to_dev
    cfg = synth.CONFIGS["C2"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2)
    t8 = np.clip(np.rint(synth.targets_for(cfg, views=2) * 255.0), 0, 255).astype(np.uint8)
    dec = t8.astype(np.float32) * (np.float32(1.0) / np.float32(255.0))   # fp32, as on the device
    rz, pt = run_forward(p, cams, DEFAULT)
    rz.render_fwd_l1(to_dev(dec))
    img0, dl0, loss0 = rz.image.clone(), rz.dL.clone(), rz.loss.clone()
    assert (dl0 != 0).any() and (dl0 == 0).sum() < dl0.numel()
    rz.dL.zero_(); rz.loss.fill_(7.0)
    rz.render_fwd_l1(torch.from_numpy(t8).cuda())
    torch.cuda.synchronize()
    assert torch.equal(rz.image, img0) and torch.equal(rz.dL, dl0)
    assert torch.allclose(rz.loss, loss0, rtol=1e-5, atol=0)   # per-warp atomics: summation order


@pytest.mark.parametrize("pattern", ["separated", "min_pair", "max_pair"])
def test_densify_decisions_near_the_threshold(orc, pattern):
    """The split decision lambda_min(S_bar) < eps_split (Thm 2) for S whose lambda_min sits
    at 1e-7 .. 1e-3 ||S||_F from eps_split — inside and outside the kernel's fp64 guard band — with the
    other eigenvalues well separated, or lambda_min nearly repeated (min_pair), or the two larger ones
    nearly repeated (max_pair): the fp32 eigenvalue outside the band and the fp64 one inside it take
    the oracle's fp64 decision on every matrix (mask bit-exact)."""
    rng = np.random.default_rng({"separated": 71, "min_pair": 72, "max_pair": 73}[pattern])
    n, eps = 40_000, -1e-6
    F = 10.0 ** rng.uniform(-5, -1, size=n)                                  # ||S||_F scale
    delta = 10.0 ** rng.uniform(-7, -3, size=n) * rng.choice([-1.0, 1.0], size=n)
    l1 = eps + delta * F
    if pattern == "separated":
        l2 = l1 + F * rng.uniform(0.2, 0.6, size=n); l3 = l2 + F * rng.uniform(0.2, 0.6, size=n)
    elif pattern == "min_pair":
        l2 = l1 + F * 10.0 ** rng.uniform(-6, -2, size=n); l3 = l2 + F * rng.uniform(0.3, 0.8, size=n)
    else:
        l2 = l1 + F * rng.uniform(0.3, 0.8, size=n); l3 = l2 + F * 10.0 ** rng.uniform(-6, -2, size=n)
    S = np.zeros((6, n), np.float64)
    for i in range(n):
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        A = Q @ np.diag([l1[i], l2[i], l3[i]]) @ Q.T
        S[:, i] = [A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]]
    S = S.astype(np.float32)
    want = np.array([orc.eig_sym3(S[:, i].astype(np.float64))[0][0] < eps for i in range(n)])
    p = synth.blob_scene(n, 77)
    rz, _, _ = _gpu_densify(p, S, n, 2 * n, denom=1.0)
    got = rz.split_mask[:n].cpu().numpy().astype(bool)
    assert want.any() and (~want).any()
    assert np.array_equal(got, want), int((got != want).sum())
