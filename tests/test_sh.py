"""NEXT f3: view-dependent colour from spherical harmonics — oracle pins (-m "not gpu") and
GPU parity of the SH projection / backward kernels."""
import numpy as np
import pytest

import synth
from helpers import affine_cam

torch = pytest.importorskip("torch")

SMOOTH = dict(alpha_min=0.0, alpha_max=1.0, t_min=0.0, dilation=0.0, bg=(0.0, 0.0, 0.0), tile=16)
DEFAULT = dict(alpha_min=1.0 / 255.0, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), tile=16)


def sh_scene(n, seed, degree, dc_scale=1.0, rest_scale=0.15):
    """Seeded scene whose colours stay well inside the unclamped range (DC dominant)."""
    rng = np.random.default_rng(seed)
    p = synth.blob_scene(n, seed).astype(np.float64)
    p[11:14] = rng.uniform(0.2, 1.2, size=(3, n)) * dc_scale
    K = (degree + 1) ** 2
    rest = rng.normal(size=(3 * (K - 1), n)) * rest_scale
    return p, rest


# ---------------------------------------------------------------- CPU pins
def test_sh_basis_orthonormal(orc):
    """The 16 real SH functions are orthonormal on the unit sphere (Gauss-Legendre x uniform-phi
    quadrature, exact for the degree-6 products)."""
    xg, wg = np.polynomial.legendre.leggauss(12)
    phis = np.linspace(0, 2 * np.pi, 24, endpoint=False)
    G = np.zeros((16, 16))
    for ct, w in zip(xg, wg):
        st = np.sqrt(1 - ct * ct)
        for ph in phis:
            Y, _ = orc.sh_basis([st * np.cos(ph), st * np.sin(ph), ct], 3)
            G += w * (2 * np.pi / len(phis)) * np.outer(Y, Y)
    assert np.allclose(G, np.eye(16), atol=1e-12)


def test_sh_basis_derivatives(orc):
    rng = np.random.default_rng(3)
    for _ in range(5):
        v = rng.normal(size=3)
        _, dY = orc.sh_basis(v, 3)
        for j in range(3):
            h = 1e-6
            e = np.zeros(3); e[j] = h
            fd = (orc.sh_basis(v + e, 3)[0] - orc.sh_basis(v - e, 3)[0]) / (2 * h)
            assert np.allclose(dY[:, j], fd, rtol=1e-7, atol=1e-8)


def test_sh_degree0_equals_rgb_model(orc):
    """Degree 0: colour = C0 f + 1/2 for every view, i.e. the rgb model with rgb = C0 f + 1/2."""
    p, _ = sh_scene(20, 4, 0)
    cams = synth.ring_cameras(2, 48, 40, 5)
    q = p.copy()
    q[11:14] = 0.28209479177387814 * p[11:14] + 0.5
    for cam in cams:
        a = orc.render(p, cam, DEFAULT, sh_degree=0)["image"]
        b = orc.render(q, cam, DEFAULT)["image"]
        assert np.allclose(a, b, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("degree,model", [(1, 0), (3, 0), (3, 1)])
def test_sh_gradients_finite_differences(orc, degree, model):
    """dL/d(SH coefficients) and dL/dp (including the view-direction path, pinhole) against central
    differences of L = sum(image * dL/dimage) on a smooth raster."""
    p, rest = sh_scene(10, 6 + degree, degree)
    if model == 0:
        cam = synth.ring_cameras(1, 40, 32, 9)[0]
    else:
        Rm, tv = synth.look_at([0.3, -4.0, 0.5])
        cam = affine_cam(40, 32, fx=9.0, cx=20.0, cy=16.0, R=Rm.astype(np.float32), t=tuple(tv))
    dl = np.random.default_rng(1).normal(size=(3, 32, 40))
    r = orc.render(p, cam, SMOOTH, dl_dimage=dl, sh_rest=rest, sh_degree=degree)
    vis = np.flatnonzero(r["decision"]["visible"])
    assert len(vis) >= 3

    def loss(pp, rr):
        return (orc.render(pp, cam, SMOOTH, sh_rest=rr, sh_degree=degree)["image"] * dl).sum()

    h = 1e-6
    for i in vis[:3]:
        for k in (0, 1, 2, 11, 12, 13):
            a, b = p.copy(), p.copy()
            a[k, i] += h; b[k, i] -= h
            fd = (loss(a, rest) - loss(b, rest)) / (2 * h)
            assert np.isclose(r["grad"][k, i], fd, rtol=2e-5, atol=1e-8), (k, i)
        for k in range(rest.shape[0]):
            a, b = rest.copy(), rest.copy()
            a[k, i] += h; b[k, i] -= h
            fd = (loss(p, a) - loss(p, b)) / (2 * h)
            assert np.isclose(r["grad_sh"][k, i], fd, rtol=2e-5, atol=1e-8), (k, i)


# ---------------------------------------------------------------- GPU parity
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2505_05587_b200 import require_cuda
    require_cuda()


def _sh_cams(model):
    if model == 0:
        return synth.ring_cameras(3, 64, 64, 21)
    out = []
    for eye in ([0.3, -4.0, 0.5], [3.0, 2.0, 1.0], [-2.5, 2.5, -1.0]):
        Rm, tv = synth.look_at(eye)
        out.append(affine_cam(64, 64, fx=12.0, cx=32.0, cy=32.0, R=Rm.astype(np.float32), t=tuple(tv)))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("degree,model", [(0, 0), (1, 0), (2, 1), (3, 0), (3, 1)])
def test_sh_render_parity(orc, degree, model):
    """SH colours (f3): forward images and the backward (14 parameter planes, S, SH rest coefficients)
    of project_sh -> render -> sh_bwd -> gauss_bwd(| 4) against the oracle, 3 views of the C1 scene."""
    _gpu()
    from gpu_run import raster_of, to_dev
    from paper_2505_05587_b200.pipeline import Rasterizer
    p, rest = sh_scene(64, 30 + degree, degree)
    p = p.astype(np.float32).astype(np.float64)
    rest = rest.astype(np.float32).astype(np.float64)
    cams = _sh_cams(model)
    V, n = len(cams), p.shape[1]
    dl = synth.dl_dimage(V, 64, 64, 40)
    rz = Rasterizer(n, V, 64, 64, raster_of(SMOOTH))
    dp, drest = to_dev(p), to_dev(rest) if rest.size else torch.zeros(0, n, device="cuda")
    grad = torch.zeros(20, n, device="cuda")
    gsh = torch.full((max(rest.shape[0], 0), n), 9.0, device="cuda")
    rz.project(dp, n, cams, drest, degree)
    rz.bin_sort(); rz.render_fwd()
    rz.render_bwd_moments(dL=to_dev(dl))
    rz.sh_bwd(dp, grad, drest, degree, gsh, accumulate=0)
    rz.gauss_bwd(dp, grad, accumulate=0 | 4)
    torch.cuda.synchronize()
    img = rz.image.cpu().numpy()
    o = np.zeros((20, n)); a = np.zeros((20, n)); osh = np.zeros((rest.shape[0], n))
    for v, cam in enumerate(cams):
        r = orc.render(p, cam, SMOOTH, dl_dimage=dl[v], sh_rest=rest, sh_degree=degree)
        assert (np.abs(img[v] - r["image"]) <= 1e-4 * np.abs(r["image"]) + 1e-6).all()
        o += r["grad"]; a += r["absg"]
        if rest.shape[0]:
            osh += r["grad_sh"]
    g = grad.cpu().numpy().astype(np.float64)
    floor = 1e-6 * np.abs(o).max(axis=1, keepdims=True)
    ok = np.abs(g - o) <= 1e-3 * np.abs(o) + 1e-5 * a + floor + 1e-30
    assert ok.all(), [(k, float(np.abs(g[k] - o[k]).max())) for k in range(20) if not ok[k].all()]
    if rest.shape[0]:
        gs = gsh.cpu().numpy().astype(np.float64)
        tol = 2e-3 * np.abs(osh) + 1e-5 * np.abs(osh).max(axis=1, keepdims=True) + 1e-30
        assert (np.abs(gs - osh) <= tol).all(), float(np.abs(gs - osh).max())


@pytest.mark.gpu
def test_sh_training_loop_parity(orc):
    """Trainer with SH degree 3 (Adam on the rest coefficients, offspring inherit them) against
    oracle/train.py: counts bit-exact, parameters and SH coefficients within the f1 tolerance."""
    _gpu()
    from oracle.train import train
    from gpu_run import raster_of
    from paper_2505_05587_b200 import Adam, Schedule, Trainer
    LR = (1e-3, 5e-3, 1e-3, 5e-2, 2.5e-3)
    GROUP = np.array([0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 4, 4, 4])
    p, rest = sh_scene(64, 50, 3, dc_scale=0.8)
    p = p.astype(np.float32); rest = rest.astype(np.float32)
    cams = synth.ring_cameras(8, 64, 64, 7)
    tg = synth.target_images(8, 64, 64, 8)

    def b(t):
        idx = [(2 * t + k) % 8 for k in range(2)]
        return [cams[i] for i in idx], tg[idx]

    cap = 512
    ora = train(p, 64, cap, b, T=8, t_start=4, t_split=3, lr=LR, eps=1e-15, rp=SMOOTH, sh_degree=3, sh_rest0=rest,
                sh_lr=1e-3)
    for lam in ora["lambda_min"]:
        assert np.abs(lam + 1e-6).min() > 1e-4 * np.abs(lam).max()
    tr = Trainer(torch.from_numpy(p).cuda(), 64, cap, 2, 64, 64, raster_of(SMOOTH), Adam(LR, 0.9, 0.999, 1e-15),
                 Schedule(4, 3), sh_degree=3, sh_rest0=torch.from_numpy(rest).cuda(), sh_lr=1e-3)
    for t in range(1, 9):
        c, y = b(t)
        tr.step(c, torch.from_numpy(np.ascontiguousarray(y)).cuda())
    torch.cuda.synchronize()
    assert [h["n_split"] for h in tr.history] == ora["n_split"] and tr.n == ora["n"]
    got = tr.params[:, :tr.n].double().cpu().numpy()
    lr = np.asarray(LR)[GROUP][:, None]
    tol = 5e-3 * lr + 1e-6 * np.abs(ora["params"])
    tol[0:3] += ora["pos_sens"][None, :]          # per-Gaussian offspring bound (test_train.py)
    assert (np.abs(got - ora["params"]) <= tol).all()
    gs = tr.sh_rest[:, :tr.n].double().cpu().numpy()
    assert (np.abs(gs - ora["sh_rest"]) <= 5e-3 * 1e-3 + 1e-6 * np.abs(ora["sh_rest"])).all()
