"""Pins for the CPU oracle against things other than itself:
SPEC/paper worked values, closed forms, textbook/library special cases, finite differences,
Lemma 1 and the paper's theorems.  CPU only."""
import math

import numpy as np
import pytest

import synth
from helpers import affine_cam, l1_loss_grad, params_from

SMOOTH = dict(alpha_min=0.0, alpha_max=1.0, t_min=0.0, dilation=0.0, bg=(0.0, 0.0, 0.0), tile=16)
SMOOTH_DIL = dict(SMOOTH, dilation=0.3)


def rand_rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def small_scene(seed, n=6, pinhole=False):
    rng = np.random.default_rng(seed)
    if pinhole:
        means = rng.uniform(-1.2, 1.2, size=(n, 3))
        scales = np.exp(np.log(0.35) + 0.3 * rng.normal(size=(n, 3)))
    else:
        means = np.concatenate([rng.uniform(-1.3, 1.3, size=(n, 2)), rng.uniform(-1, 1, size=(n, 1))], 1)
        scales = np.exp(np.log(0.3) + 0.3 * rng.normal(size=(n, 3)))
    quats = rng.normal(size=(n, 4))
    quats *= rng.uniform(0.8, 1.2, size=(n, 1)) / np.linalg.norm(quats, axis=1, keepdims=True)
    opac = rng.uniform(0.3, 0.9, size=n)
    rgb = rng.uniform(0, 1, size=(n, 3))
    p = params_from(means, scales, quats, opac, rgb)
    W, H = 24, 20
    if pinhole:
        cams = synth.ring_cameras(2, W, H, seed + 7, radius=5.0)
        for c in cams:
            c["fx"] = c["fy"] = np.float32(22.0)
    else:
        cams = []
        for v in range(2):
            R = rand_rot(np.random.default_rng(seed + 11 + v))
            # camera-space xy spans the means; R only makes P a general 2x3
            cams.append(affine_cam(W, H, fx=6.0, cx=12.0, cy=10.0, R=R))
        # re-centre world means so that the camera-space projection of the first view is in frame
    tg = np.random.default_rng(seed + 99).uniform(0, 1, size=(2, 3, H, W))
    return p, cams, tg


# ---------------------------------------------------------------------------------------------
# Projection: SPEC examples, textbook homogeneous projection.
# ---------------------------------------------------------------------------------------------
def test_affine_projection_spec_examples(orc):
    cam = affine_cam(8, 8)  # P = [I2 | 0], b = 0
    rp = dict(SMOOTH)
    p = params_from([[3, 4, 5], [0, 0, 0], [0, 0, 0]], [[1, 1, 1], [1, 1, 1], [1, 2, 3]])
    pr = orc.project(p, cam, rp)
    assert np.array_equal(pr["mu"][0], [3.0, 4.0])            # S:L50  (3,4,5) -> (3,4)
    assert np.allclose(pr["cov2d"][1], [1, 0, 1], atol=1e-15)  # S:L60  Sigma = I3 -> I2
    assert np.allclose(pr["cov2d"][2], [1, 0, 4], atol=1e-15)  # S:L61  diag(1,4,9) -> diag(1,4)


def test_sigma_spec_examples(orc):
    cam = affine_cam(8, 8)
    p = params_from([[2.0, 3.0, 1.0]], [[1, 1, 1]], opac=[0.7])
    o = 1 / (1 + math.exp(-float(p[10, 0])))
    assert orc.eval_sigma(p, 0, cam, 2.0, 3.0, SMOOTH) == pytest.approx(o, rel=1e-15)
    r = math.sqrt(2 * math.log(2))
    assert orc.eval_sigma(p, 0, cam, 2.0 + r, 3.0, SMOOTH) == pytest.approx(o / 2, rel=1e-14)
    p0 = params_from([[2.0, 3.0, 1.0]], [[1, 1, 1]], opac=[0.0])
    assert orc.eval_sigma(p0, 0, cam, 2.5, 3.0, SMOOTH) == 0.0


def test_pinhole_mean_matches_homogeneous_projection(orc):
    cam = synth.ring_cameras(1, 640, 480, 3)[0]
    rng = np.random.default_rng(0)
    p = params_from(rng.uniform(-1, 1, size=(50, 3)), [0.05, 0.05, 0.05])
    pr = orc.project(p, cam, synth_rp())
    K = np.array([[cam["fx"], 0, cam["cx"]], [0, cam["fy"], cam["cy"]], [0, 0, 1]], dtype=np.float64)
    Rt = np.concatenate([np.asarray(cam["R"], np.float64), np.asarray(cam["t"], np.float64)[:, None]], 1)
    X = np.concatenate([p[0:3].astype(np.float64), np.ones((1, 50))])
    h = K @ Rt @ X                                           # textbook x ~ K [R|t] X
    assert np.allclose(pr["mu"], (h[:2] / h[2]).T, rtol=1e-13, atol=1e-10)
    # conic is the inverse of the (dilated) projected covariance: Q Sigma2D = I
    cov, con = pr["cov2d"], pr["conic"]
    for i in range(50):
        S = np.array([[cov[i, 0], cov[i, 1]], [cov[i, 1], cov[i, 2]]])
        Q = np.array([[con[i, 0], con[i, 1]], [con[i, 1], con[i, 2]]])
        assert np.allclose(Q @ S, np.eye(2), atol=1e-12)


def synth_rp():
    return dict(alpha_min=1 / 255, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0, 0, 0), tile=16)


def test_decision_chain_conservative_and_consistent(orc):
    """Every pixel where the fp64 alpha >= alpha_min lies inside the fp32 rect (Z4)."""
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cam = synth.cameras_for(cfg)[0]
    rp = synth_rp()
    d = orc.decide(p, cam, rp)
    pr = orc.project(p, cam, rp)
    W, H = cam["width"], cam["height"]
    ys, xs = np.mgrid[0:H, 0:W]
    for i in np.flatnonzero(d["visible"]):
        dx, dy = xs + 0.5 - pr["mu"][i, 0], ys + 0.5 - pr["mu"][i, 1]
        c = pr["conic"][i]
        m = c[0] * dx * dx + 2 * c[1] * dx * dy + c[2] * dy * dy
        alpha = np.minimum(0.99, pr["opacity"][i] * np.exp(-0.5 * m))
        k, j = np.nonzero(alpha >= rp["alpha_min"])
        r = d["rect"][i]
        assert (j >= r[0]).all() and (j <= r[1]).all() and (k >= r[2]).all() and (k <= r[3]).all()
        T = rp["tile"]
        assert d["tiles_touched"][i] == (r[1] // T - r[0] // T + 1) * (r[3] // T - r[2] // T + 1)
    # invisible ones never reach alpha_min anywhere in the image
    for i in np.flatnonzero(d["visible"] == 0)[:20]:
        dx, dy = xs + 0.5 - pr["mu"][i, 0], ys + 0.5 - pr["mu"][i, 1]
        c = pr["conic"][i]
        m = c[0] * dx * dx + 2 * c[1] * dx * dy + c[2] * dy * dy
        assert (pr["opacity"][i] * np.exp(-0.5 * m) < rp["alpha_min"] * (1 + 1e-4)).all()


# ---------------------------------------------------------------------------------------------
# Compositing: SPEC examples, invariants, brute force == AABB scatter.
# ---------------------------------------------------------------------------------------------
def test_composite_spec_examples(orc):
    cam = affine_cam(16, 16)
    rgb = np.float32([0.2, 0.5, 0.9]).astype(np.float64)  # stored as fp32
    one = params_from([[10.5, 7.5, 1.0]], [[1, 1, 1]], opac=[1.0], rgb=[rgb])
    r = orc.render(one, cam, SMOOTH)
    assert np.array_equal(r["image"][:, 7, 10], rgb)               # pixel = c exactly
    r = orc.render(one, cam, dict(SMOOTH, alpha_max=0.99))
    assert np.allclose(r["image"][:, 7, 10], 0.99 * np.array(rgb), rtol=1e-15)
    two = params_from([[10.5, 7.5, 1.0], [10.5, 7.5, 1.0]], [[1, 1, 1]] * 2, opac=[0.5, 0.5], rgb=[rgb, rgb])
    r = orc.render(two, cam, SMOOTH)
    assert np.allclose(r["image"][:, 7, 10], 0.75 * np.array(rgb), rtol=1e-15)


# ---------------------------------------------------------------------------------------------
# Depth order.  P:L129 "sorts points according to view-dependent depth" and Eq. eqn:alpha_blend
# (P:L131-134): C = sum_i c_i alpha_i T_i with T_i = prod_{j<i} (1 - alpha_j), so the Gaussian
# with T_1 = 1 is the one nearest the camera (smallest camera-space z).  Two Gaussians on one pixel
# ray, o = 0.5 each, smooth mode (alpha = sigma = 0.5 at the mean): the pixel must be
# 0.5 c_near + 0.25 c_far whichever index the near one has; a back-to-front reading would give
# 0.5 c_far + 0.25 c_near.
# ---------------------------------------------------------------------------------------------
RED, BLUE = np.array([1.0, 0.0, 0.0]), np.array([0.0, 0.0, 1.0])


@pytest.mark.parametrize("near_first", [True, False])
@pytest.mark.parametrize("z_near,z_far", [(1.0, 2.0), (-0.5, 0.25), (-3.0, -1.0)])
def test_occlusion_nearer_gaussian_composites_first_affine(orc, near_first, z_near, z_far):
    cam = affine_cam(16, 16)                              # P = [I2 | 0]: camera z = world z
    means = [[10.5, 7.5, z_near], [10.5, 7.5, z_far]]
    rgb = [RED, BLUE]
    if not near_first:                                    # the near one gets the larger index
        means, rgb = means[::-1], rgb[::-1]
    p = params_from(means, [[1, 1, 1]] * 2, opac=[0.5, 0.5], rgb=rgb)
    r = orc.render(p, cam, SMOOTH)
    assert np.allclose(r["image"][:, 7, 10], 0.5 * RED + 0.25 * BLUE, rtol=0, atol=1e-15)
    assert r["final_T"][7, 10] == pytest.approx(0.25, abs=1e-15)


def test_occlusion_nearer_gaussian_composites_first_pinhole(orc):
    # camera at the origin looking down +z (R = I, t = 0): the optical axis hits pixel (8, 8) centre
    cam = dict(affine_cam(16, 16, fx=10.0, cx=8.5, cy=8.5), model=0)
    for near_first in (True, False):
        means = [[0.0, 0.0, 2.0], [0.0, 0.0, 5.0]]
        rgb = [RED, BLUE]
        sc = [[0.2, 0.2, 0.2], [0.5, 0.5, 0.5]]           # same projected footprint (s / z)
        if not near_first:
            means, rgb, sc = means[::-1], rgb[::-1], sc[::-1]
        p = params_from(means, sc, opac=[0.5, 0.5], rgb=rgb)
        r = orc.render(p, cam, SMOOTH)
        assert np.allclose(r["image"][:, 8, 8], 0.5 * RED + 0.25 * BLUE, rtol=0, atol=1e-15), near_first


def test_depth_key_monotone_across_zero_affine(orc):
    """C7: key = orderable-uint32(z_fp32) must increase strictly with z over negative, zero and positive
    depths (affine camera: no near-plane cull), so ascending-key order is near-to-far."""
    z = np.array([-1e6, -37.0, -1.0, -0.5, -1e-3, -1e-30, 0.0, 1e-30, 1e-3, 0.25, 1.0, 2.0, 1e6])
    cam = affine_cam(16, 16)
    p = params_from(np.stack([np.full_like(z, 8.0), np.full_like(z, 8.0), z], 1), [[1, 1, 1]] * z.size)
    d = orc.decide(p, cam, SMOOTH)
    assert d["visible"].all()
    k = d["key"].astype(np.int64)
    assert (np.diff(k) > 0).all(), k
    # shuffled indices: the oracle's render order (ascending key) is the z order
    perm = np.random.default_rng(1).permutation(z.size)
    dk = orc.decide(p[:, perm], cam, SMOOTH)["key"]
    assert np.array_equal(np.argsort(dk, kind="stable"), np.argsort(z[perm], kind="stable"))


def test_depth_order_of_a_front_layer_hides_the_back(orc):
    """Many Gaussians: an opaque-ish layer (alpha_max clamp) in front of a second layer leaves the
    pixel at the front colour up to T_min early termination — the back layer's colour must not show.
    Checked pixel by pixel against the closed form of Eq. eqn:alpha_blend for a uniform front stack."""
    cam = affine_cam(16, 16)
    rp = dict(SMOOTH, alpha_max=0.99, t_min=1e-3)
    k = 3                                                 # three front Gaussians at the pixel centre
    means = [[8.5, 8.5, 1.0 + 0.1 * j] for j in range(k)] + [[8.5, 8.5, 5.0]]
    rgb = [RED] * k + [BLUE]
    order = [3, 0, 2, 1]                                  # indices unrelated to depth
    p = params_from([means[i] for i in order], [[1, 1, 1]] * 4, opac=[0.999999] * 4, rgb=[rgb[i] for i in order])
    r = orc.render(p, cam, rp)
    # first front Gaussian: alpha = alpha_max, T -> 1 - alpha_max ~ 0.01; the second would leave
    # T (1 - alpha) ~ 1e-4 < t_min: terminate.  Only the nearest one is composited; blue never is.
    amax = float(np.float32(0.99))
    assert np.allclose(r["image"][:, 8, 8], amax * RED, rtol=0, atol=1e-15)
    assert r["n_comp"][8, 8] >= 1
    assert r["image"][2, 8, 8] == 0.0


def test_bruteforce_equals_aabb_and_range(orc):
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    for model in (0, 1):
        cam = synth.cameras_for(cfg, model=model)[0]
        dl = synth.dl_dimage(1, cam["width"], cam["height"], 4)[0]
        a = orc.render(p, cam, synth_rp(), dl_dimage=dl)
        b = orc.render(p, cam, synth_rp(), dl_dimage=dl, brute_force=True)
        assert a["pairs"] == b["pairs"] > 0
        for k in ("image", "final_T", "n_comp"):
            assert np.array_equal(a[k], b[k])
        assert np.allclose(a["grad"], b["grad"], rtol=1e-12, atol=1e-18)
        assert a["image"].min() >= 0 and a["image"].max() <= 1      # S:L146 convexity


def test_permutation_invariance(orc):
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cam = synth.cameras_for(cfg)[0]
    perm = np.random.default_rng(5).permutation(p.shape[1])
    a = orc.render(p, cam, synth_rp())
    b = orc.render(p[:, perm], cam, synth_rp())
    assert np.array_equal(a["image"], b["image"])


# ---------------------------------------------------------------------------------------------
# Gradients: central finite differences of the whole l1 loss, smooth mode.
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("pinhole,rp", [(False, SMOOTH), (False, SMOOTH_DIL), (True, SMOOTH_DIL)])
def test_gradients_match_finite_differences(orc, pinhole, rp):
    p, cams, tg = small_scene(3 if pinhole else 4, pinhole=pinhole)
    p64 = p.astype(np.float64)
    _, an = l1_loss_grad(orc, p64, cams, tg, rp)
    fd = np.zeros((14, p.shape[1]))
    for k in range(14):
        for i in range(p.shape[1]):
            h = 1e-6 * max(1.0, abs(p64[k, i]))
            pp, pm = p64.copy(), p64.copy()
            pp[k, i] += h
            pm[k, i] -= h
            fd[k, i] = (l1_loss_grad(orc, pp, cams, tg, rp, False)[0] - l1_loss_grad(orc, pm, cams, tg, rp, False)[0]) / (2 * h)
    scale = np.abs(an[:14]).max()
    err = np.abs(fd - an[:14])
    assert (err <= 2e-5 * np.abs(an[:14]) + 2e-7 * scale).all(), (err / (np.abs(an[:14]) + 1e-12)).max()


# ---------------------------------------------------------------------------------------------
# Position Hessian of sigma (App. C.4) and the Lemma-1 pin for S.
# ---------------------------------------------------------------------------------------------
def test_position_hessian_spec_examples(orc):
    cam = affine_cam(8, 8)
    p = params_from([[2.0, 3.0, 1.0]], [[1, 1, 1]], opac=[1.0])
    H = orc.position_hessian(p, 0, cam, 2.0, 3.0, SMOOTH)
    assert np.array_equal(H, -np.diag([1.0, 1.0, 0.0]))
    p0 = params_from([[2.0, 3.0, 1.0]], [[1, 1, 1]], opac=[0.0])
    assert np.array_equal(orc.position_hessian(p0, 0, cam, 2.7, 3.1, SMOOTH), np.zeros((3, 3)))


def test_position_hessian_matches_finite_differences(orc):
    rng = np.random.default_rng(7)
    for trial in range(20):
        R = rand_rot(rng)
        cam = affine_cam(32, 32, fx=rng.uniform(2, 8), fy=rng.uniform(2, 8), cx=16, cy=16, R=R)
        p = params_from(rng.uniform(-1, 1, size=(1, 3)), np.exp(rng.normal(np.log(0.5), 0.3, size=(1, 3))),
                        rng.normal(size=(1, 4)), [rng.uniform(0.2, 0.9)])
        mu = orc.project(p, cam, SMOOTH)["mu"][0]
        x, y = mu + rng.normal(scale=2.0, size=2)
        H = orc.position_hessian(p, 0, cam, x, y, SMOOTH)
        p64 = p.astype(np.float64)
        h = 1e-4
        fd = np.zeros((3, 3))
        for a in range(3):
            for b in range(3):
                vals = []
                for sa, sb in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
                    q = p64.copy()
                    q[a, 0] += sa * h
                    q[b, 0] += sb * h
                    vals.append(orc.eval_sigma(q, 0, cam, x, y, SMOOTH))
                fd[a, b] = (vals[0] - vals[1] - vals[2] + vals[3]) / (4 * h * h)
        assert np.linalg.norm(fd - H) <= 1e-5 * np.linalg.norm(H) + 1e-12, trial


def test_lemma1_splitting_matrix_equals_loss_hessian(orc):
    """l1 + smooth compositing + affine camera: C is affine in each sigma_i and l1 is piecewise
    linear, so T_i = 0 in Lemma 1 and S_i equals the exact position Hessian of L."""
    p, cams, tg = small_scene(11, n=5)
    p64 = p.astype(np.float64)
    _, acc = l1_loss_grad(orc, p64, cams, tg, SMOOTH_DIL)
    checked = 0
    for i in range(p.shape[1]):
        S = np.array([[acc[14, i], acc[15, i], acc[16, i]], [acc[15, i], acc[17, i], acc[18, i]],
                      [acc[16, i], acc[18, i], acc[19, i]]])
        Hfd = np.zeros((3, 3))
        for b in range(3):
            h = 1e-5
            pp, pm = p64.copy(), p64.copy()
            pp[b, i] += h
            pm[b, i] -= h
            gp = l1_loss_grad(orc, pp, cams, tg, SMOOTH_DIL)[1]
            gm = l1_loss_grad(orc, pm, cams, tg, SMOOTH_DIL)[1]
            Hfd[:, b] = (gp[0:3, i] - gm[0:3, i]) / (2 * h)
        Hfd = 0.5 * (Hfd + Hfd.T)
        if np.linalg.norm(S) < 1e-9:
            continue
        assert np.linalg.norm(S - Hfd) <= 1e-5 * np.linalg.norm(S), (i, S, Hfd)
        checked += 1
    assert checked >= 3


def test_splitting_matrix_zero_residual(orc):
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cam = synth.cameras_for(cfg)[0]
    r = orc.render(p, cam, synth_rp(), dl_dimage=np.zeros((3, 64, 64)))
    assert np.array_equal(r["grad"], np.zeros_like(r["grad"]))


# ---------------------------------------------------------------------------------------------
# Eigen (App. A.3) against LAPACK and identities.
# ---------------------------------------------------------------------------------------------
def test_eigen_spec_examples(orc):
    lam, V = orc.eig_sym3(np.diag([3.0, 2.0, 1.0]))
    assert np.array_equal(lam, [1, 2, 3]) and np.array_equal(V[:, 0], [0, 0, 1])
    lam, V = orc.eig_sym3(np.eye(3))
    assert np.array_equal(lam, [1, 1, 1]) and np.array_equal(V, np.eye(3))
    lam, V = orc.eig_sym3(np.diag([1.0, 2.0, 3.0]))
    assert lam[0] == 1 and np.array_equal(V[:, 0], [1, 0, 0])
    lam, V = orc.eig_sym3(-np.eye(3))
    assert lam[0] == -1 and np.array_equal(V[:, 0], [1, 0, 0])


def test_eigen_random_against_lapack(orc):
    rng = np.random.default_rng(1)
    for _ in range(1000):
        A = rng.normal(size=(3, 3)) * 10 ** rng.uniform(-4, 2)
        A = 0.5 * (A + A.T)
        lam, V = orc.eig_sym3(A)
        ref = np.linalg.eigvalsh(A)
        nf = np.linalg.norm(A)
        assert np.allclose(lam, ref, rtol=0, atol=1e-12 * (1 + nf))
        assert np.linalg.norm(A @ V - V * lam) <= 1e-10 * (1 + nf)
        assert abs(lam.sum() - np.trace(A)) <= 1e-12 * (1 + nf)
        assert abs(np.prod(lam) - np.linalg.det(A)) <= 1e-10 * (1 + nf) ** 3
        assert np.allclose(V.T @ V, np.eye(3), atol=1e-12)
        big = np.argmax(np.abs(V[:, 0]))
        assert V[big, 0] > 0


# ---------------------------------------------------------------------------------------------
# Split rule and offspring (Thm 2; Alg.1)
# ---------------------------------------------------------------------------------------------
def _acc_from_S(mats, n, cap):
    acc = np.zeros((20, cap))
    for i, A in enumerate(mats):
        acc[14:20, i] = [A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]]
    return acc


def test_split_rule_spec_examples(orc):
    mats = [np.eye(3), np.diag([-1.0, 2.0, 3.0]), np.diag([-1e-7, 2.0, 3.0])]
    p = params_from(np.zeros((3, 3)), [0.1, 0.1, 0.1], opac=[0.8, 0.8, 0.8])
    pp = np.zeros((14, 8), np.float32)
    pp[:, :3] = p
    r = orc.densify(pp, _acc_from_S(mats, 3, 8), 3, 8, eta=-1.0, eps_abs=0.1)
    assert list(r["mask"]) == [0, 1, 0]
    assert r["lambda_min"][1] == -1.0
    assert r["n_split"] == 1 and list(r["dest"]) == [-1, 3, -1]
    # offspring: children at (+-0.1, 0, 0) with opacity 0.4 each
    o = 1 / (1 + np.exp(-r["params"][10, [1, 3]]))
    assert np.allclose(o, [0.4, 0.4], rtol=1e-15)
    assert np.allclose(r["params"][0:3, 1], [0.1, 0, 0], atol=1e-15)
    assert np.allclose(r["params"][0:3, 3], [-0.1, 0, 0], atol=1e-15)
    assert np.array_equal(r["params"][3:10, 3], r["params"][3:10, 1])   # Z14: covariance copied
    assert np.array_equal(r["params"][11:14, 3], r["params"][11:14, 1])
    assert np.array_equal(r["acc"][14:20, :4], np.zeros((6, 4)))       # Z23


def test_offspring_invariants(orc):
    rng = np.random.default_rng(2)
    n, cap = 10, 24
    p = np.zeros((14, cap), np.float32)
    p[:, :n] = synth.blob_scene(n, 5)
    mats = []
    for i in range(n):
        A = rng.normal(size=(3, 3)); A = A + A.T
        A += (0.0 if i % 3 == 0 else 10.0) * np.eye(3)   # 4 indefinite (i = 0, 3, 6, 9)
        mats.append(A)
    r = orc.densify(p, _acc_from_S(mats, n, cap), n, cap, eta=0.5)
    assert r["n_split"] == 4 and list(np.flatnonzero(r["mask"])) == [0, 3, 6, 9]
    assert list(r["dest"][r["mask"] == 1]) == [10, 11, 12, 13]
    o_par = 1 / (1 + np.exp(-p[10, :n].astype(np.float64)))
    o_new = 1 / (1 + np.exp(-r["params"][10, :n + 4]))
    assert abs(o_new.sum() - o_par.sum()) <= 1e-12                   # S:L387 opacity conservation
    for i, b in zip([0, 3, 6, 9], [10, 11, 12, 13]):
        mid = 0.5 * (r["params"][0:3, i] + r["params"][0:3, b])
        assert np.allclose(mid, p[0:3, i], atol=1e-15)               # mean(offspring) = parent
    keep = r["mask"] == 0
    assert np.array_equal(r["params"][:, :n][:, keep], p[:, :n][:, keep].astype(np.float64))
    # capacity: n + n_split > capacity -> error, params untouched (C16)
    r2 = orc.densify(p, _acc_from_S(mats, n, cap), n, 12, eta=0.5)
    assert r2["n_split"] == -1 and np.array_equal(r2["params"], p.astype(np.float64))


def test_theorem2_optimality_and_psd_no_gain(orc):
    """Delta = 1/2 sum_j w_j d_j^T S d_j >= lambda_min/2 over admissible splits;
    PSD S -> every sampled Delta >= 0 and no split."""
    rng = np.random.default_rng(3)
    for trial in range(50):
        A = rng.normal(size=(3, 3)); A = A + A.T
        if trial % 2:
            A += (abs(np.linalg.eigvalsh(A)[0]) + 0.1) * np.eye(3)
        lam, V = orc.eig_sym3(A)
        m = rng.integers(2, 5, size=2000)
        best = np.inf
        for mm in (2, 3, 4):
            sel = m == mm
            k = int(sel.sum())
            w = rng.dirichlet(np.ones(mm), size=k)
            d = rng.normal(size=(k, mm, 3))
            d /= np.maximum(1.0, np.linalg.norm(d, axis=2, keepdims=True))
            delta = 0.5 * np.einsum("kj,kja,ab,kjb->k", w, d, A, d)
            best = min(best, delta.min())
        sdc = 0.5 * V[:, 0] @ A @ V[:, 0]
        assert abs(sdc - lam[0] / 2) <= 1e-12 * (1 + np.abs(A).max())
        if lam[0] < 0:
            assert sdc <= best + 1e-12          # Thm 2 part 2: the SDC split attains the bound
        else:
            assert best >= -1e-12               # Thm 2 part 1: no split can decrease the loss


def test_theorem1_merged_slot_second_order(orc):
    """Merged-slot split of Gaussian i at +-eps v_min, w = 1/2 (mu = 0):
    (L(eps) - L) / eps^2 -> lambda_min(S_i)/2 with an O(eps^2) remainder (odd orders cancel)."""
    p, cams, tg = small_scene(21, n=5)
    p64 = p.astype(np.float64)
    L0, acc = l1_loss_grad(orc, p64, cams, tg, SMOOTH_DIL)
    i = int(np.argmin([orc.eig_sym3(acc[14:20, j])[0][0] for j in range(p.shape[1])]))
    lam, V = orc.eig_sym3(acc[14:20, i])
    assert lam[0] < 0
    v = V[:, 0]
    errs = []
    for eps in (0.1, 0.05, 0.025, 0.0125):
        L = 0.0
        for cam, t in zip(cams, tg):
            r = orc.render(p64, cam, SMOOTH_DIL, split=dict(index=i, w=[0.5, 0.5], delta=[eps * v, -eps * v]))
            L += np.abs(r["image"] - t).mean()
        errs.append((L - L0) / eps ** 2 - lam[0] / 2)
    ratios = [errs[k] / errs[k + 1] for k in range(3)]
    assert all(2.5 <= r <= 5.5 for r in ratios), (errs, ratios)
    assert abs(errs[-1]) < 0.05 * abs(lam[0] / 2)


def test_budget_and_gate_variants_spec_examples(orc):
    """App. A.2: increment budget keeps the least lambda_min (lambda = (-3,-1,-2), K = 2
    keeps -3 and -2; K = 0 keeps none), ties by index; the compactest gate also requires a small
    accumulated position gradient."""
    mats = [np.diag([-3.0, 1, 2]), np.diag([-1.0, 1, 2]), np.diag([-2.0, 1, 2]), np.eye(3)]
    p = np.zeros((14, 16))
    p[:, :4] = params_from(np.zeros((4, 3)), [0.1, 0.1, 0.1])
    r = orc.densify(p, _acc_from_S(mats, 4, 16), 4, 16, budget=2)
    assert list(r["mask"]) == [1, 0, 1, 0] and list(r["dest"]) == [4, -1, 5, -1]
    r = orc.densify(p, _acc_from_S(mats, 4, 16), 4, 16, budget=0)
    assert list(r["mask"]) == [0, 0, 0, 0] and r["n_split"] == 0
    r = orc.densify(p, _acc_from_S(mats, 4, 16), 4, 16, budget=5)
    assert list(r["mask"]) == [1, 1, 1, 0]
    ties = [np.diag([-1.0, 1, 2])] * 5
    r = orc.densify(p, _acc_from_S(ties, 5, 16), 5, 16, budget=3)
    assert list(r["mask"]) == [1, 1, 1, 0, 0]
    acc = _acc_from_S(mats, 4, 16)
    acc[0:3, 0] = [3.0, 0.0, 4.0]          # |G| = 5
    acc[0:3, 2] = [0.1, 0.0, 0.0]          # |G| = 0.1
    r = orc.densify(p, acc, 4, 16, eps_grad=1.0)
    assert list(r["mask"]) == [0, 1, 1, 0]
    acc10 = acc.copy()
    acc10[14:20] *= 10.0                    # same S_bar with denom = 10; |G / denom| = 0.5 for index 0
    r = orc.densify(p, acc10, 4, 16, eps_grad=1.0, denom=10.0)
    assert list(r["mask"]) == [1, 1, 1, 0]
    # gate 2 (C24): planes 0, 1 = (sum of view-gradient norms, visible views); split iff mean >= eps
    acc2 = _acc_from_S(mats, 4, 16)
    acc2[0:2, 0] = [0.3, 2.0]               # mean 0.15
    acc2[0:2, 1] = [1.0, 0.0]               # never visible
    acc2[0:2, 2] = [0.1, 4.0]               # mean 0.025
    r = orc.densify(p, acc2, 4, 16, grad_gate=0.1)
    assert list(r["mask"]) == [1, 0, 0, 0] and list(r["dest"]) == [4, -1, -1, -1]
