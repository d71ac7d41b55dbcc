"""NEXT f3: the photometric loss with the SSIM term (P:L150 footnote) — oracle pins (-m "not gpu")
and GPU parity of the fused l1 + SSIM loss/gradient kernels."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")


def _imgs(seed, H=20, W=23):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, 1, size=(3, H, W))
    y = np.clip(x + 0.2 * rng.normal(size=x.shape), 0, 1)
    return x, y


def test_window_and_filter_match_library():
    """The 11x11 window is the normalised outer product of the sigma-1.5 Gaussian; the plain shifted-sum
    filter equals scipy's zero-padded correlation."""
    from scipy import ndimage
    from oracle.ssim import filt, window
    w = window()
    assert np.isclose(w.sum(), 1.0) and np.allclose(w, w.T) and np.allclose(w, w[::-1, ::-1])
    x, _ = _imgs(1)
    ref = np.stack([ndimage.correlate(x[c], w, mode="constant", cval=0.0) for c in range(3)])
    assert np.allclose(filt(x, w), ref, rtol=1e-13, atol=1e-14)


def test_ssim_identity_and_symmetry():
    from oracle.ssim import ssim, ssim_map
    x, y = _imgs(2)
    assert np.allclose(ssim_map(x, x)[0], 1.0, rtol=0, atol=1e-14)
    assert np.isclose(ssim(x, y), ssim(y, x), rtol=1e-14)
    assert ssim(x, y) < 0.99


def test_ssim_closed_form_for_a_brightness_shift():
    """x = y + c: away from the border (full window mass) sigma_x = sigma_y = sigma_xy, so the
    structure/contrast factor is 1 and S = (2 mu_y (mu_y + c) + C1) / (mu_y^2 + (mu_y + c)^2 + C1)."""
    from scipy import ndimage
    from oracle.ssim import C1, ssim_map, window
    _, y = _imgs(3, 24, 26)
    c = 0.07
    S = ssim_map(y + c, y)[0]
    for ch in range(3):
        mu = ndimage.correlate(y[ch], window(), mode="constant", cval=0.0)
        ref = (2 * mu * (mu + c) + C1) / (mu ** 2 + (mu + c) ** 2 + C1)
        assert np.allclose(S[ch, 5:-5, 5:-5], ref[5:-5, 5:-5], rtol=1e-12, atol=1e-13)


def test_loss_gradient_finite_differences():
    from oracle.ssim import loss_and_grad
    x, y = _imgs(4, 13, 11)
    L, g = loss_and_grad(x, y)
    rng = np.random.default_rng(0)
    h = 1e-6
    for _ in range(25):
        idx = tuple(rng.integers(0, s) for s in x.shape)
        if abs(x[idx] - y[idx]) < 1e-3:
            continue
        a, b = x.copy(), x.copy()
        a[idx] += h; b[idx] -= h
        fd = (loss_and_grad(a, y)[0] - loss_and_grad(b, y)[0]) / (2 * h)
        assert np.isclose(g[idx], fd, rtol=1e-5, atol=1e-10), idx


@pytest.mark.gpu
@pytest.mark.parametrize("V,H,W", [(1, 64, 64), (3, 45, 77), (2, 545, 980)])
def test_l1_ssim_parity(V, H, W):
    """Per-view loss and dL/dimage of the fused kernels against the oracle (ragged tiles included)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.ssim import loss_and_grad
    from paper_2505_05587_b200 import _lib
    x = synth.target_images(V, W, H, 91)
    y = synth.target_images(V, W, H, 92)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    dL = torch.zeros_like(dx)
    loss = torch.zeros(V, device="cuda")
    ws = torch.empty(_lib.loss_workspace_size(V, H, W), dtype=torch.uint8, device="cuda")
    _lib.l1_ssim_grad(dx, dy, 0.2, 1.0 / V, dL, loss, ws)
    torch.cuda.synchronize()
    g = dL.cpu().numpy().astype(np.float64)
    lo = loss.cpu().numpy()
    for v in range(V):
        Lo, go = loss_and_grad(x[v].astype(np.float64), y[v].astype(np.float64))
        assert np.isclose(lo[v], Lo, rtol=2e-5), (lo[v], Lo)
        go = go / V
        assert (np.abs(g[v] - go) <= 1e-3 * np.abs(go) + 1e-4 * np.abs(go).max()).all(), np.abs(g[v] - go).max()
