"""The 3DGS photometric loss with the SSIM term (NEXT f3; P:L150 footnote "we ignore the SSIM term
for simplicity" — the training objective 3DGS actually uses).  TEST INFRASTRUCTURE ONLY.

Readings (C23):
  L_view = (1 - lam) mean |C - C_hat| + lam (1 - SSIM(C, C_hat)),  lam = 0.2,
  SSIM = mean over channels and pixels of the SSIM map with an 11 x 11 Gaussian window (sigma 1.5,
  normalised), zero padding outside the image ("same" filtering), C1 = 0.01^2, C2 = 0.03^2:
    mu_x = w * x, sigma_x^2 = w * x^2 - mu_x^2, sigma_xy = w * (x y) - mu_x mu_y,
    S = (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2)).
  The gradient is the chain rule written out: with the per-pixel partials G1 = dS/dmu_x,
  G11 = dS/d(w * x^2), G12 = dS/d(w * x y) (the window is symmetric, so the adjoint of the
  filter is the same zero-padded filter):
    dSSIM/dx_p = (1/N) [ (w * G1)(p) + 2 x_p (w * G11)(p) + y_p (w * G12)(p) ].
The filter is the plain definition: a sum over the 121 window offsets of shifted, zero-padded
copies (no separable pass, no FFT).
"""
from __future__ import annotations

import numpy as np

C1 = 0.01 ** 2
C2 = 0.03 ** 2


def window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    t = np.arange(size) - size // 2
    g = np.exp(-(t * t) / (2.0 * sigma * sigma))
    g /= g.sum()
    return np.outer(g, g)


def filt(img: np.ndarray, w: np.ndarray) -> np.ndarray:
    """(w * img)(p) = sum_{a,b} w[a, b] img[p + (a - r, b - r)], zero outside the image; img [..., H, W]."""
    r = w.shape[0] // 2
    H, W = img.shape[-2:]
    pad = np.zeros(img.shape[:-2] + (H + 2 * r, W + 2 * r))
    pad[..., r:r + H, r:r + W] = img
    out = np.zeros(img.shape, dtype=np.float64)
    for a in range(w.shape[0]):
        for b in range(w.shape[1]):
            out += w[a, b] * pad[..., a:a + H, b:b + W]
    return out


def ssim_map(x, y, w=None):
    w = window() if w is None else w
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64)
    mx, my = filt(x, w), filt(y, w)
    exx, eyy, exy = filt(x * x, w), filt(y * y, w), filt(x * y, w)
    sxx, syy, sxy = exx - mx * mx, eyy - my * my, exy - mx * my
    an, bn = 2 * mx * my + C1, 2 * sxy + C2
    ad, bd = mx * mx + my * my + C1, sxx + syy + C2
    S = an * bn / (ad * bd)
    return S, dict(mx=mx, my=my, an=an, bn=bn, ad=ad, bd=bd)


def ssim(x, y):
    return float(ssim_map(x, y)[0].mean())


def ssim_grad(x, y):
    """dSSIM/dx for SSIM = mean of the map over [3][H][W]."""
    w = window()
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64)
    S, q = ssim_map(x, y, w)
    D = q["ad"] * q["bd"]
    G1 = (2 * q["my"] * q["bn"] - 2 * q["my"] * q["an"]) / D - S * (2 * q["mx"] / q["ad"] - 2 * q["mx"] / q["bd"])
    G11 = -S / q["bd"]
    G12 = 2 * q["an"] / D
    N = x.size
    return (filt(G1, w) + 2 * x * filt(G11, w) + y * filt(G12, w)) / N


def loss_and_grad(image, target, lam: float = 0.2):
    """One view: (loss, dL/dimage) for L = (1 - lam) mean|C - C_hat| + lam (1 - SSIM)."""
    x = np.asarray(image, dtype=np.float64); y = np.asarray(target, dtype=np.float64)
    N = x.size
    l1 = np.abs(x - y).sum() / N
    loss = (1 - lam) * l1 + lam * (1 - ssim(x, y))
    g = (1 - lam) * np.sign(x - y) / N - lam * ssim_grad(x, y)
    return loss, g
