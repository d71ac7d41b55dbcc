"""3DGS Adaptive Density Control (the paper's baseline) on fp64 planes.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Readings (C22):
  * the statistic E[||grad_{Pi(p)} L||_2] is the mean over the views in which the Gaussian
    is visible (passes the decision chain) of the per-view 2D-mean gradient norm, in pixel units;
  * ||Sigma||_2 is the spectral norm of the covariance, max_k s_k^2;
  * clone ("p_j - p proportional to grad_p L"): the parent stays, its copy is displaced
    by -clone_step * G / denom (G = the window's accumulated position gradient);
  * split: both offspring at p + R(q) diag(s) z_j with the caller's z_j ~ N(0, I) and
    Sigma_j = 0.64 Sigma (log-scale + ln 0.8); opacity unchanged (w = 1);
  * layout as SDC: offspring A in the parent's slot, B appended at n + rank (rank over selected
    Gaussians in index order).
"""
from __future__ import annotations

import numpy as np


def quat_to_rot(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def view_grad_statistic(grad_mu_per_view, visible_per_view):
    """(sum over visible views of ||dL/dPi(p)||, number of visible views) from per-view [2][n] grads."""
    s = 0.0
    c = 0.0
    for gm, vis in zip(grad_mu_per_view, visible_per_view):
        v = np.asarray(vis) != 0
        s = s + np.where(v, np.hypot(gm[0], gm[1]), 0.0)
        c = c + v.astype(np.float64)
    return s, c


def adc_densify(params, G, stat_sum, stat_cnt, n, capacity, eps_adc, tau_adc, clone_step, scale_factor, denom,
                normals):
    """params [14][>=n], G [3][>=n] accumulated position gradient, stat_sum/stat_cnt [>=n],
    normals [6][>=n] (z_0 = rows 0-2, z_1 = rows 3-5).  Returns dict(params [14][n + n_new], kind [n]
    (0 keep, 1 clone, 2 split), dest [n], n_new); n_new = -1 (nothing applied) if over capacity."""
    P = np.array(params, dtype=np.float64)[:, :n]
    kind = np.zeros(n, np.uint8)
    for i in range(n):
        g = stat_sum[i] / stat_cnt[i] if stat_cnt[i] > 0 else 0.0       # E[||grad_Pi(p) L||]
        if g >= eps_adc:
            sigma_norm = np.exp(2.0 * P[3:6, i]).max()                      # ||Sigma||_2 = max s_k^2
            kind[i] = 1 if sigma_norm <= tau_adc else 2
    sel = np.flatnonzero(kind)
    dest = np.full(n, -1, np.int64)
    dest[sel] = n + np.arange(len(sel))
    if n + len(sel) > capacity:
        return dict(params=P, kind=kind, dest=dest, n_new=-1)
    out = np.zeros((14, n + len(sel)))
    out[:, :n] = P
    for i in sel:
        b = dest[i]
        out[:, b] = P[:, i]
        if kind[i] == 1:
            out[0:3, b] = P[0:3, i] - clone_step * np.asarray(G[:, i], dtype=np.float64) / denom
        else:
            R = quat_to_rot(P[6:10, i])
            s = np.exp(P[3:6, i])
            for slot, z in ((i, normals[0:3, i]), (b, normals[3:6, i])):
                out[0:3, slot] = P[0:3, i] + R @ (s * np.asarray(z, dtype=np.float64))
                out[3:6, slot] = P[3:6, i] + np.log(scale_factor)
    return dict(params=out, kind=kind, dest=dest, n_new=len(sel))
