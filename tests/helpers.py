"""Small test helpers: explicit scenes/cameras and oracle-only loss evaluation (no product code)."""
from __future__ import annotations

import numpy as np


def params_from(means, scales, quats=None, opac=None, rgb=None) -> np.ndarray:
    means = np.atleast_2d(np.asarray(means, dtype=np.float64))
    n = means.shape[0]
    scales = np.broadcast_to(np.asarray(scales, dtype=np.float64), (n, 3))
    quats = np.tile([1.0, 0, 0, 0], (n, 1)) if quats is None else np.broadcast_to(np.asarray(quats, dtype=np.float64), (n, 4))
    opac = np.full(n, 0.5) if opac is None else np.broadcast_to(np.asarray(opac, dtype=np.float64), (n,))
    rgb = np.full((n, 3), 0.5) if rgb is None else np.broadcast_to(np.asarray(rgb, dtype=np.float64), (n, 3))
    p = np.empty((14, n))
    p[0:3] = means.T
    p[3:6] = np.log(scales).T
    p[6:10] = quats.T
    with np.errstate(divide="ignore"):
        p[10] = np.log(opac) - np.log1p(-opac)
    p[11:14] = rgb.T
    return p.astype(np.float32)


def affine_cam(width, height, fx=1.0, fy=None, cx=0.0, cy=0.0, R=None, t=(0.0, 0.0, 0.0)):
    R = np.eye(3) if R is None else np.asarray(R)
    return dict(R=np.asarray(R, np.float32), t=np.asarray(t, np.float32), fx=np.float32(fx),
                fy=np.float32(fx if fy is None else fy), cx=np.float32(cx), cy=np.float32(cy), width=int(width),
                height=int(height), model=1, znear=np.float32(0.2), guard=np.float32(1.3))


def l1_loss_grad(orc, params, cams, targets, rp, want_grad=True):
    """Sum over views of mean-over-3HW |C - target| (Z8) and, optionally, its oracle
    gradient planes [20][n] (14 grads + S)."""
    p64 = np.asarray(params, dtype=np.float64)
    n = p64.shape[1]
    L = 0.0
    acc = np.zeros((20, n))
    for cam, tgt in zip(cams, targets):
        r = orc.render(p64, cam, rp)
        res = r["image"] - np.asarray(tgt, np.float64)
        L += np.abs(res).mean()
        if want_grad:
            dl = np.sign(res) / res.size
            rb = orc.render(p64, cam, rp, dl_dimage=dl)
            acc += rb["grad"]
    return L, acc
