"""ctypes front-end to liboracle.so — the SteepGS CPU ORACLE.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package.  It is independent of the CUDA product: it includes/links nothing from
paper_2505_05587_b200/ or include/, and the product never imports it.

Every array crossing into C is float64 (the fp32 inputs from `synth` widen exactly).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

DEFAULT_RASTER = dict(alpha_min=1.0 / 255.0, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), tile=16)
SMOOTH_RASTER = dict(alpha_min=0.0, alpha_max=1.0, t_min=0.0, dilation=0.0, bg=(0.0, 0.0, 0.0), tile=16)


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C11 + OpenMP, -ffp-contract=off so the fp32 decision chain is
    evaluated operation by operation)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", "-o", _SO, src, "-lm"])
    return _SO


class Camera(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("model", C.c_int32), ("znear", C.c_double), ("guard", C.c_double)]


class Raster(C.Structure):
    _fields_ = [("alpha_min", C.c_double), ("alpha_max", C.c_double), ("t_min", C.c_double),
                ("dilation", C.c_double), ("bg", C.c_double * 3), ("tile", C.c_int32)]


class SH(C.Structure):
    _fields_ = [("rest", C.c_void_p), ("ld", C.c_int64), ("degree", C.c_int32)]


class Split(C.Structure):
    _fields_ = [("index", C.c_int64), ("m", C.c_int32), ("w", C.c_double * 4), ("delta", (C.c_double * 3) * 4)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        L.orc_decide_f32.restype = C.c_int64
        L.orc_decide_f32.argtypes = [P, C.c_int64, C.c_int64, P, P, P, P, P, P]
        L.orc_project_f64.restype = None
        L.orc_project_f64.argtypes = [P, C.c_int64, C.c_int64, P, P, P, P, P, P, P]
        L.orc_eval_sigma.restype = C.c_double
        L.orc_eval_sigma.argtypes = [P, C.c_int64, C.c_int64, P, P, C.c_double, C.c_double]
        L.orc_position_hessian.restype = None
        L.orc_position_hessian.argtypes = [P, C.c_int64, C.c_int64, P, P, C.c_double, C.c_double, P]
        L.orc_render_view.restype = C.c_int64
        L.orc_render_view.argtypes = [P, C.c_int64, C.c_int64, P, P, P, P, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, P, P, P, P, P, P, P, P, P, P, P, P]
        L.orc_sh_basis.restype = None
        L.orc_sh_basis.argtypes = [P, C.c_int32, P, P]
        L.orc_eig_sym3.restype = C.c_int
        L.orc_eig_sym3.argtypes = [P, P, P]
        L.orc_densify.restype = C.c_int64
        L.orc_densify.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, P, C.c_int64, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_int32, C.c_double, C.c_int64, P, P, P]
        L.orc_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def camera(cam: dict) -> Camera:
    c = Camera()
    c.R[:] = [float(x) for x in np.asarray(cam["R"], dtype=np.float64).reshape(9)]
    c.t[:] = [float(x) for x in np.asarray(cam["t"], dtype=np.float64).reshape(3)]
    c.fx, c.fy, c.cx, c.cy = float(cam["fx"]), float(cam["fy"]), float(cam["cx"]), float(cam["cy"])
    c.width, c.height, c.model = int(cam["width"]), int(cam["height"]), int(cam["model"])
    c.znear, c.guard = float(cam["znear"]), float(cam["guard"])
    return c


def raster(rp: dict | None = None) -> Raster:
    rp = DEFAULT_RASTER if rp is None else rp
    r = Raster()
    r.alpha_min, r.alpha_max, r.t_min, r.dilation = (float(np.float32(rp[k])) for k in
                                                     ("alpha_min", "alpha_max", "t_min", "dilation"))
    r.bg[:] = [float(np.float32(b)) for b in rp["bg"]]
    r.tile = int(rp["tile"])
    return r


def f64(params) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(params, dtype=np.float64))


def decide(params, cam: dict, rp: dict | None = None) -> dict:
    p = f64(params)
    n = p.shape[1]
    vis = np.zeros(n, np.uint8)
    key = np.zeros(n, np.uint32)
    rect = np.zeros((n, 4), np.int32)
    tt = np.zeros(n, np.int32)
    c, r = camera(cam), raster(rp)
    nv = lib().orc_decide_f32(_ptr(p), n, n, C.byref(c), C.byref(r), _ptr(vis), _ptr(key), _ptr(rect), _ptr(tt))
    return dict(visible=vis, key=key, rect=rect, tiles_touched=tt, n_visible=int(nv))


def project(params, cam: dict, rp: dict | None = None) -> dict:
    p = f64(params)
    n = p.shape[1]
    mu = np.zeros((n, 2)); cov = np.zeros((n, 3)); con = np.zeros((n, 3)); o = np.zeros(n); z = np.zeros(n)
    c, r = camera(cam), raster(rp)
    lib().orc_project_f64(_ptr(p), n, n, C.byref(c), C.byref(r), _ptr(mu), _ptr(cov), _ptr(con), _ptr(o), _ptr(z))
    return dict(mu=mu, cov2d=cov, conic=con, opacity=o, depth=z)


def eval_sigma(params, i: int, cam: dict, x: float, y: float, rp: dict | None = None) -> float:
    p = f64(params)
    c, r = camera(cam), raster(rp)
    return lib().orc_eval_sigma(_ptr(p), p.shape[1], i, C.byref(c), C.byref(r), x, y)


def position_hessian(params, i: int, cam: dict, x: float, y: float, rp: dict | None = None) -> np.ndarray:
    p = f64(params)
    H = np.zeros(9)
    c, r = camera(cam), raster(rp)
    lib().orc_position_hessian(_ptr(p), p.shape[1], i, C.byref(c), C.byref(r), x, y, _ptr(H))
    return H.reshape(3, 3)


def render(params, cam: dict, rp: dict | None = None, window=None, brute_force: bool = False,
           dl_dimage=None, split: dict | None = None, decision: dict | None = None, sh_rest=None,
           sh_degree: int | None = None) -> dict:
    """One view: image/T/n_comp/ambiguity over `window` = (x0, y0, w, h) (default: full image);
    with dl_dimage ([3][h][w] over the window) also grad[20][n] (14 param grads + 6 S planes),
    absg[20][n] (sum of |per-pair contribution|), absS[6][n] (the S entries' per-pair term magnitudes
    |g sigma| (|U_a U_b| + |(P^T Q P)_ab|), summed: the error scale of a moment-based S),
    amb_g[n] and grad_mu[2][n] (dL/dPi(p), the ADC statistic's per-view gradient).
    sh_degree (0..3) with sh_rest [3 ((deg + 1)^2 - 1)][n]: SH colours (f3; DC = planes 11-13), and
    with dl_dimage also grad_sh [3 ((deg + 1)^2 - 1)][n]."""
    p = f64(params)
    n = p.shape[1]
    if window is None:
        window = (0, 0, int(cam["width"]), int(cam["height"]))
    x0, y0, w, h = (int(v) for v in window)
    d = decision if decision is not None else decide(params, cam, rp)
    img = np.zeros((3, h, w)); T = np.zeros((h, w)); nc = np.zeros((h, w), np.int32); amb = np.zeros((h, w), np.uint8)
    grad = absg = ambg = dl = gmu = None
    if dl_dimage is not None:
        dl = np.ascontiguousarray(np.asarray(dl_dimage, dtype=np.float64).reshape(3, h, w))
        grad = np.zeros((20, n)); absg = np.zeros((26, n)); ambg = np.zeros(n, np.uint8); gmu = np.zeros((2, n))
    sp = None
    if split is not None:
        sp = Split()
        sp.index, sp.m = int(split["index"]), len(split["w"])
        for j, (wj, dj) in enumerate(zip(split["w"], split["delta"])):
            sp.w[j] = float(wj)
            sp.delta[j][:] = [float(v) for v in dj]
    shs = None
    gsh = None
    if sh_degree is not None:
        K = (int(sh_degree) + 1) ** 2
        rest = np.ascontiguousarray(np.zeros((max(3 * (K - 1), 1), n)) if sh_rest is None or K == 1
                                    else np.asarray(sh_rest, dtype=np.float64)[:3 * (K - 1), :n])
        shs = SH()
        shs.rest, shs.ld, shs.degree = rest.ctypes.data, n, int(sh_degree)
        if dl_dimage is not None:
            gsh = np.zeros((max(3 * (K - 1), 1), n))
    c, r = camera(cam), raster(rp)
    pairs = lib().orc_render_view(_ptr(p), n, n, C.byref(c), C.byref(r), _ptr(d["visible"]), _ptr(d["key"]),
                                  x0, y0, w, h, int(brute_force), C.byref(sp) if sp is not None else None,
                                  _ptr(dl), _ptr(img), _ptr(T), _ptr(nc), _ptr(amb), _ptr(grad), _ptr(absg), _ptr(ambg),
                                  _ptr(gmu), C.byref(shs) if shs is not None else None, _ptr(gsh))
    if pairs < 0:
        raise MemoryError("oracle render failed")
    if gsh is not None and sh_degree == 0:
        gsh = np.zeros((0, n))
    absS = None
    if absg is not None:   # rows 20-25: the S entries' term magnitudes (test infrastructure)
        absg, absS = absg[:20].copy(), absg[20:].copy()
    return dict(image=img, final_T=T, n_comp=nc, amb_px=amb, grad=grad, absg=absg, absS=absS, amb_g=ambg,
                grad_mu=gmu, grad_sh=gsh, pairs=int(pairs), decision=d)


def sh_basis(direction, degree: int = 3):
    """(Y[16], dY[16][3]) of the real SH basis (3DGS ordering) at a unit direction."""
    v = np.ascontiguousarray(np.asarray(direction, dtype=np.float64))
    Y = np.zeros(16); dY = np.zeros(48)
    lib().orc_sh_basis(_ptr(v), int(degree), _ptr(Y), _ptr(dY))
    return Y, dY.reshape(16, 3)


def eig_sym3(A) -> tuple[np.ndarray, np.ndarray]:
    """A: 3x3 symmetric or 6-vector (xx,xy,xz,yy,yz,zz) -> (lam ascending [3], V [3,3] columns)."""
    A = np.asarray(A, dtype=np.float64)
    if A.shape == (3, 3):
        A = np.array([A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]])
    a6 = np.ascontiguousarray(A)
    lam = np.zeros(3); V = np.zeros(9)
    lib().orc_eig_sym3(_ptr(a6), _ptr(lam), _ptr(V))
    return lam, V.reshape(3, 3)


def densify(params, acc, n: int, capacity: int, denom: float = 1.0, eps_split: float = -1e-6,
            eta: float = 0.5, eps_abs: float = 0.0, eps_grad: float | None = None, budget: int | None = None,
            grad_gate: float | None = None) -> dict:
    """In-place SDC densify on float64 copies.  params [14][cap], acc [20][cap].  eps_grad: compactest
    gate; budget: increment budget (App. A.2)."""
    p = np.ascontiguousarray(np.array(params, dtype=np.float64))
    a = np.ascontiguousarray(np.array(acc, dtype=np.float64))
    ld, ldg = p.shape[1], a.shape[1]
    mask = np.zeros(n, np.uint8); dest = np.zeros(n, np.int32); lam = np.zeros(n)
    gate, eg = (2, float(grad_gate)) if grad_gate is not None else ((0, 0.0) if eps_grad is None
                                                                     else (1, float(eps_grad)))
    ns = lib().orc_densify(_ptr(p), ld, n, capacity, _ptr(a), ldg, denom, eps_split, eta, eps_abs, gate, eg,
                           -1 if budget is None else int(budget), _ptr(mask), _ptr(dest), _ptr(lam))
    return dict(params=p, acc=a, mask=mask, dest=dest, lambda_min=lam, n_split=int(ns))


def num_threads() -> int:
    return int(lib().orc_num_threads())
