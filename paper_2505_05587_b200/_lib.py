"""Thin ctypes binding of libsteepgs.so (include/steepgs.h).  Argument marshalling only: every step
of the hot path runs in the library's sm_100a kernels.  There is no fallback: if the library or a
compute-capability-10.x device is missing, every call raises."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# STEEPGS_LIB selects another build of the same library (the debug-checked libsteepgs_checked.so,
# tests/test_checked_build.py); the default is the in-tree release build
LIB_PATH = os.environ.get("STEEPGS_LIB") or os.path.join(_HERE, "libsteepgs.so")

STATUS = {0: "ok", 1: "invalid argument", 2: "workspace too small", 3: "capacity exceeded",
          5: "unsupported device", 6: "CUDA error"}


class SteepGSError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str):
        super().__init__(f"{fn}: {STATUS.get(status, status)} ({detail})")
        self.status = status


class Camera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("model", C.c_int32), ("znear", C.c_float), ("guard", C.c_float)]


class RasterParams(C.Structure):
    _fields_ = [("alpha_min", C.c_float), ("alpha_max", C.c_float), ("t_min", C.c_float),
                ("dilation", C.c_float), ("bg", C.c_float * 3), ("tile", C.c_int32)]


class DensifyParams(C.Structure):
    _fields_ = [("eps_split", C.c_float), ("eta", C.c_float), ("eps_abs", C.c_float),
                ("eps_grad", C.c_float), ("denom", C.c_float), ("gate", C.c_int32), ("budget", C.c_int64)]


class AdcParams(C.Structure):
    _fields_ = [("eps_adc", C.c_float), ("tau_adc", C.c_float), ("clone_step", C.c_float),
                ("scale_factor", C.c_float), ("denom", C.c_float), ("reserved", C.c_int32)]


class AdamParams(C.Structure):
    _fields_ = [("lr", C.c_double * 5), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class Binning(C.Structure):
    _fields_ = [("ids", C.c_void_p), ("ranges", C.c_void_p), ("n_instances", C.c_void_p),
                ("n_visible", C.c_void_p), ("overflow", C.c_void_p), ("tile_last", C.c_void_p),
                ("inst_mask", C.c_void_p),
                ("max_instances", C.c_int64),
                ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("V", C.c_int32),
                ("generation", C.c_uint64), ("fwd_token", C.c_uint64), ("tile_order", C.c_void_p)]


SPLAT_BYTES = 64
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I64, I32, F = C.c_void_p, C.c_int64, C.c_int32, C.c_float
        sig = {
            "steepgs_project": [P, I64, I64, P, I32, P, P, P, P, P, P],
            "steepgs_bin_sort_workspace_size": [I64, I32, I32, I32, I64, P],
            "steepgs_bin_sort": [P, P, P, I64, P, I32, P, P, C.c_size_t, I64, P, P],
            "steepgs_render_fwd": [P, I64, P, P, I32, P, P, P, P, P, P],
            "steepgs_render_fwd_l1": [P, I64, P, P, I32, P, P, P, P, P, F, P, P, P, P],
            "steepgs_render_fwd_l1_u8": [P, I64, P, P, I32, P, P, P, P, P, F, P, P, P, P],
            "steepgs_render_bwd_moments": [P, I64, P, P, I32, P, P, P, P, P, P],
            "steepgs_gauss_bwd_split": [P, I64, I64, P, I32, P, P, P, I64, I32, P, P, P],
            "steepgs_copy_planes": [P, I64, P, I64, I64, I32, I32, P],
            "steepgs_l1_grad": [P, P, I32, I64, F, P, P, P],
            "steepgs_render_bwd_split": [P, I64, I64, P, P, P, I32, P, P, P, P, P, P, I64, I32, P, P, P],
            "steepgs_densify_workspace_size": [I64, P],
            "steepgs_densify": [P, I64, I64, I64, P, I64, P, P, P, P, P, P, P, C.c_size_t, P],
            "steepgs_densify_host_count": [P, I64, I64, I64, P, I64, P, P, P, P, P, P, P, C.c_size_t, P, P],
            "steepgs_adc_workspace_size": [I64, P],
            "steepgs_densify_adc": [P, I64, I64, I64, P, I64, P, P, I64, P, P, P, P, P, P, C.c_size_t, P],
            "steepgs_adam_step": [P, I64, I64, P, I64, P, P, I64, P, I64, P, I32, P],
            "steepgs_reset_moments": [P, P, I64, I64, P, P, I32, I32, P],
            "steepgs_project_sh": [P, I64, I64, P, I64, I32, P, I32, P, P, P, P, P, P],
            "steepgs_sh_bwd": [P, I64, I64, P, I64, I32, P, I32, P, P, I64, P, I64, I32, P],
            "steepgs_adam_step_planes": [P, I64, I32, I64, P, I64, P, P, I64, P, I64, P],
            "steepgs_copy_offspring": [P, I64, I32, I64, P, P],
            "steepgs_prune_workspace_size": [I64, P],
            "steepgs_prune_decide": [P, I64, I64, F, P, P, P, C.c_size_t, P],
            "steepgs_compact_planes": [P, I64, P, I64, I32, I64, P, P],
            "steepgs_loss_workspace_size": [I32, I32, I32, P],
            "steepgs_l1_ssim_grad": [P, P, I32, I32, I32, F, F, P, P, P, C.c_size_t, P],
            "steepgs_debug_checks": [P, P, P, I32],
            "steepgs_scatter_chunk": [I64, I32, P],
            "steepgs_gauss_bwd_scatter": [P, I64, I64, P, I32, P, P, P, I32, I32, I64, P],
            "steepgs_reduce_bcast": [P, I32, I32, I64, I64, P, I64, I32, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.steepgs_last_error.restype = C.c_char_p
        L.steepgs_launch_count.restype = C.c_uint64
        L.steepgs_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(fn: str, status: int):
    if status != 0:
        raise SteepGSError(fn, status, lib().steepgs_last_error().decode())


def ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return int(t)


def stream_ptr(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def cameras(cams: list[dict]):
    arr = (Camera * len(cams))()
    for k, c in enumerate(cams):
        arr[k].R[:] = [float(x) for x in np.asarray(c["R"], dtype=np.float32).reshape(9)]
        arr[k].t[:] = [float(x) for x in np.asarray(c["t"], dtype=np.float32).reshape(3)]
        arr[k].fx, arr[k].fy, arr[k].cx, arr[k].cy = (float(np.float32(c[key])) for key in ("fx", "fy", "cx", "cy"))
        arr[k].width, arr[k].height, arr[k].model = int(c["width"]), int(c["height"]), int(c["model"])
        arr[k].znear, arr[k].guard = float(np.float32(c["znear"])), float(np.float32(c["guard"]))
    return arr


def raster_params(alpha_min=1.0 / 255.0, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), tile=16):
    r = RasterParams()
    r.alpha_min, r.alpha_max, r.t_min, r.dilation = alpha_min, alpha_max, t_min, dilation
    r.bg[:] = [float(b) for b in bg]
    r.tile = tile
    return r


def densify_params(eps_split=-1e-6, eta=0.5, eps_abs=0.0, denom=1.0, eps_grad=None, budget=None, grad_gate=None):
    """eps_grad: compactest gate (gate 1); grad_gate: 3DGS-style view-gradient condition (gate 2)."""
    if grad_gate is not None and eps_grad is not None:
        raise ValueError("densify: eps_grad (compactest gate, App. A.2) and grad_gate (C24) are exclusive gates")
    d = DensifyParams()
    d.eps_split, d.eta, d.eps_abs, d.denom = eps_split, eta, eps_abs, denom
    if grad_gate is not None:
        d.gate, d.eps_grad = 2, float(grad_gate)
    else:
        d.gate, d.eps_grad = (0, 0.0) if eps_grad is None else (1, float(eps_grad))
    d.budget = -1 if budget is None else int(budget)
    return d


def project(params, ld, n, cams_arr, V, rp, splats, depth_key, tile_rect, tiles_touched, stream=None):
    _check("steepgs_project", lib().steepgs_project(ptr(params), ld, n, cams_arr, V, C.byref(rp), ptr(splats),
                                                    ptr(depth_key), ptr(tile_rect), ptr(tiles_touched),
                                                    stream_ptr(stream)))


def bin_sort_workspace_size(n, V, width, height, max_instances) -> int:
    out = C.c_size_t(0)
    _check("steepgs_bin_sort_workspace_size",
           lib().steepgs_bin_sort_workspace_size(n, V, width, height, max_instances, C.byref(out)))
    return int(out.value)


def bin_sort(depth_key, tile_rect, tiles_touched, n, cams_arr, V, rp, ws, max_instances, stream=None) -> Binning:
    b = Binning()
    _check("steepgs_bin_sort", lib().steepgs_bin_sort(ptr(depth_key), ptr(tile_rect), ptr(tiles_touched), n, cams_arr,
                                                      V, C.byref(rp), ptr(ws), ws.numel() * ws.element_size(),
                                                      max_instances, C.byref(b), stream_ptr(stream)))
    return b


def render_fwd(splats, n, binning, cams_arr, V, rp, image, final_T, n_contrib, pair_counts=None, stream=None):
    _check("steepgs_render_fwd", lib().steepgs_render_fwd(ptr(splats), n, C.byref(binning), cams_arr, V, C.byref(rp),
                                                          ptr(image), ptr(final_T), ptr(n_contrib), ptr(pair_counts),
                                                          stream_ptr(stream)))


def render_fwd_l1(splats, n, binning, cams_arr, V, rp, image, final_T, n_contrib, target, scale, dL, loss=None,
                  pair_counts=None, stream=None):
    _check("steepgs_render_fwd_l1",
           lib().steepgs_render_fwd_l1(ptr(splats), n, C.byref(binning), cams_arr, V, C.byref(rp), ptr(image),
                                       ptr(final_T), ptr(n_contrib), ptr(target), float(scale), ptr(dL), ptr(loss),
                                       ptr(pair_counts), stream_ptr(stream)))


def render_fwd_l1_u8(splats, n, binning, cams_arr, V, rp, image, final_T, n_contrib, target, scale, dL, loss=None,
                     pair_counts=None, stream=None):
    _check("steepgs_render_fwd_l1_u8",
           lib().steepgs_render_fwd_l1_u8(ptr(splats), n, C.byref(binning), cams_arr, V, C.byref(rp), ptr(image),
                                          ptr(final_T), ptr(n_contrib), ptr(target), float(scale), ptr(dL), ptr(loss),
                                          ptr(pair_counts), stream_ptr(stream)))


def render_bwd_moments(splats, n, binning, cams_arr, V, rp, final_T, n_contrib, dL, moments, stream=None):
    _check("steepgs_render_bwd_moments",
           lib().steepgs_render_bwd_moments(ptr(splats), n, C.byref(binning), cams_arr, V, C.byref(rp), ptr(final_T),
                                            ptr(n_contrib), ptr(dL), ptr(moments), stream_ptr(stream)))


def gauss_bwd_split(params, ld, n, cams_arr, V, rp, moments, grad_S, ldg, accumulate, tiles_touched=None,
                    view_grad_stats=None, stream=None):
    _check("steepgs_gauss_bwd_split",
           lib().steepgs_gauss_bwd_split(ptr(params), ld, n, cams_arr, V, C.byref(rp),
                                         ptr(moments), ptr(grad_S), ldg, int(accumulate), ptr(tiles_touched),
                                         ptr(view_grad_stats), stream_ptr(stream)))


def copy_planes(dst, src, n, first, count, stream=None):
    _check("steepgs_copy_planes", lib().steepgs_copy_planes(ptr(dst), dst.shape[1], ptr(src), src.shape[1], n, first,
                                                            count, stream_ptr(stream)))


def l1_grad(image, target, V, count, scale, dL, loss=None, stream=None):
    _check("steepgs_l1_grad", lib().steepgs_l1_grad(ptr(image), ptr(target), V, count, scale, ptr(dL), ptr(loss),
                                                    stream_ptr(stream)))


def render_bwd_split(params, ld, n, splats, binning, cams_arr, V, rp, final_T, n_contrib, dL,
                     moments, grad_S, ldg, accumulate, tiles_touched=None, view_grad_stats=None, stream=None):
    _check("steepgs_render_bwd_split",
           lib().steepgs_render_bwd_split(ptr(params), ld, n, ptr(splats), C.byref(binning),
                                          cams_arr, V, C.byref(rp), ptr(final_T), ptr(n_contrib), ptr(dL),
                                          ptr(moments), ptr(grad_S), ldg, int(accumulate), ptr(tiles_touched),
                                          ptr(view_grad_stats), stream_ptr(stream)))


def densify_workspace_size(n) -> int:
    out = C.c_size_t(0)
    _check("steepgs_densify_workspace_size", lib().steepgs_densify_workspace_size(n, C.byref(out)))
    return int(out.value)


def densify(params, ld, n, capacity, grad_S, ldg, dp, mask, dest, lam, n_split, status, ws, stream=None):
    _check("steepgs_densify", lib().steepgs_densify(ptr(params), ld, n, capacity, ptr(grad_S), ldg, C.byref(dp),
                                                    ptr(mask), ptr(dest), ptr(lam), ptr(n_split), ptr(status),
                                                    ptr(ws), ws.numel() * ws.element_size(), stream_ptr(stream)))


def adc_params(eps_adc, tau_adc, clone_step=0.0, scale_factor=0.8, denom=1.0):
    a = AdcParams()
    a.eps_adc, a.tau_adc, a.clone_step, a.scale_factor, a.denom = (float(eps_adc), float(tau_adc), float(clone_step),
                                                                   float(scale_factor), float(denom))
    return a


def adc_workspace_size(n) -> int:
    out = C.c_size_t(0)
    _check("steepgs_adc_workspace_size", lib().steepgs_adc_workspace_size(n, C.byref(out)))
    return int(out.value)


def densify_adc(params, n, capacity, grad_S, stats, normals, ap, kind, dest, n_new, status, ws, stream=None):
    assert stats.shape[1] == grad_S.shape[1]
    _check("steepgs_densify_adc",
           lib().steepgs_densify_adc(ptr(params), params.shape[1], n, capacity, ptr(grad_S), grad_S.shape[1],
                                     ptr(stats), ptr(normals), normals.shape[1], C.byref(ap), ptr(kind), ptr(dest),
                                     ptr(n_new), ptr(status), ptr(ws), ws.numel() * ws.element_size(),
                                     stream_ptr(stream)))


def adam_params(lr, beta1=0.9, beta2=0.999, eps=1e-15):
    a = AdamParams()
    a.lr[:] = [float(x) for x in lr]
    a.beta1, a.beta2, a.eps = float(beta1), float(beta2), float(eps)
    return a


def adam_step(params, n, grad_S, m, v, ap, step, gacc=None, gacc_accumulate=True, stream=None):
    _check("steepgs_adam_step", lib().steepgs_adam_step(ptr(params), params.shape[1], n, ptr(grad_S), grad_S.shape[1],
                                                        ptr(m), ptr(v), m.shape[1], C.byref(ap), int(step), ptr(gacc),
                                                        int(bool(gacc_accumulate)), stream_ptr(stream)))


def reset_moments(m, v, n, split_mask, n_split, mask_value=1, stream=None):
    _check("steepgs_reset_moments", lib().steepgs_reset_moments(ptr(m), ptr(v), m.shape[1], n, ptr(split_mask),
                                                                ptr(n_split), int(mask_value), m.shape[0],
                                                                stream_ptr(stream)))


def project_sh(params, ld, n, sh_rest, sh_degree, cams_arr, V, rp, splats, depth_key, tile_rect, tiles_touched,
               stream=None):
    _check("steepgs_project_sh", lib().steepgs_project_sh(
        ptr(params), ld, n, ptr(sh_rest), sh_rest.shape[1] if sh_rest is not None else 0, int(sh_degree), cams_arr, V,
        C.byref(rp), ptr(splats), ptr(depth_key), ptr(tile_rect), ptr(tiles_touched), stream_ptr(stream)))


def sh_bwd(params, n, sh_rest, sh_degree, cams_arr, V, moments, grad_S, grad_sh, accumulate, stream=None):
    _check("steepgs_sh_bwd", lib().steepgs_sh_bwd(
        ptr(params), params.shape[1], n, ptr(sh_rest), sh_rest.shape[1] if sh_rest is not None else 0, int(sh_degree),
        cams_arr, V, ptr(moments), ptr(grad_S), grad_S.shape[1], ptr(grad_sh),
        grad_sh.shape[1] if grad_sh is not None else 0, int(accumulate), stream_ptr(stream)))


def adam_step_planes(params, n, grad, m, v, ap, step, stream=None):
    _check("steepgs_adam_step_planes", lib().steepgs_adam_step_planes(
        ptr(params), params.shape[1], params.shape[0], n, ptr(grad), grad.shape[1], ptr(m), ptr(v), m.shape[1],
        C.byref(ap), int(step), stream_ptr(stream)))


def loss_workspace_size(V, H, W) -> int:
    out = C.c_size_t(0)
    _check("steepgs_loss_workspace_size", lib().steepgs_loss_workspace_size(V, H, W, C.byref(out)))
    return int(out.value)


def l1_ssim_grad(image, target, lam, scale, dL, loss, ws, stream=None):
    V, _, H, W = image.shape
    _check("steepgs_l1_ssim_grad", lib().steepgs_l1_ssim_grad(ptr(image), ptr(target), V, H, W, float(lam), float(scale),
                                                              ptr(dL), ptr(loss), ptr(ws), ws.numel() * ws.element_size(),
                                                              stream_ptr(stream)))


def prune_workspace_size(n) -> int:
    out = C.c_size_t(0)
    _check("steepgs_prune_workspace_size", lib().steepgs_prune_workspace_size(n, C.byref(out)))
    return int(out.value)


def prune_decide(params, n, logit_min, new_index, n_keep, ws, stream=None):
    _check("steepgs_prune_decide", lib().steepgs_prune_decide(ptr(params), params.shape[1], n, float(logit_min),
                                                              ptr(new_index), ptr(n_keep), ptr(ws),
                                                              ws.numel() * ws.element_size(), stream_ptr(stream)))


def compact_planes(src, dst, n, new_index, stream=None):
    assert src.shape[0] == dst.shape[0]
    _check("steepgs_compact_planes", lib().steepgs_compact_planes(ptr(src), src.shape[1], ptr(dst), dst.shape[1],
                                                                  src.shape[0], n, ptr(new_index), stream_ptr(stream)))


def copy_offspring(arr, n, dest_index, stream=None):
    _check("steepgs_copy_offspring", lib().steepgs_copy_offspring(ptr(arr), arr.shape[1], arr.shape[0], n,
                                                                  ptr(dest_index), stream_ptr(stream)))


def launch_count() -> int:
    return int(lib().steepgs_launch_count())


def version() -> str:
    return lib().steepgs_version().decode()


def debug_checks(reset: bool = False) -> dict:
    """Device-side invariant checks of the checked build (see steepgs.h): compiled, failures, first_line."""
    c, f, l = C.c_int32(0), C.c_uint64(0), C.c_uint32(0)
    _check("steepgs_debug_checks", lib().steepgs_debug_checks(C.byref(c), C.byref(f), C.byref(l), int(bool(reset))))
    return dict(compiled=bool(c.value), failures=int(f.value), first_line=int(l.value))


def scatter_chunk(n: int, R: int) -> int:
    c = C.c_int64(0)
    _check("steepgs_scatter_chunk", lib().steepgs_scatter_chunk(int(n), int(R), C.byref(c)))
    return int(c.value)


def _ptr_array(ptrs):
    arr = (C.c_uint64 * len(ptrs))()
    for k, p in enumerate(ptrs):
        arr[k] = int(p)
    return arr


def gauss_bwd_scatter(params, ld, n, cams_arr, V, rp, moments, peer_partials, R, rank, chunk, stream=None):
    """peer_partials: R device pointers (ints) of the owners' [R][20][chunk] partial buffers."""
    _check("steepgs_gauss_bwd_scatter",
           lib().steepgs_gauss_bwd_scatter(ptr(params), ld, n, cams_arr, V, C.byref(rp), ptr(moments),
                                           _ptr_array(peer_partials), R, rank, chunk, stream_ptr(stream)))


def reduce_bcast(partials, R, rank, n, chunk, peer_grad_S, ldg, accumulate=0, stream=None):
    """peer_grad_S: R device pointers (ints) of the ranks' [20][ldg] grad_S."""
    _check("steepgs_reduce_bcast",
           lib().steepgs_reduce_bcast(ptr(partials), R, rank, n, chunk, _ptr_array(peer_grad_S), ldg, int(accumulate),
                                      stream_ptr(stream)))
