"""Run the CUDA path (through the C ABI) on seeded numpy inputs and bring results back to numpy."""
from __future__ import annotations

import numpy as np
import torch

from paper_2505_05587_b200 import _lib
from paper_2505_05587_b200.pipeline import Raster, Rasterizer


def raster_of(rp: dict) -> Raster:
    return Raster(rp["alpha_min"], rp["alpha_max"], rp["t_min"], rp["dilation"], tuple(rp["bg"]))


def to_dev(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def splat_fields(rz: Rasterizer, n: int):
    """Decode the [V][n] 64-byte splat records (include/steepgs.h)."""
    raw = rz.splats[: rz.V * n * 64].view(rz.V, n, 64).cpu()
    mean = raw[:, :, 0:16].contiguous().view(torch.float64).view(rz.V, n, 2).numpy()
    f = raw[:, :, 16:64].contiguous().view(torch.float32).view(rz.V, n, 12).numpy().astype(np.float64)
    hl2e = 0.5 / np.log(2.0)
    conic = np.stack([f[..., 0] / hl2e, f[..., 1] / (2 * hl2e), f[..., 2] / hl2e], -1)
    return dict(mean=mean, conic=conic, log2_opacity=f[..., 3], rgb=f[..., 4:7], opacity=f[..., 7],
                extent=f[..., 8:10], tau=f[..., 10])


def run_forward(params: np.ndarray, cams, rp: dict, max_instances=None):
    n = params.shape[1]
    V = len(cams)
    rz = Rasterizer(max(n, 1), V, cams[0]["width"], cams[0]["height"], raster_of(rp), max_instances=max_instances)
    p = to_dev(params)
    rz.project(p, n, cams)
    rz.bin_sort()
    rz.render_fwd()
    torch.cuda.synchronize()
    return rz, p


def run_backward(rz: Rasterizer, p, dl: np.ndarray, accumulate=False, grad_S=None):
    n = rz.n
    if grad_S is None:
        grad_S = torch.zeros(20, p.shape[1], dtype=torch.float32, device="cuda")
    rz.render_bwd(p, grad_S, dL=to_dev(dl), accumulate=accumulate)
    torch.cuda.synchronize()
    return grad_S[:, :n].cpu().numpy().astype(np.float64)


def decisions(rz: Rasterizer, n: int):
    V = rz.V
    tt = rz.tiles_touched[: V * n].view(V, n).cpu().numpy()
    key = rz.depth_key[: V * n].view(V, n).cpu().numpy().view(np.uint32)
    rect = rz.tile_rect[: V * n * 2].view(V, n, 2).cpu().numpy().view(np.uint32)
    x0, x1 = rect[..., 0] & 0xFFFF, rect[..., 0] >> 16
    y0, y1 = rect[..., 1] & 0xFFFF, rect[..., 1] >> 16
    return dict(tiles_touched=tt, key=key, tile_rect=np.stack([x0, x1, y0, y1], -1).astype(np.int64))
