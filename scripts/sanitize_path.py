"""The whole hot path on small seeded inputs, for compute-sanitizer:
C1 (64 Gaussians, 64x64) with 2 views in both camera models and raster modes, plus a denser
2k-Gaussian 128x96 scene so the render rings wrap several times (lists of several batches), then
project -> bin/sort -> fwd (+ fused l1) -> bwd moments -> gauss_bwd + S -> densify (fused, budget,
non-fused capacity) -> Adam.  Run as: compute-sanitizer --tool <t> --kernel-name kns=sgs python
scripts/sanitize_path.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_run import raster_of, to_dev  # noqa: E402
from paper_2505_05587_b200 import _lib  # noqa: E402
from paper_2505_05587_b200.pipeline import Rasterizer  # noqa: E402

DEFAULT = dict(alpha_min=1.0 / 255.0, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0.1, 0.2, 0.3), tile=16)
SMOOTH = dict(alpha_min=0.0, alpha_max=1.0, t_min=0.0, dilation=0.0, bg=(0.0, 0.0, 0.0), tile=16)


def one(p, cams, rp, cap_mult=2, budget=None):
    n = p.shape[1]
    W, H = cams[0]["width"], cams[0]["height"]
    V = len(cams)
    cap = cap_mult * n if cap_mult else n + n // 3
    rz = Rasterizer(cap, V, W, H, raster_of(rp))
    P = torch.zeros(14, cap, device="cuda")
    P[:, :n] = to_dev(p)
    G = torch.zeros(20, cap, device="cuda")
    tg = to_dev(synth.target_images(V, W, H, 5))
    pc = torch.zeros(2, dtype=torch.int64, device="cuda")
    rz.project(P, n, cams)
    rz.bin_sort()
    rz.render_fwd_l1(tg, pair_counts=pc)
    rz.render_bwd_moments()
    rz.gauss_bwd(P, G, accumulate=0)
    m = torch.zeros(14, cap, device="cuda")
    v = torch.zeros(14, cap, device="cuda")
    gacc = torch.zeros(3, cap, device="cuda")
    _lib.adam_step(P, n, G, m, v, _lib.adam_params((1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3)), 1, gacc, False)
    rz.densify(P, G, n, cap, denom=float(V), budget=budget)
    _lib.reset_moments(m, v, n, rz.split_mask, rz.n_split)
    torch.cuda.synchronize()
    return int(rz.n_split.item()), int(pc[0].item())


def main():
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    out = []
    for model in (0, 1):
        cams = synth.cameras_for(cfg, views=2, model=model)
        for rp in (DEFAULT, SMOOTH):
            out.append(one(p, cams, rp))
    out.append(one(p, synth.cameras_for(cfg, views=2), DEFAULT, cap_mult=0))            # non-fused densify
    out.append(one(p, synth.cameras_for(cfg, views=2), DEFAULT, budget=8))             # budget select
    dense = synth.surface_scene(2000, 77)
    cams = synth.ring_cameras(2, 128, 96, 78)
    out.append(one(dense, cams, DEFAULT))
    print("sanitize path ok:", out)


if __name__ == "__main__":
    main()
