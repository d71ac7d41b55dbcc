"""The whole hot path on seeded inputs for the debug-checked build (SURVEY §5's sanitizer row;
compute-sanitizer is closed on the GPU pool): C1 (64 Gaussians, 64x64) with 2
views in both camera models and raster modes, the non-fused and budget densify paths, a denser
2k-Gaussian 128x96 scene, and C2 at full size with 2 views (lists of hundreds of batches: every ring
stage is reused many times), each through project -> bin/sort -> fwd (+ fused l1) -> bwd moments ->
gauss_bwd + S -> Adam -> densify -> reset_moments.  Prints one JSON line: the device-side check
counters (steepgs_debug_checks) and per-scenario results (image / ids hashes, n_split, pair counts,
gradient sums) so a checked run can be compared with a release run.
Run as:  STEEPGS_LIB=paper_2505_05587_b200/libsteepgs_checked.so python scripts/checked_path.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import hashlib  # noqa: E402
import json  # noqa: E402

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
    rz = Rasterizer(cap, V, W, H, raster_of(rp), max_instances=int(4 * V * n) + 4096)
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
    torch.cuda.synchronize()
    b = rz.binning_arrays()
    img_h = hashlib.sha1(rz.image.cpu().numpy().tobytes()).hexdigest()[:16]
    ids_h = hashlib.sha1(b["ids"].numpy().tobytes()).hexdigest()[:16]
    gsum = [float(x) for x in G[:, :n].double().abs().sum(1).cpu()]
    m = torch.zeros(14, cap, device="cuda")
    v = torch.zeros(14, cap, device="cuda")
    gacc = torch.zeros(3, cap, device="cuda")
    _lib.adam_step(P, n, G, m, v, _lib.adam_params((1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3)), 1, gacc, False)
    rz.densify(P, G, n, cap, denom=float(V), budget=budget)
    _lib.reset_moments(m, v, n, rz.split_mask, rz.n_split)
    torch.cuda.synchronize()
    return dict(image=img_h, ids=ids_h, n_instances=b["n_instances"], n_split=int(rz.n_split.item()),
                pairs=[int(x) for x in pc.cpu()], grad_abs_sum=gsum)


def main():
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    out = {}
    for model in (0, 1):
        cams = synth.cameras_for(cfg, views=2, model=model)
        for name, rp in (("default", DEFAULT), ("smooth", SMOOTH)):
            out[f"C1 model {model} {name}"] = one(p, cams, rp)
    out["C1 non-fused densify"] = one(p, synth.cameras_for(cfg, views=2), DEFAULT, cap_mult=0)
    out["C1 budget densify"] = one(p, synth.cameras_for(cfg, views=2), DEFAULT, budget=8)
    out["2k 128x96"] = one(synth.surface_scene(2000, 77), synth.ring_cameras(2, 128, 96, 78), DEFAULT)
    c2 = synth.CONFIGS["C2"]
    out["C2 2 views"] = one(synth.scene_for(c2), synth.cameras_for(c2, views=2), DEFAULT)
    print(json.dumps(dict(checks=_lib.debug_checks(reset=True), scenarios=out)))


if __name__ == "__main__":
    main()
