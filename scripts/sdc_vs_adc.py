"""SDC (SteepGS, Alg. 1) vs ADC (3DGS) on a synthetic scene (NEXT f4's comparison; the paper's
headline is ~50% fewer Gaussians at matched quality, P:L43 / Table 1).

A "ground-truth" surface scene (synth.surface_scene, 120k Gaussians) is rendered by the forward kernel
from 24 ring cameras to give target images; the student starts from 15k Gaussians of a different
seed (a sparse, wrong point cloud) and trains for --steps steps, one view per step (3DGS's batch),
densifying every 100 steps from step 500 to --densify-until.  Both runs use the same Adam settings,
schedule and views; only the density control differs.  Prints a markdown table (Gaussian count,
L1 and PSNR over all 24 views at the end) and writes it to --out.

    python scripts/sdc_vs_adc.py --steps 3000 --out profiles/r01_sdc_vs_adc.md
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2505_05587_b200 import Adam, Raster, Rasterizer, Schedule, Trainer  # noqa: E402


def render_views(params, n, cams, W, H):
    rz = Rasterizer(n, len(cams), W, H, Raster())
    rz.project(params, n, cams)
    rz.bin_sort(check=True)
    rz.render_fwd()
    return rz.image.clone()


def evaluate(tr, cams, targets, W, H):
    img = render_views(tr.params, tr.n, cams, W, H)
    l1 = float((img - targets).abs().mean())
    mse = float(((img.clamp(0, 1) - targets) ** 2).mean())
    return l1, 10 * math.log10(1.0 / max(mse, 1e-12))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--densify-until", type=int, default=2500)
    ap.add_argument("--width", type=int, default=490)
    ap.add_argument("--height", type=int, default=272)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    W, H = args.width, args.height
    torch.manual_seed(0)
    cams = synth.ring_cameras(24, W, H, 5)
    gt = torch.from_numpy(synth.surface_scene(120_000, 11)).cuda()
    targets = render_views(gt, gt.shape[1], cams, W, H)
    init = torch.from_numpy(synth.surface_scene(15_000, 12)).cuda()
    n0, cap = init.shape[1], 1_500_000
    adam = Adam(lr=(7e-4, 5e-3, 1e-3, 5e-2, 2.5e-3))
    rows = []
    g3dgs = 0.0004 / W                        # 3DGS's 0.0002 NDC gradient threshold in pixel units (C22)
    arms = [("no densification", dict(density="sdc", t_start=10 ** 9)),
            ("SDC (Alg. 1, no condition on G)", dict(density="sdc")),
            ("SDC + 3DGS gradient condition (C24)", dict(density="sdc", grad_gate=g3dgs)),
            ("ADC (3DGS)", dict(density="adc", eps_adc=g3dgs))]
    for name, kw in arms:
        kw = dict(dict(t_start=500, t_split=100, tau_adc=(0.01 * 4.4) ** 2, min_opacity=0.005), **kw)
        sched = Schedule(**kw)
        tr = Trainer(init, n0, cap, 1, W, H, Raster(), adam, sched, seed=1)
        order = np.random.default_rng(3).permutation(np.arange(args.steps) % len(cams))
        t0 = time.time()
        counts = []
        note = ""
        for t in range(1, args.steps + 1):
            if t > args.densify_until and sched.densify_at(t):
                sched.t_start = 10 ** 9                                     # densification over
            v = int(order[t - 1])
            try:
                tr.step([cams[v]], targets[v:v + 1])
            except RuntimeError as e:                                       # capacity exceeded
                note = f"stopped at step {t}: {e}"
                break
            if t % 500 == 0:
                counts.append((t, tr.n, round(evaluate(tr, cams, targets, W, H)[1], 2)))
        torch.cuda.synchronize()
        dt = time.time() - t0
        l1, psnr = evaluate(tr, cams, targets, W, H)
        rows.append(dict(density=name, n_final=tr.n, l1=l1, psnr=psnr, seconds=dt, counts=counts,
                         splits=[h["n_split"] for h in tr.history], note=note))
    lines = ["| density control | final #Gaussians | L1 (24 views) | PSNR dB | train s | step: #Gaussians (PSNR) every 500 steps |",
             "|---|---:|---:|---:|---:|---|"]
    for r in rows:
        lines.append(f"| {r['density']}{' (' + r['note'] + ')' if r['note'] else ''} | {r['n_final']} | {r['l1']:.5f} | {r['psnr']:.2f} | {r['seconds']:.1f} | "
                     + ", ".join(f"{t}:{c} ({p} dB)" for t, c, p in r["counts"]) + " |")
    table = "\n".join(lines)
    print(table)
    print(json.dumps(rows))
    if args.out:
        with open(args.out, "w") as f:
            f.write("# SDC vs ADC on a synthetic scene (scripts/sdc_vs_adc.py)\n\n")
            f.write(f"Student 15k -> trained {args.steps} steps (1 view/step, {W}x{H}, densify every 100 from 500 "
                    f"to {args.densify_until}); target = 120k-Gaussian synthetic surface scene rendered from 24 ring "
                    "cameras.  Same Adam settings, schedule and view order for both; only density control differs.\n\n")
            f.write(table + "\n")


if __name__ == "__main__":
    main()
