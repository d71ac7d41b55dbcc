"""Markdown tables of profiles/<tag>_configs.md from the bench lines of scripts/gpu_configs.sh.

    python scripts/configs_table.py gpurun_out > profiles/r01_configs.md
"""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
ROUND = sys.argv[2] if len(sys.argv) > 2 else "2"


def line(name):
    with open(os.path.join(d, f"cfg_{name}.json")) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def m(x):
    return f"{x / 1e6:.1f}M"


print(f"# All BASELINE configs on 1×B200 (bench.py --config Cx, 8 views per step; round {ROUND})\n")
print("`python bench.py --config Cx --no-cpu-baseline` on the gpurun box (`scripts/gpu_configs.sh`, same build as the "
      f"C2 headline in `r0{ROUND}_summary.md`).  C1 is the oracle-sized parity case (64 Gaussians) and is not a bench line.  "
      "Per-stage ms are CUDA-event means over the timed steps.\n")
print("| config | n | W×H | ms/view | e2e ms/view | ms/step | project | bin_sort | fwd | bwd | gauss_bwd+S | densify | "
      "N_vis | I | contributing pairs | split |")
print("|---|---:|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
for c in ("C2", "C3", "C4", "C5"):
    j = line(c)
    s, k, cf = j["stages"], j["counts"], j["config"]
    print(f"| {c} | {cf['n'] / 1e6:.1f}M | {cf['width']}×{cf['height']} | {j['value']:.3f} | {j['e2e']['value']:.3f} | "
          f"{j['ms_per_step']:.2f} | {s['project']['ms']:.3f} | {s['bin_sort']['ms']:.3f} | {s['render_fwd']['ms']:.3f} | "
          f"{s['render_bwd']['ms']:.3f} | {s['gauss_bwd_S']['ms']:.3f} | {s['densify']['ms']:.3f} | {m(k['n_visible'])} | "
          f"{m(k['n_instances'])} | {k['contributing_pairs'] / 1e6:.0f}M | {k['split_frac']:.2f} |")
print("\nThe 3DGS training workload shape (NEXT f3): C2 with view-dependent SH colour (degree 3, 45 rest coefficients "
      "per Gaussian) and the (1 − λ)ℓ1 + λ(1 − SSIM) loss (`bench.py --sh-degree 3 [--ssim 0.2]`; the loss "
      "kernels are timed in the `l1_grad` stage):\n")
print("| workload | ms/view | e2e ms/view | project | bin_sort | fwd | loss | bwd | sh_bwd + gauss_bwd | densify |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
for c in ("C2_sh3", "C2_sh3_ssim"):
    j = line(c)
    s = j["stages"]
    print(f"| {j['config']['workload']} | {j['value']:.3f} | {j['e2e']['value']:.3f} | {s['project']['ms']:.3f} | "
          f"{s['bin_sort']['ms']:.3f} | {s['render_fwd']['ms']:.3f} | {s['l1_grad']['ms']:.3f} | {s['render_bwd']['ms']:.3f} | "
          f"{s['gauss_bwd_S']['ms']:.3f} | {s['densify']['ms']:.3f} |")
print("\nDensify throughput at C4 (2.5M Gaussians; SURVEY §8(d1) asks for a ~10% split, here via the App. A.2 increment "
      "budget K = 0.1 n, which adds the on-device radix select of the K-th least λ_min):\n")
print("| densify rule | split fraction | densify ms | densify Gaussians/s |")
print("|---|---:|---:|---:|")
for c, rule in (("C4", "λ_min < −1e-6 (P:L401)"), ("C4_budget", "budget K = 0.1 n (App. A.2)")):
    j = line(c)
    print(f"| {rule} | {j['counts']['split_frac']:.2f} | {j['stages']['densify']['ms']:.3f} | "
          f"{j['densify_gaussians_per_s'] / 1e9:.1f}×10⁹ |")
