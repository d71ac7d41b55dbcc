"""profiles/r0<N>_summary.md from the round's committed profile files (no GPU needed):

    python scripts/round_summary.py 2

reads profiles/r0N_bench_default.json (the default bench line) and profiles/r0N_ncu_full_metrics.json
(scripts/ncu_extract.py of the ncu --set full capture of one timed step)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = sys.argv[1] if len(sys.argv) > 1 else "2"
P = os.path.join(ROOT, "profiles")
b = json.load(open(os.path.join(P, f"r0{N}_bench_default.json")))
m = json.load(open(os.path.join(P, f"r0{N}_ncu_full_metrics.json")))
st = b["stages"]
L = [f"# Round {N} profile summary — C2 (1.0M Gaussians, 980×545), 8 views per step, 1×B200\n",
     f"Sources (gpurun B200 box, clocks uncontrolled): `r0{N}_bench_default.json` (the default `python bench.py` line "
     f"of this build), `r0{N}_launches.csv` (`ncu --metrics gpu__time_duration.sum --clock-control none` launch list "
     f"of one bench step, cold-cache, serialised), `r0{N}_ncu_full_metrics.json` (`ncu --set full --clock-control none "
     f"--import-source on` of the 13 kernels of one timed step, `scripts/gpu_round_profile.sh` + "
     f"`scripts/ncu_extract.py`), `traffic.json` (DRAM bytes per launch, bench's `roofline.traffic`), "
     f"`r0{N}_configs.md` (C2-C5 and the f2/f3 workloads), `r02/checked_build.md`, `r02_oracle_mutations.md`.\n",
     f"Bench line: **{b['value']} ms/view** device ({b['ms_per_step']} ms per 8-view step, whole-step graph replays; "
     f"{b.get('ms_per_step_with_stage_events')} ms with the per-stage events), e2e {b['e2e']['value']:.4f} ms/view, "
     f"v1 (one view per step, SURVEY §8(d1)) {b['v1']['value']} ms/view (fwd+bwd+S {b['v1']['fwd_bwd_S_ms_per_view']}), "
     f"CPU oracle {b['cpu_baseline']['value']} ms/view on {b['cpu_baseline']['cores']} threads (whole views, median of 3); "
     f"clocks {b['clocks']}.\n",
     f"Dominant kernel `{b['roofline']['kernel']}`: {b['roofline']['achieved']} T lane-op/s of {b['roofline']['peak']} = "
     f"**{b['roofline']['frac']}** of the FP32 lane-op roofline (45 lane-ops × "
     f"{b['roofline']['units_per_launch']['contributing_pairs']} contributing pairs per launch); whole path "
     f"{b['path_hbm']['frac']} of the HBM roofline.\n",
     "| kernel | ncu µs | bench stage ms | DRAM MB | issue % | lanes | warp instr | top stalls |",
     "|---|---:|---:|---:|---:|---:|---:|---|"]
smap = {"k_project": "project", "k_render_fwd": "render_fwd", "k_render_bwd2": "render_bwd", "k_gauss_bwd": "gauss_bwd_S",
        "k_densify_decide": "densify"}
for r in m["rows"]:
    k = r["kernel"]
    dram = (r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)) / 1e6
    top = ", ".join(f"{a} {v:.0f}%" for a, v in list(r.get("top_stalls_pct", {}).items())[:3])
    stage = st.get(smap[k], {}).get("ms", "") if k in smap else ""
    L.append(f"| {k} | {r['gpu__time_duration.sum'] * 1e3:.0f} | {stage} | {dram:.0f} | "
             f"{r.get('sm__inst_issued.avg.pct_of_peak_sustained_active', 0):.0f} | "
             f"{r.get('smsp__thread_inst_executed_per_inst_executed.ratio', 0):.1f} | "
             f"{r.get('smsp__inst_executed.sum', 0) / 1e6:.0f}M | {top} |")
pairs = b["roofline"]["units_per_launch"]["contributing_pairs"]
lanes = {r["kernel"]: r["smsp__inst_executed.sum"] * 32 / pairs for r in m["rows"] if r["kernel"] in ("k_render_fwd", "k_render_bwd2")}
L.append(f"\nbin_sort stage (count + scan + compact + 4 depth passes + duplicate + 2 tile passes + ranges + tile order): {st['bin_sort']['ms']} ms.\n")
L.append("Lane slots per contributing pair (warp instructions × 32 / contributing pairs): "
         + ", ".join(f"{k} {v:.0f}" for k, v in lanes.items()) + " (round 1: k_render_bwd 195, k_render_fwd 99).  "
         "Round-2 changes and dead ends with their numbers: DESIGN.md §10 (round 2).\n")
L.append("DRAM traffic of the raster kernels against their algorithmic bytes: the longest-list-first tile "
         "order (binning.tile_order) keeps all views' splat records and moments in flight, so render_fwd / "
         "render_bwd2 read about 1.6x what the raster (view-major) order read (462 / 654 MB per step); both "
         "kernels are issue-bound and the order is faster overall — the per-view alternative that restores "
         "the traffic is measured in DESIGN.md §5 (k_tile_order).\n")
open(os.path.join(P, f"r0{N}_summary.md"), "w").write("\n".join(L) + "\n")
print("\n".join(L))
