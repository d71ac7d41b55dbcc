"""Summarise an `ncu --set full` report of one bench step into profiles/:

    python scripts/ncu_extract.py gpurun_out/prof_full.ncu-rep r02

writes profiles/<tag>_ncu_full_metrics.json (per launch: DRAM bytes, duration, SM / memory
throughput, registers, executed instructions, issue-slot utilisation, top stall reasons) and
profiles/traffic.json (per kernel: DRAM read + write bytes per launch, the `roofline.traffic` of
bench.py).  Runs here (no GPU needed): it only reads the report with `ncu -i`.
"""
from __future__ import annotations

import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
       "smsp__inst_executed.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio",             # warp efficiency (active lanes)
       "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",        # global RED (atomic) traffic
       "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"]


def short(name: str) -> str:
    base = name.split("(")[0]
    for pre in ("void ", "sgs::", "<unnamed>::", "unnamed>::"):
        base = base.replace(pre, "")
    return base.split("<")[0].strip()


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    stall = [i for i, c in enumerate(hdr)
             if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued")]
    recs = []
    for r in rows[2:]:
        d = {"id": int(r[hdr.index("ID")]), "kernel": short(r[hdr.index("Kernel Name")])}
        for m in RAW:
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    x = float(v) if v else 0.0
                except ValueError:          # "no data" / "n/a"
                    continue
                if u == "Kbyte":
                    x *= 1e3
                elif u == "Mbyte":
                    x *= 1e6
                elif u == "Gbyte":
                    x *= 1e9
                elif u == "usecond":
                    x *= 1e-3
                elif u == "nsecond":
                    x *= 1e-6
                d[m] = x
        tot = sum(float(r[i].replace(",", "") or 0) for i in stall) or 1.0
        top = sorted(((float(r[i].replace(",", "") or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                      for i in stall), reverse=True)[:5]
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for v, k in top}
        recs.append(d)
    meta = {"units": {"dram__bytes_*": "byte", "gpu__time_duration.sum": "ms", "*pct*": "%",
                      "launch__registers_per_thread": "register/thread", "smsp__inst_executed.sum": "warp inst"},
            "source": f"ncu --set full --clock-control none of one bench step ({os.path.basename(rep)})",
            "rows": recs}
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_metrics.json"), "w") as f:
        json.dump(meta, f, indent=1)
    traffic = {}
    for d in recs:
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        e = traffic.setdefault(d["kernel"], {"bytes_per_launch": 0.0, "launches": 0})
        e["bytes_per_launch"] += b
        e["launches"] += 1
    for k, e in traffic.items():
        e["bytes_per_launch"] /= e["launches"]
        e.update(views=8, workload="C2 (1.0M Gaussians, 980x545), 8 views per launch",
                 source=f"profiles/{tag}_ncu_full_metrics.json: ncu --set full --clock-control none, "
                        "dram__bytes_read.sum + dram__bytes_write.sum")
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    for d in recs:
        print(f"{d['kernel']:20s} {d.get('gpu__time_duration.sum', 0):8.3f} ms  DRAM "
              f"{(d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e6:8.1f} MB "
              f"({d.get('FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed', 0):4.1f}%)  "
              f"issue {d.get('sm__inst_issued.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
              f"lanes {d.get('smsp__thread_inst_executed_per_inst_executed.ratio', 0):4.1f}  "
              f"RED sectors {d.get('l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum', 0):.3g}  {d['top_stalls_pct']}")


if __name__ == "__main__":
    main()
