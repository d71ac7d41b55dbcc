"""Print the last bench step's kernels from an ncu launch list (gpurun_out/launches.csv)."""
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
last = int(sys.argv[2]) if len(sys.argv) > 2 else 14
rows = list(csv.reader(open(path)))
h, out = None, []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0][-48:], float(d["Metric Value"]) / 1e3))
for k, v in out[-last:]:
    print(f"{v:9.1f} us  {k}")
