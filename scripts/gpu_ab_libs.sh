# bench stage times with each library in $LIBS (STEEPGS_LIB; "default" = the in-tree build), twice.
# ARGS overrides the bench flags (default: C2 8 views, no v1 line); with the v1 line enabled its
# stages are printed too.
: > gpurun_out/ab_summary.txt
ARGS=${ARGS---no-v1}
for r in 1 2; do
  for L in $LIBS; do
    [ "$L" = "default" ] && L=""
    STEEPGS_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $ARGS > gpurun_out/ab_lib.log 2>&1
    python - "${L:-default}" >> gpurun_out/ab_summary.txt <<'PY'
import json, sys
for line in open("gpurun_out/ab_lib.log"):
    if line.startswith("{"):
        d = json.loads(line)
        st = {k: x["ms"] for k, x in d["stages"].items() if x["ms"] > 0}
        print(f"{sys.argv[1]}: value {d['value']} " + " ".join(f"{k}={x:.4f}" for k, x in st.items()))
        if d.get("v1"):
            v = d["v1"]
            print(f"   v1 {v['value']} " + " ".join(f"{k}={x:.4f}" for k, x in v["stages_ms"].items()))
        break
else:
    print(sys.argv[1], "no JSON")
PY
  done
done
cat gpurun_out/ab_summary.txt
