# A/B of kernel variants selected by an environment variable (measurement only):
#   VAR=STEEPGS_BWD VALS="1 2 3" TESTS="tests/test_gpu_parity.py -k bwd" bash scripts/gpu_ab.sh
# For each value: the selected GPU tests, then two bench runs (stage times to gpurun_out/ab_summary.txt).
: > gpurun_out/ab_summary.txt
for v in $VALS; do
  if [ -n "$TESTS" ]; then
    env $VAR=$v timeout 600 python -m pytest $TESTS -q -x --timeout 400 -p no:cacheprovider > gpurun_out/ab_tests_$v.log 2>&1
    echo "$VAR=$v tests: $(tail -1 gpurun_out/ab_tests_$v.log)" >> gpurun_out/ab_summary.txt
  fi
done
for r in 1 2; do
  for v in $VALS; do
    env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-v1 ${BENCH_ARGS} > gpurun_out/ab_bench_$v.log 2>&1
    python - "$v" >> gpurun_out/ab_summary.txt <<'PY'
import json, sys
v = sys.argv[1]
for line in open(f"gpurun_out/ab_bench_{v}.log"):
    if line.startswith("{"):
        d = json.loads(line)
        st = {k: x["ms"] for k, x in d["stages"].items() if x["ms"] > 0}
        print(f"{v}: value {d['value']} ms/view  " + " ".join(f"{k}={x:.4f}" for k, x in st.items()))
        break
else:
    print(f"{v}: no JSON line")
PY
  done
done
cat gpurun_out/ab_summary.txt
