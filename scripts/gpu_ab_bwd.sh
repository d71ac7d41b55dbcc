timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -q -x --timeout 400 -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo exit=$? >> gpurun_out/ab_tests.log
for v in 1 2 1 2; do STEEPGS_BWD=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-v1 > gpurun_out/ab_bench_$v.log 2>&1; python - <<'PY' >> gpurun_out/ab_summary.txt
import json,os
v=os.environ.get("V","")
PY
grep -o '"render_bwd": {"ms": [0-9.]*' gpurun_out/ab_bench_$v.log | sed "s/^/v$v /" >> gpurun_out/ab_summary.txt; grep -o '"value": [0-9.]*' gpurun_out/ab_bench_$v.log | head -1 | sed "s/^/v$v /" >> gpurun_out/ab_summary.txt; done
