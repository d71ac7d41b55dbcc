# e2e A/B of the target-copy placement (bench.py --h2d-at); 1 GPU, results under gpurun_out/
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do for m in start after_sort; do
  timeout 200 python bench.py --no-cpu-baseline --h2d-at $m > gpurun_out/h2d_$m.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/h2d_$m.json')); print('$m', d['value'], round(d['e2e']['value'], 5))"
done; done
