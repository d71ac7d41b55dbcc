# A/B of kernel source variants (_variants/<name>.cu, git-ignored, copied over $TARGET, rebuilt in place, benched)
# usage: TARGET=paper_2505_05587_b200/csrc/x.cu bash scripts/gpu_variant_ab.sh name1 name2 ...
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "$@"; do
  cp _variants/$v.cu $TARGET
  python -c "from paper_2505_05587_b200 import build; build.build()" > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', d['value'], {k:v['ms'] for k,v in d['stages'].items() if k in ('gauss_bwd_S','bin_sort','render_fwd','render_bwd','project')})"
done; done
