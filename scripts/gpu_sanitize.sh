# compute-sanitizer over the whole hot path on small inputs (scripts/sanitize_path.py), our kernels only
# (namespace sgs); logs to gpurun_out/sanitize_<tool>.log.  Run on the GPU box through gpurun.
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for t in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$t" = "racecheck" ] && extra="--racecheck-report all"
  timeout 900 $CS --tool $t $extra --kernel-name kns=sgs --print-limit 50 python scripts/sanitize_path.py \
    > gpurun_out/sanitize_$t.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$t.log
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize path ok\|exit=" gpurun_out/sanitize_*.log
