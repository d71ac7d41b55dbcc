# ncu --set full of kernel $K under each value of $VAR in $VALS -> gpurun_out/prof_$v.ncu-rep (1 GPU)
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-v1"
for v in $VALS; do
  env $VAR=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-3} -c 1 \
    -o gpurun_out/prof_$v $B > gpurun_out/ncu_$v.log 2>&1
done
echo done
