# ncu --set full of kernel $K with each library in $LIBS (STEEPGS_LIB) -> gpurun_out/prof_lib<i>.ncu-rep
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-v1"
i=0
for L in $LIBS; do
  STEEPGS_LIB=$L timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-3} -c 1 \
    -o gpurun_out/prof_lib$i $B > gpurun_out/ncu_lib$i.log 2>&1
  i=$((i+1))
done
echo done
