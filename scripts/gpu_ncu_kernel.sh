# ncu --set full on launches of the kernels matching $K (regex) in a bench step (1 GPU);
# S launches skipped, C captured, BARGS extra bench flags (e.g. "--views 1").
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-v1 $BARGS"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-3} -c ${C:-1} -o gpurun_out/prof_k $B > gpurun_out/ncu_k.log 2>&1
echo done
