# ncu --set full on one launch of the kernel matching $K (regex) in a bench step (1 GPU)
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-v1"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-3} -c ${C:-1} -o gpurun_out/prof_k $B > gpurun_out/ncu_k.log 2>&1
echo done
