# ncu --set full on the two render kernels of one bench step (1 GPU)
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_render_(fwd|bwd)" -s 6 -c 2 -o gpurun_out/prof_render $B > gpurun_out/ncu_render.log 2>&1
echo done
