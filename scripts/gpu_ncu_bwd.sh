# ncu --set full on one k_render_bwd launch of a bench step (1 GPU)
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_render_bwd" -s 3 -c 1 -o gpurun_out/prof_bwd $B > gpurun_out/ncu_bwd.log 2>&1
echo done
