# ncu --set full of the hot kernels of the last bench step (1 GPU): skip the 3 warm-up steps.
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_(render_bwd|render_fwd|radix_pass|gauss_bwd|project|densify_decide|densify_apply|duplicate|compact)" -s 39 -c 13 -o gpurun_out/prof_full $B > gpurun_out/ncu_full.log 2>&1
echo done
