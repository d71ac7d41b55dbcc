# Round profile: plain bench (default args), ncu launch list of one step, ncu --set full of the
# hot kernels.  1 GPU.  Results under gpurun_out/ (copied to profiles/ by hand).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
lscpu | head -20 > gpurun_out/lscpu.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-v1"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_(render_bwd|render_fwd|radix_pass|gauss_bwd|project|densify_decide|densify_apply|duplicate|compact)" -s 39 -c 13 -o gpurun_out/prof_full $B > gpurun_out/ncu_full.log 2>&1
echo done
