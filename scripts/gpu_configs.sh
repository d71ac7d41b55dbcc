# Bench lines for every BASELINE config and the f3 / f2 workload variants (1 GPU); results under gpurun_out/
for C in C2 C3 C4 C5; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/cfg_$C.json 2> gpurun_out/cfg_$C.err
done
timeout 600 python bench.py --sh-degree 3 --no-cpu-baseline > gpurun_out/cfg_C2_sh3.json 2> gpurun_out/cfg_C2_sh3.err
timeout 600 python bench.py --sh-degree 3 --ssim 0.2 --no-cpu-baseline > gpurun_out/cfg_C2_sh3_ssim.json 2> gpurun_out/cfg_C2_sh3_ssim.err
timeout 600 python bench.py --config C4 --budget-frac 0.1 --no-cpu-baseline > gpurun_out/cfg_C4_budget.json 2> gpurun_out/cfg_C4_budget.err
echo done
