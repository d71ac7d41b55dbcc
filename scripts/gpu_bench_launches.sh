# Default bench line + the ncu launch list of one step (1 GPU); results under gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
bash scripts/gpu_launches.sh
