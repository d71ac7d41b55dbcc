set -x
timeout 600 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/bench_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 48 -c 16 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(render_bwd|render_fwd|gauss_bwd|radix_pass|project|densify_decide)" -s 20 -c 8 -o gpurun_out/prof1 $B > gpurun_out/ncu_full.log 2>&1
echo done
