# GPU tests, then one bench run (called through gpurun; writes under gpurun_out/)
timeout 600 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo exit=$? >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo exit=$? >> gpurun_out/bench.log
