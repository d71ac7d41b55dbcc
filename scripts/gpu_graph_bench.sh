cd $GRAFT_REPO_ROOT
timeout 300 python bench.py > gpurun_out/g_default.json 2> gpurun_out/g_default.err; echo "exit=$?" >> gpurun_out/g_default.err
timeout 300 python bench.py --no-graph --no-cpu-baseline > gpurun_out/g_nograph.json 2> gpurun_out/g_nograph.err
timeout 300 python bench.py --sh-degree 3 --ssim 0.2 --no-cpu-baseline > gpurun_out/g_sh.json 2> gpurun_out/g_sh.err
timeout 300 python bench.py --config C4 --budget-frac 0.1 --no-cpu-baseline > gpurun_out/g_c4b.json 2> gpurun_out/g_c4b.err
