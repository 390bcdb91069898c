mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_pairwise.py tests/test_gpu_cluster.py -m gpu -q -x > gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg3 or cfg4" -m gpu -q -s >> gpurun_out/r2o_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
timeout 600 python tools/prof_cdist4.py > gpurun_out/r2o_cdist4_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k cdist_tc_kernel -s 5 -c 1 \
    --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum \
    -o gpurun_out/prof_cdist4 python tools/prof_cdist4.py > gpurun_out/r2o_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2o_ncu.log
