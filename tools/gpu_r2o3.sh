mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2o3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2o3_tests.log
timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg1" -m gpu -q -s >> gpurun_out/r2o3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2o3_tests.log
DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > gpurun_out/r2o3_trace.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > gpurun_out/r2o3_bench.json 2> gpurun_out/r2o3_bench.err
