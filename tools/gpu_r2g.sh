mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2g_cluster.log 2>&1; echo rc=$? >> gpurun_out/r2g_cluster.log
timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg1" -m gpu -q -s > gpurun_out/r2g_cfg.log 2>&1; echo rc=$? >> gpurun_out/r2g_cfg.log
for v in r4 r2 r4s3; do
  DNDC_PERSIST_DELTA=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > gpurun_out/r2g_bench_$v.json 2> gpurun_out/r2g_bench_$v.err
  DNDC_PERSIST_DELTA=$v DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > gpurun_out/r2g_trace_$v.log 2>&1
done
