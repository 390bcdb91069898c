mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2d_cluster.log 2>&1; echo rc=$? >> gpurun_out/r2d_cluster.log
timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg1 or cfg4" tests/test_gpu_pairwise.py -m gpu -q -s > gpurun_out/r2d_cfg.log 2>&1; echo rc=$? >> gpurun_out/r2d_cfg.log
for v in s2b4 s3b3 s4b2; do
  DNDC_PERSIST=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > gpurun_out/r2d_bench_$v.json 2> gpurun_out/r2d_bench_$v.err
  DNDC_PERSIST=$v DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > gpurun_out/r2d_trace_$v.log 2>&1
done
