mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q -s > gpurun_out/r2b_cluster.log 2>&1; echo rc=$? >> gpurun_out/r2b_cluster.log
for v in "" s4b2 0; do
  DNDC_PERSIST=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/r2b_bench_$v.json 2> gpurun_out/r2b_bench_$v.err; echo "rc=$?" >> gpurun_out/r2b_bench_$v.err
done
timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg1 or cfg4" tests/test_gpu_pairwise.py -m gpu -q -s > gpurun_out/r2b_cfg.log 2>&1; echo rc=$? >> gpurun_out/r2b_cfg.log
