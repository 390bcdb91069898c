mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_pairwise.py -m gpu -x -q > gpurun_out/r2h_tests.log 2>&1; echo rc=$? >> gpurun_out/r2h_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
DNDC_FULL_ITERS=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > gpurun_out/r2h_bench_f1.json 2> gpurun_out/r2h_bench_f1.err
DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > gpurun_out/r2h_trace.log 2>&1
python tools/prof_persist.py > gpurun_out/r2h_plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:kmeans_persist_kernel -s 4 -c 2 -o gpurun_out/prof_persist_r2h python tools/prof_persist.py > gpurun_out/r2h_ncu.log 2>&1
