mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_cluster.py -m gpu -q -x > gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg3" -m gpu -q -s >> gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
timeout 600 python tools/prof_cfg3.py > gpurun_out/r2s_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k kmeans_tc_kernel -s 25 -c 1 -o gpurun_out/prof_cfg3_r2s python tools/prof_cfg3.py > gpurun_out/r2s_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2s_ncu.log
