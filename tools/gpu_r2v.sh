mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
DNDC_TC_WGS=3 timeout 300 python tools/time_cfg3.py > gpurun_out/r2v_cfg3_wg3.log 2>&1
DNDC_TC_WGS=3 timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_cluster.py -m gpu -q -x > gpurun_out/r2v_tests_wg3.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests_wg3.log
DNDC_TC_WGS=3 timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg3" -m gpu -q -s >> gpurun_out/r2v_tests_wg3.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_tests_wg3.log
timeout 600 python tools/cdist_ab.py variants/STOREONLY.so variants/LINEAR.so > gpurun_out/r2v_cdist_ab.log 2>&1
