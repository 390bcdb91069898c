mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_tc.py -m gpu -x -q > gpurun_out/r2p3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2p3_tests.log
timeout 900 python -m pytest tests/test_gpu_configs.py -k "cfg3 or cfg1" -m gpu -x -q >> gpurun_out/r2p3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2p3_tests.log
timeout 300 python tools/time_cfg3.py > gpurun_out/r2p3_cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r2p3_cfg3_launches.csv python tools/prof_cfg3.py > gpurun_out/r2p3_ncu1.log 2>&1
