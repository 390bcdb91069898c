mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_moments.py tests/test_gpu_pairwise.py -m gpu -x -q > gpurun_out/r2z_tests.log 2>&1; echo rc=$? >> gpurun_out/r2z_tests.log
timeout 300 python tools/time_cfg3.py > gpurun_out/r2z_cfg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2z_cfg3_launches.csv python tools/prof_cfg3.py > gpurun_out/r2z_ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_kernel -s 25 -c 1 -o gpurun_out/r2z_cfg3_delta python tools/prof_cfg3.py > gpurun_out/r2z_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_kernel -s 20 -c 1 -o gpurun_out/r2z_cfg3_full python tools/prof_cfg3.py > gpurun_out/r2z_ncu3.log 2>&1
