mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2e_cluster.log 2>&1; echo rc=$? >> gpurun_out/r2e_cluster.log
timeout 900 python -m pytest tests/test_gpu_reftests.py tests/test_gpu_cpp.py -m gpu -q -s > gpurun_out/r2e_cpp.log 2>&1; echo rc=$? >> gpurun_out/r2e_cpp.log
python tools/prof_persist.py > gpurun_out/r2e_plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:persist -s 2 -c 1 -o gpurun_out/prof_persist_r2e python tools/prof_persist.py > gpurun_out/r2e_ncu.log 2>&1
