mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > gpurun_out/r2c_trace.log 2>&1
for v in mma model; do
DNDC_CDTC_NORM=$v timeout 600 python -m pytest tests/test_gpu_configs.py -k "cfg4" tests/test_gpu_pairwise.py -m gpu -q -s > gpurun_out/r2c_cfg_$v.log 2>&1; echo rc=$? >> gpurun_out/r2c_cfg_$v.log
done
