mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_cluster.py -m gpu -x -q > gpurun_out/r2i_tests.log 2>&1; echo rc=$? >> gpurun_out/r2i_tests.log
for lib in paper_2007_13552_b200/libdndc.so variants/STREAM.so variants/NOACC.so; do
  echo "== $lib" >> gpurun_out/r2i_ab.log
  DNDC_LIB_PATH=$lib DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py >> gpurun_out/r2i_ab.log 2>&1
done
