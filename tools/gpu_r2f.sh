mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_reftests.py -m gpu -q > gpurun_out/r2f_ref.log 2>&1; echo rc=$? >> gpurun_out/r2f_ref.log
for st in 100 70 40; do
  DNDC_PERSIST_STATIC=$st DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > gpurun_out/r2f_trace_$st.log 2>&1
done
python tools/prof_persist.py > gpurun_out/r2f_plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:kmeans_persist_kernel -s 2 -c 1 -o gpurun_out/prof_persist_r2f python tools/prof_persist.py > gpurun_out/r2f_ncu.log 2>&1
