mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
cp paper_2007_13552_b200/libdndc_trace.so paper_2007_13552_b200/libdndc.so
timeout 300 python tools/tcd_trace.py > gpurun_out/r2z2_trace.log 2>&1
