mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kmeans_tcd -s 10 -c 1 -o gpurun_out/r2n3_tcd python tools/prof_cfg3.py > gpurun_out/r2n3_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_refine -s 10 -c 1 -o gpurun_out/r2n3_refine python tools/prof_cfg3.py > gpurun_out/r2n3_ncu2.log 2>&1
cp paper_2007_13552_b200/libdndc_trace.so paper_2007_13552_b200/libdndc.so
timeout 300 python tools/tcd_trace.py > gpurun_out/r2n3_trace.log 2>&1
