mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/cfg3_change_stats.py > gpurun_out/r2d3_stats.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_refine -s 25 -c 1 -o gpurun_out/r2d3_refine python tools/prof_cfg3.py > gpurun_out/r2d3_ncu4.log 2>&1
cp paper_2007_13552_b200/libdndc_trace.so paper_2007_13552_b200/libdndc.so
timeout 300 python tools/tcd_trace.py > gpurun_out/r2d3_trace.log 2>&1
