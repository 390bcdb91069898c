mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tcd_kernel -s 5 -c 1 -o gpurun_out/r2y2_tcd python tools/prof_cfg3.py > gpurun_out/r2y2_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_refine -s 25 -c 1 -o gpurun_out/r2y2_refine python tools/prof_cfg3.py > gpurun_out/r2y2_ncu4.log 2>&1
