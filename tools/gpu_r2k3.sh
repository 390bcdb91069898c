mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_accum -s 0 -c 1 -o gpurun_out/r2k3_accum python tools/prof_cfg3.py > gpurun_out/r2k3_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_refine -s 10 -c 1 -o gpurun_out/r2k3_refine python tools/prof_cfg3.py > gpurun_out/r2k3_ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kmeans_tcd -s 10 -c 1 -o gpurun_out/r2k3_tcd python tools/prof_cfg3.py > gpurun_out/r2k3_ncu3.log 2>&1
