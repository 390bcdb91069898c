mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_kernel -s 25 -c 1 -o gpurun_out/r2v_cfg3_delta python tools/prof_cfg3.py > gpurun_out/r2v_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_kernel -s 20 -c 1 -o gpurun_out/r2v_cfg3_full python tools/prof_cfg3.py > gpurun_out/r2v_ncu3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tc_refine -s 25 -c 1 -o gpurun_out/r2v_cfg3_refine python tools/prof_cfg3.py > gpurun_out/r2v_ncu4.log 2>&1
