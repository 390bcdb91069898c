mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
DNDC_LIB_PATH=variants/CHECKS.so timeout 600 python tools/sanitize_smoke.py > gpurun_out/r2n_checks.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_checks.log
DNDC_LIB_PATH=variants/CHECKS.so timeout 600 python tools/prof_persist.py >> gpurun_out/r2n_checks.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_checks.log
timeout 600 python tools/prof_cdist4.py > gpurun_out/r2n_cdist4_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"cdist_tc_kernel<2" -s 1 -c 1 \
    --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active \
    -o gpurun_out/prof_cdist4 python tools/prof_cdist4.py > gpurun_out/r2n_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2n_ncu.log
