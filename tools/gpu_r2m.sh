mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python tools/sanitize_smoke.py > gpurun_out/r2m_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/r2m_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/r2m_memcheck.log
