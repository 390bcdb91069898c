#!/bin/bash
# A/B of the persistent cfg1 kernel: CUDA-core scores (DNDC_PERSIST_TC=0) vs
# tensor-core scores (default), plus the k-means GPU tests on the default.
set -u
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
for tc in 0 1; do
  DNDC_PERSIST_VERBOSE=1 DNDC_PERSIST_TC=$tc timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > $OUT/abp_bench_tc$tc.json 2> $OUT/abp_bench_tc$tc.err
  echo "tc=$tc rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_configs.py -x -q > $OUT/abp_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/abp_pytest.log
DNDC_PERSIST_TRACE=1 timeout 300 python tools/persist_trace.py > $OUT/abp_trace.txt 2>&1
tail -3 $OUT/abp_pytest.log
for tc in 0 1; do python -c "
import json;d=json.load(open('$OUT/abp_bench_tc$tc.json'));r=d['roofline'];print('tc=$tc',round(d['value']),r['kernel'],round(r['frac'],3),r['avg_launch_ms'],d.get('refined_rows_last_fit'))"; done
head -30 $OUT/abp_trace.txt
grep -h "\[dndc\]" $OUT/abp_bench_tc*.err | sort | uniq
