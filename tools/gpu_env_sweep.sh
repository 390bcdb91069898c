#!/bin/bash
# Env sweep of the persistent cfg1 fit (each a short bench run): full-iteration
# count, static tile share, and the tensor-core score variant.
set -u
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
: > $OUT/sweep.txt
run() {
  env "$@" timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > $OUT/sweep_one.json 2>/dev/null
  python -c "
import json,sys;d=json.load(open('$OUT/sweep_one.json'));r=d['roofline'];print(sys.argv[1:], round(d['value']),round(r['frac'],4),round(r['avg_launch_ms'],4),d['ms_per_step'],d.get('refined_rows_last_fit'))" "$@" >> $OUT/sweep.txt 2>&1
}
run X=0
run DNDC_FULL_ITERS=1
run DNDC_FULL_ITERS=3
run DNDC_PERSIST_STATIC=50
run DNDC_PERSIST_STATIC=85
run DNDC_PERSIST_STATIC=100
run DNDC_PERSIST_TC=1
run X=0
cat $OUT/sweep.txt
