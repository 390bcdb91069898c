#!/bin/bash
# Delta-kernel instantiation sweep (DNDC_PERSIST_DELTA), short bench runs.
set -u
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/sweep2.txt
run() {
  env DNDC_PERSIST_VERBOSE=1 "$@" timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > $OUT/sweep_one.json 2> $OUT/sweep_one.err
  grep '\[dndc\].*delta' $OUT/sweep_one.err | head -1 >> $OUT/sweep2.txt
  python -c "
import json,sys;d=json.load(open('$OUT/sweep_one.json'));r=d['roofline'];print(sys.argv[1:], round(d['value']),round(r['frac'],4),round(r['avg_launch_ms'],4),d['ms_per_step'],d.get('refined_rows_last_fit'),d.get('final_inertia'))" "$@" >> $OUT/sweep2.txt 2>&1
}
run X=0
run DNDC_PERSIST_PAIR=1
run X=0
run DNDC_PERSIST_PAIR=1
run X=0
cat $OUT/sweep2.txt
