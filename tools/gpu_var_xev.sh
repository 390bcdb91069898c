#!/bin/bash
# default library vs variants/*.so: cfg3 shard fit time and the cfg1 bench line (one process each).
OUT=gpurun_out
: > $OUT/var_xev.txt
for rep in 1 2; do
for lib in paper_2007_13552_b200/libdndc.so variants/*.so; do
  echo "== $lib" >> $OUT/var_xev.txt
  DNDC_LIB_PATH=$lib timeout 300 python tools/time_cfg3.py >> $OUT/var_xev.txt 2>&1
  DNDC_LIB_PATH=$lib timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-cdist --no-configs 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.readline());r=d['roofline'];print('cfg1',round(d['value']),round(r['frac'],4),r['avg_launch_ms'])" >> $OUT/var_xev.txt
done
done
cat $OUT/var_xev.txt
