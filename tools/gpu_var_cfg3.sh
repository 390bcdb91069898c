#!/bin/bash
# cfg3 shard fit time for the default library and variants/*.so (one process each).
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/var_cfg3.txt
for lib in paper_2007_13552_b200/libdndc.so variants/*.so; do
  echo "== $lib" >> $OUT/var_cfg3.txt
  DNDC_LIB_PATH=$lib timeout 300 python tools/time_cfg3.py >> $OUT/var_cfg3.txt 2>&1
  DNDC_LIB_PATH=$lib timeout 300 python tools/time_cfg3.py >> $OUT/var_cfg3.txt 2>&1
done
cat $OUT/var_cfg3.txt
