#!/bin/bash
# cfg2 cdist time: the default library and variants/*.so (tools/cdist_ab.py), twice.
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python tools/cdist_ab.py variants/*.so > $OUT/var_cdist.txt 2>&1
timeout 900 python tools/cdist_ab.py variants/*.so >> $OUT/var_cdist.txt 2>&1
cat $OUT/var_cdist.txt
