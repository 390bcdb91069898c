#!/bin/bash
# Quick GPU session: the GPU suite (stop at first failure) and one N=1 bench line.
set -u
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/chk_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/chk_pytest_gpu.log
timeout 600 python bench.py > $OUT/chk_bench.json 2> $OUT/chk_bench.err; echo "bench rc=$?" >> $OUT/chk_bench.err
tail -3 $OUT/chk_pytest_gpu.log; cat $OUT/chk_bench.json
