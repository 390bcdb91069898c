#!/bin/bash
# Multi-GPU k-means session (gpurun --gpus N): dist_check on the NVLink path,
# the cfg1 bench at N=1 and N, and the persistent-kernel trace at N.
N=${1:-2}
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_configs.py -x -q > $OUT/sc_pytest.log 2>&1; tail -1 $OUT/sc_pytest.log
timeout 900 $TR --master-port 29521 tools/dist_check.py > $OUT/sc_dist_check_p$N.log 2>&1; echo "rc=$?" >> $OUT/sc_dist_check_p$N.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > $OUT/sc_bench_n1.json 2> $OUT/sc_bench_n1.err
timeout 900 $TR --master-port 29522 bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline --no-cdist --no-configs > $OUT/sc_bench_n$N.json 2> $OUT/sc_bench_n$N.err
DNDC_PERSIST_TRACE=1 timeout 600 $TR --master-port 29523 tools/persist_trace.py > $OUT/sc_trace_n$N.txt 2>&1
grep -c PASS $OUT/sc_dist_check_p$N.log; grep -v PASS $OUT/sc_dist_check_p$N.log | tail -5
for f in $OUT/sc_bench_n1.json $OUT/sc_bench_n$N.json; do grep '^{' $f | python -c "
import json,sys;d=json.loads(sys.stdin.readline());r=d['roofline'];print('$f',round(d['value']),d['ms_per_step'],r['avg_launch_ms'],round(r['frac'],4))"; done
grep -A25 '^iter' $OUT/sc_trace_n$N.txt | head -24
