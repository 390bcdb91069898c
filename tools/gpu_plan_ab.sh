#!/bin/bash
# N-GPU bench with (DNDC_PLAN_AGREE=1) and without the per-fit plan agreement
# (a host-synchronised allgather; profiles/r02_plan_agreement_ab_n4.txt was taken
# with the experiment's original switch, noplan=1 meaning no agreement).
N=${1:-2}
OUT=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
: > $OUT/plan_ab.txt
for v in 0 1 0 1; do
  if [ $v = 0 ]; then export DNDC_PLAN_AGREE=1; else unset DNDC_PLAN_AGREE; fi
  timeout 600 $TR --master-port 2953$v bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline --no-cdist --no-configs 2>/dev/null | grep '^{' | python -c "
import json,sys;d=json.loads(sys.stdin.readline());r=d['roofline'];print('noplan=$v',round(d['value']),d['ms_per_step'],r['avg_launch_ms'])" >> $OUT/plan_ab.txt
done
cat $OUT/plan_ab.txt
