#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), launch list and one full
# ncu capture of the dominant kernel.  Outputs under gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/gpu_info.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" >> $OUT/bench_ref.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_small -s 12 -c 1 \
      -o $OUT/prof_assign python tools/prof_kmeans.py 5000000 18 8 20 > $OUT/ncu_full.log 2>&1
fi
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json; cat $OUT/bench_ref.json
