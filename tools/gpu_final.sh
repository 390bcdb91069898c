#!/bin/bash
# Round-end GPU session (1 GPU): the whole GPU suite, smoke, both bench arms,
# the launch list of one bench step and one ncu capture of the dominant
# kernel (the persistent k-means delta launch).  Outputs under gpurun_out/final_*.
set -u
OUT=gpurun_out
mkdir -p $OUT
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $OUT/final_gpu_info.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rA > $OUT/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/final_pytest_gpu.log
for t in pairwise cluster moments; do cpp/build/ref_test_$t > $OUT/final_reftest_$t.log 2>&1; echo "rc=$?" >> $OUT/final_reftest_$t.log; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/final_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/final_smoke.log
timeout 900 python bench.py > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench rc=$?" >> $OUT/final_bench.err
timeout 900 python bench.py --impl reference > $OUT/final_bench_ref.json 2> $OUT/final_bench_ref.err; echo "ref rc=$?" >> $OUT/final_bench_ref.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > $OUT/final_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/final_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cdist --no-configs > $OUT/final_ncu_launch.log 2>&1
fi
tail -3 $OUT/final_pytest_gpu.log; tail -2 $OUT/final_smoke.log; cat $OUT/final_bench.json; cat $OUT/final_bench_ref.json
# one full ncu capture of the dominant kernel (the persistent delta launch),
# after its plain run exited 0
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 python tools/prof_persist.py > $OUT/final_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_persist_kernel -s 5 -c 1 \
      -o $OUT/final_prof_persist_delta -f python tools/prof_persist.py > $OUT/final_ncu_full.log 2>&1
  echo "ncu full rc=$?" >> $OUT/final_ncu_full.log
fi
