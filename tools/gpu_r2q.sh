mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    tools/dist_check.py > gpurun_out/r2q_dist_check_p2.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_dist_check_p2.log
DNDC_PERSIST_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 tools/persist_trace.py > gpurun_out/r2q_trace_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 20 --warmup 5 --no-configs --no-cdist > gpurun_out/r2q_bench_n2.json 2> gpurun_out/r2q_bench_n2.err
timeout 600 python tools/cdist_ab.py variants/STOREONLY.so > gpurun_out/r2q_cdist_ab.log 2>&1
timeout 300 python tools/write_bw.py > gpurun_out/r2q_write_bw.log 2>&1
