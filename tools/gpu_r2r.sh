mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
    tools/dist_check.py > gpurun_out/r2r_dist_check_p4.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_dist_check_p4.log
DNDC_P2P=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 \
    tools/dist_check.py > gpurun_out/r2r_dist_check_p4_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_dist_check_p4_nccl.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 \
    bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2r_bench_n4.json 2> gpurun_out/r2r_bench_n4.err
DNDC_PERSIST_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 tools/persist_trace.py > gpurun_out/r2r_trace_n4.log 2>&1
