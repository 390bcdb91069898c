mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
DNDC_PERSIST_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tools/persist_trace.py --rows 5000000 > gpurun_out/r2p_trace_n2.log 2>&1
