# Multi-GPU session (gpurun --gpus N): dist_check on the NVLink and NCCL paths,
# the bench at N GPUs, and the reference unit tests (p > GPUs share GPUs).
N=${1:-2}
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    tools/dist_check.py > gpurun_out/multi_dist_check_p$N.log 2>&1; echo "rc=$?" >> gpurun_out/multi_dist_check_p$N.log
DNDC_P2P=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
    tools/dist_check.py > gpurun_out/multi_dist_check_p${N}_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/multi_dist_check_p${N}_nccl.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus $N --steps 20 --warmup 5 --no-configs > gpurun_out/multi_bench_n$N.json 2> gpurun_out/multi_bench_n$N.err; echo "rc=$?" >> gpurun_out/multi_bench_n$N.err
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-configs --no-cpu-baseline > gpurun_out/multi_bench_n1.json 2> gpurun_out/multi_bench_n1.err
timeout 900 python -m pytest tests/test_gpu_reftests.py tests/test_gpu_cpp.py -m gpu -q > gpurun_out/multi_cpp_p$N.log 2>&1; echo "rc=$?" >> gpurun_out/multi_cpp_p$N.log
# ncu of the single-GPU delta kernel (after the plain runs above)
if [ "$N" = "2" ] && [ "${NCU:-1}" = "1" ]; then
  python tools/prof_persist.py > gpurun_out/multi_plain.log 2>&1 && \
  CUDA_VISIBLE_DEVICES=0 ncu --set full --import-source on --clock-control none -k regex:kmeans_persist_kernel -s 5 -c 1 \
      -o gpurun_out/prof_persist_delta python tools/prof_persist.py > gpurun_out/multi_ncu.log 2>&1
fi
