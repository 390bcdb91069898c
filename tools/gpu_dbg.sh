mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_configs.py -k "delta_equals_full" -m gpu -x -q > gpurun_out/dbg1.log 2>&1
DNDC_TC_NO_DELTA=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/time_cfg3.py > gpurun_out/dbg2.log 2>&1
DNDC_TC_NO_DELTA=1 timeout 300 python -c "
import paper_2007_13552_b200.api as dnd
comm = dnd.Communicator(0)
for n in (5_000_000, 20_001, 6_250_000):
    x = dnd.random_uniform((n, 64), 0, 42, comm)
    m = dnd.kmeans_fit(x, 64, 3, 0.0, 42)
    print(n, 'ok', m.refined_rows, flush=True)
" > gpurun_out/dbg3.log 2>&1
