# A/B timing of paper_2007_13552_b200/libdndc.so vs libdndc_var.so on the cfg3 shard
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
TAG=${TAG:-ab}
timeout 300 python tools/time_cfg3.py > gpurun_out/${TAG}_a.log 2>&1
timeout 300 python -m pytest tests/test_gpu_configs.py -k "cfg3_slice_matches" -m gpu -x -q >> gpurun_out/${TAG}_a.log 2>&1
cp paper_2007_13552_b200/libdndc.so /tmp/liba.so
cp paper_2007_13552_b200/libdndc_var.so paper_2007_13552_b200/libdndc.so
timeout 300 python tools/time_cfg3.py > gpurun_out/${TAG}_b.log 2>&1
timeout 300 python -m pytest tests/test_gpu_configs.py -k "cfg3_slice_matches" -m gpu -x -q >> gpurun_out/${TAG}_b.log 2>&1
cp /tmp/liba.so paper_2007_13552_b200/libdndc.so
timeout 300 python tools/time_cfg3.py >> gpurun_out/${TAG}_a.log 2>&1
