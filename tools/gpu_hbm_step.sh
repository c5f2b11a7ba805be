# Per-kernel DRAM bytes and duration of two eager train steps (BERT and the
# MoE stack), caches flushed before each kernel (ncu default): achieved HBM
# GB/s of the elementwise / layout / SGD kernels and DRAM traffic of the GEMMs.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size
python tools/step_once.py 1 > /dev/null
timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -c 2000 --csv --log-file gpurun_out/hbm_bert.csv python tools/step_once.py 2 > gpurun_out/hbm_bert.log 2>&1; tail -2 gpurun_out/hbm_bert.log
HAP_PROFILE_WORKLOAD=moe timeout 900 ncu --metrics $M --clock-control none --profile-from-start off -c 2000 --csv --log-file gpurun_out/hbm_moe.csv python tools/step_once.py 2 > gpurun_out/hbm_moe.log 2>&1; tail -2 gpurun_out/hbm_moe.log
