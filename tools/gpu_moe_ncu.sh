export HAP_PROFILE_WORKLOAD=moe
python tools/step_once.py 1 > /dev/null
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -c 200 --csv --log-file gpurun_out/moe_launches_split.csv python tools/step_once.py 1 > /dev/null 2>&1
HAP_GEMM_SPLIT_BF16=0 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -c 200 --csv --log-file gpurun_out/moe_launches_nosplit.csv python tools/step_once.py 1 > /dev/null 2>&1
ls -la gpurun_out/
