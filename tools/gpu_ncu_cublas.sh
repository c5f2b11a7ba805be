mkdir -p gpurun_out
# cuBLAS vs ours on the bench shapes: kernel names (tile configs) and tensor-pipe activity
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -c 400 --csv --log-file gpurun_out/cublas_cmp.csv python tools/gemm_bench.py > gpurun_out/cublas_cmp.log 2>&1; tail -1 gpurun_out/cublas_cmp.log
HAP_AUTOTUNE=0 timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -c 2000 --csv --log-file gpurun_out/step_launches.csv python tools/step_once.py 2 > gpurun_out/ncu_step.log 2>&1; tail -1 gpurun_out/ncu_step.log
