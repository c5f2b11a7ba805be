set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_executor.py -x -q -k "moe or mlp or bert or sufficient" 2>&1 | tail -3
timeout 300 python bench.py --workload moe --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
HAP_GEMM_SPLIT_BF16=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
