echo "== default"; python tools/gemm_small.py
python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
python bench.py --workload moe --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
