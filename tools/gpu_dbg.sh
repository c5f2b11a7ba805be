for i in 1 2; do
 (cd build/ab_head && python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('HEAD', d['ms_per_step'], d['roofline']['gemm_ms_per_step'])")
 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW ', d['ms_per_step'], d['roofline']['gemm_ms_per_step'])"
done
python bench.py --workload moe --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -q -x 2>&1 | tail -1
