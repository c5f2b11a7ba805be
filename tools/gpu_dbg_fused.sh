python tools/gemm_bench.py 2>&1 | head -6
echo nosk; HAP_GEMM_SK=0 python tools/gemm_bench.py 2>&1 | head -6
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "stream_k or fused" 2>&1 | tail -1
