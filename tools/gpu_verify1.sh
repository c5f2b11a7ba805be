mkdir -p gpurun_out/v1
nvidia-smi > gpurun_out/v1/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v1/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v1/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v1/status.txt
timeout 600 python bench.py > gpurun_out/v1/bench.json 2> gpurun_out/v1/bench.err; echo "bench rc=$?" >> gpurun_out/v1/status.txt
timeout 600 python bench.py --workload moe > gpurun_out/v1/bench_moe.json 2> gpurun_out/v1/bench_moe.err; echo "bench moe rc=$?" >> gpurun_out/v1/status.txt
timeout 600 python bench.py --workload vitmoe > gpurun_out/v1/bench_vitmoe.json 2> gpurun_out/v1/bench_vitmoe.err; echo "bench vitmoe rc=$?" >> gpurun_out/v1/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/v1/bench_ref.json 2> gpurun_out/v1/bench_ref.err; echo "bench ref rc=$?" >> gpurun_out/v1/status.txt
