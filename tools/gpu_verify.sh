# Round-end style verification: GPU tests, smoke, bench N=1 (+ reference arm), bench N=2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -3 gpurun_out/bench_n1.err; cat gpurun_out/bench_n1.json | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err; tail -3 gpurun_out/ref_n1.err; cat gpurun_out/ref_n1.json | cut -c1-600
