mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -2 gpurun_out/bench_n1.err; python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], d['roofline']['gemm_ms_per_step'], d['gpu_launches'], d['cpu_baseline'])"
timeout 600 python bench.py --workload moe --no-cpu-baseline > gpurun_out/moe_n1.json 2> gpurun_out/moe_n1.err; python -c "import json;d=json.load(open('gpurun_out/moe_n1.json'));print('moe', d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout 600 python bench.py --impl reference --steps 100 --warmup 5 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err; cut -c1-300 gpurun_out/ref_n1.json
