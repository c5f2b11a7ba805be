mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -2 gpurun_out/bench_n1.err; python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));r=d['roofline'];print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], r['frac'], r['frac_burst'], r['gemm_ms_per_step'], r['gemm_share_of_step'], d['cpu_baseline'])"
timeout 600 python bench.py --workload moe --no-cpu-baseline > gpurun_out/moe_n1.json 2> gpurun_out/moe_n1.err; python -c "import json;d=json.load(open('gpurun_out/moe_n1.json'));print('moe', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['gemm_share_of_step'])"
