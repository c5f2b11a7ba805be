mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -2 gpurun_out/bench_n1.err; python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], d['roofline']['gemm_ms_per_step'], d['gpu_launches'])"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -c 2000 --csv --log-file gpurun_out/step_launches.csv python tools/step_once.py 2 > gpurun_out/ncu_step.log 2>&1; tail -1 gpurun_out/ncu_step.log
