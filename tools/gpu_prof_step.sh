# One N=1 bench line (clock sampler check) and a warm-cache, in-order ncu launch
# list of two eager train steps of the bench workload.
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -3 gpurun_out/bench_n1.err; cut -c1-300 gpurun_out/bench_n1.json; python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['clocks'], d['roofline']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -c 2000 --csv --log-file gpurun_out/step_launches.csv python tools/step_once.py 2 > gpurun_out/ncu_step.log 2>&1; tail -2 gpurun_out/ncu_step.log
