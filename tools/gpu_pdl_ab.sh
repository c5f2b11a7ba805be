mkdir -p gpurun_out
for v in 0 1; do
HAP_PDL=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/pdl$v.json 2> gpurun_out/pdl$v.err; python -c "import json;d=json.load(open('gpurun_out/pdl$v.json'));r=d['roofline'];print('pdl=$v bert', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], r['gemm_ms_per_step'])"
HAP_PDL=$v timeout 600 python bench.py --workload moe --no-cpu-baseline > gpurun_out/pdlm$v.json 2> gpurun_out/pdlm$v.err; python -c "import json;d=json.load(open('gpurun_out/pdlm$v.json'));r=d['roofline'];print('pdl=$v moe', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], r['gemm_ms_per_step'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --cache-control none -c 2000 --csv --log-file gpurun_out/step_launches.csv python tools/step_once.py 2 > gpurun_out/ncu_step.log 2>&1; tail -1 gpurun_out/ncu_step.log
