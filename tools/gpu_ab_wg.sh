mkdir -p gpurun_out
for v in 0 1; do
HAP_WGRAD_STREAM=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/wg$v.json 2> gpurun_out/wg$v.err; grep "side stream" gpurun_out/wg$v.err; python -c "import json;d=json.load(open('gpurun_out/wg$v.json'));r=d['roofline'];print('wg=$v', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], r['gemm_ms_per_step'])"
done
HAP_WGRAD_STREAM=1 timeout 600 python bench.py --workload moe --no-cpu-baseline > gpurun_out/moe_wg1.json 2> gpurun_out/moe_wg1.err; python -c "import json;d=json.load(open('gpurun_out/moe_wg1.json'));print('moe wg1', d['value'], d['ms_per_step'])"
timeout 900 python -m pytest tests -m gpu -x -q -k "executor or smoke" 2>&1 | tail -2
timeout 300 python tools/gemm_bench.py --sweep --json gpurun_out/gemm_sweep.json
