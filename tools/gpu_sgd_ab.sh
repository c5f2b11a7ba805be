# A/B of the overlapped SGD update (HAP_SGD_OVERLAP): GPU suite, then bench
# lines for both workloads with it off and on (twice each).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in bert moe; do for o in 0 1 0 1; do
  HAP_SGD_OVERLAP=$o timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ab_${w}_$o.json 2> gpurun_out/ab_${w}_$o.err
  python -c "import json;d=json.load(open('gpurun_out/ab_${w}_$o.json'));print('$w overlap=$o', d['value'], d['ms_per_step'], d['gpu_launches'], d['loss'])"
done; done
