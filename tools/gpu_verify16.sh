O=gpurun_out/v16
mkdir -p $O
HAP_PROFILE_WORKLOAD=vitmoe2 timeout 600 python tools/op_profile.py > $O/vitmoe2_ops.log 2>&1; echo "ops rc=$?" >> $O/status.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
for w in bert moe vitmoe; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/status.txt
done
