O=gpurun_out/v14
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
for w in bert moe vitmoe; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?" >> $O/status.txt
timeout 300 python tools/gemm_step_table.py --json $O/gemm_table_bert.json > $O/gemm_table_bert.log 2>&1; echo "table rc=$?" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_bert.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/status.txt
