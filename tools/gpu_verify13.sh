O=gpurun_out/v13
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_peer_ranks.py::test_peer_ranks_in_one_process_match_oracle > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python tools/gemm_step_table.py --json $O/gemm_table_bert.json > $O/gemm_table_bert.log 2>&1; echo "table rc=$?" >> $O/status.txt
for w in bert moe vitmoe; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/status.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
