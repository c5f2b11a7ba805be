mkdir -p gpurun_out/v8
timeout 300 python tools/gemm_trace.py --json gpurun_out/v8/trace.json > gpurun_out/v8/trace.log 2>&1; echo "trace rc=$?" >> gpurun_out/v8/status.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_peer_ranks.py::test_peer_ranks_in_one_process_match_oracle > gpurun_out/v8/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v8/status.txt
timeout 300 python tools/gemm_step_table.py --json gpurun_out/v8/gemm_table_bert.json > gpurun_out/v8/gemm_table_bert.log 2>&1; echo "table rc=$?" >> gpurun_out/v8/status.txt
timeout 600 python bench.py > gpurun_out/v8/bench.json 2> gpurun_out/v8/bench.err; echo "bench rc=$?" >> gpurun_out/v8/status.txt
timeout 600 python bench.py --workload moe > gpurun_out/v8/bench_moe.json 2> gpurun_out/v8/bench_moe.err; echo "bench moe rc=$?" >> gpurun_out/v8/status.txt
timeout 600 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v8/peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/v8/status.txt
