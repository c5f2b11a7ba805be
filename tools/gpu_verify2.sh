mkdir -p gpurun_out/v2
timeout 300 python tools/gemm_step_table.py --json gpurun_out/v2/gemm_table_bert.json > gpurun_out/v2/gemm_table_bert.log 2>&1; echo "table rc=$?" >> gpurun_out/v2/status.txt
timeout 1300 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=60 --deselect tests/test_gpu_peer_ranks.py::test_peer_ranks_in_one_process_match_oracle > gpurun_out/v2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v2/status.txt
timeout 900 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v2/peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/v2/status.txt
