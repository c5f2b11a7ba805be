mkdir -p gpurun_out/v9
timeout 600 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v9/peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/v9/status.txt
HAP_P2P_COOP=0 timeout 600 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v9/peer_nocoop.log 2>&1; echo "peer nocoop rc=$?" >> gpurun_out/v9/status.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --deselect tests/test_gpu_peer_ranks.py::test_peer_ranks_in_one_process_match_oracle > gpurun_out/v9/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v9/status.txt
