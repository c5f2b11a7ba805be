mkdir -p gpurun_out/v6
HAP_P2P_COOP=0 timeout 1200 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v6/peer_nocoop.log 2>&1; echo "peer nocoop rc=$?" >> gpurun_out/v6/status.txt
