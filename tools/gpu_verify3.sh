mkdir -p gpurun_out/v3
timeout 300 python tools/gemm_trace.py --json gpurun_out/v3/trace.json > gpurun_out/v3/trace.log 2>&1; echo "trace rc=$?" >> gpurun_out/v3/status.txt
timeout 600 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v3/peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/v3/status.txt
