mkdir -p gpurun_out/v4
timeout 300 python tools/gemm_trace.py --json gpurun_out/v4/trace.json > gpurun_out/v4/trace.log 2>&1; echo "trace rc=$?" >> gpurun_out/v4/status.txt
timeout 900 python tests/multi/peer_ranks.py --verbose --rotate > gpurun_out/v4/peer.log 2>&1; echo "peer rc=$?" >> gpurun_out/v4/status.txt
