mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tools/coll_bench.py --json gpurun_out/coll4_push.json > gpurun_out/coll4_push.log 2>&1; tail -16 gpurun_out/coll4_push.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tests/multi/nccl_parity.py > gpurun_out/parity4_push.log 2>&1; tail -5 gpurun_out/parity4_push.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -2
