timeout 900 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/multi/nccl_parity.py 2>&1 | grep -v OMP | tail -8
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload moe --gpus 2 --steps 20 --warmup 5 2>&1 | grep metric | cut -c1-250
HAP_NO=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 2>&1 | grep metric | cut -c1-250
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tools/coll_bench.py --rows 8,512,4096,65536,262144 --reps 50 2>&1 | grep all_gather
