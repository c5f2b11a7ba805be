mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm --format=csv,noheader
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tests/multi/nccl_parity.py > gpurun_out/parity4.log 2>&1; grep "nccl parity\|FAIL" gpurun_out/parity4.log | head -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; grep -i error gpurun_out/bench_n4.err | tail -2; tail -1 gpurun_out/bench_n4.json | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --workload moe > gpurun_out/moe_n4.json 2> gpurun_out/moe_n4.err; grep -i error gpurun_out/moe_n4.err | tail -2; tail -1 gpurun_out/moe_n4.json | cut -c1-300
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 bench.py --gpus 4 --impl reference > gpurun_out/ref_n4.json 2> gpurun_out/ref_n4.err; tail -1 gpurun_out/ref_n4.json | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 tools/coll_bench.py --json gpurun_out/coll4.json > gpurun_out/coll4.log 2>&1; tail -3 gpurun_out/coll4.log
