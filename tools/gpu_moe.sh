set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "sufficient or cuda_graph" 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/multi/nccl_parity.py moe 2>&1 | tail -15
timeout 300 python bench.py --workload moe --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/moe_n1.json 2> gpurun_out/moe_n1.err; tail -3 gpurun_out/moe_n1.err; cat gpurun_out/moe_n1.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload moe --gpus 2 --steps 20 --warmup 5 > gpurun_out/moe_n2.json 2> gpurun_out/moe_n2.err; tail -3 gpurun_out/moe_n2.err; cat gpurun_out/moe_n2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bert_n2.json 2> gpurun_out/bert_n2.err; tail -3 gpurun_out/bert_n2.err; cat gpurun_out/bert_n2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tools/coll_bench.py --rows 8,64,512,2048,4096,16384 --reps 50 --json gpurun_out/coll_small_2.json 2>&1 | tail -20
