mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/multi/nccl_parity.py > gpurun_out/parity.log 2>&1; grep -v "^\s*$" gpurun_out/parity.log | grep -iv "warn\|OMP_NUM\|\*\*\*" | tail -8
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --workload moe > gpurun_out/moe_n2.json 2> gpurun_out/moe_n2.err; grep -i "error" gpurun_out/moe_n2.err | tail -2; python -c "import json;d=json.loads(open('gpurun_out/moe_n2.json').read().strip().splitlines()[-1]);print('moe n2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'])"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
