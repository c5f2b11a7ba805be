mkdir -p gpurun_out
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/coll_bench.py --json gpurun_out/coll${N}_push.json > gpurun_out/coll${N}_push.log 2>&1; tail -16 gpurun_out/coll${N}_push.log
