#!/bin/bash
# Final bench lines at N GPUs with the committed collective fits: every workload
# with the cost model's choices, plus BERT-MoE with each gradient sync forced.
N=${1:-2}
OUT=gpurun_out/mf$N
mkdir -p $OUT
port=29700
trun() { local t=$1; shift; port=$((port + 1)); timeout $t python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port "$@"; }
for args in "--workload bert" "--workload moe" "--workload moe --grad-sync sfb" "--workload moe --grad-sync all_reduce" "--workload vitmoe"; do
  tag=$(echo $args | tr -d '-' | tr ' ' '_')
  trun 900 bench.py --gpus $N --steps 20 --warmup 5 $args > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err
  echo "bench $args rc=$?" >> $OUT/status.txt
done
