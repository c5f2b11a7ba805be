#!/bin/bash
# Short multi-GPU session: collective sweep + fit (COLL=1), the NCCL-group
# parity run, and the cost-model-chosen bench lines.  Outputs in gpurun_out/ml$N/.
N=${1:-2}
OUT=gpurun_out/ml$N
mkdir -p $OUT
port=29600
trun() { local t=$1; shift; port=$((port + 1)); timeout $t python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port "$@"; }
if [ "${COLL:-1}" = "1" ]; then
  trun 900 tools/coll_fit.py --json $OUT/coll_fit.json > $OUT/coll_fit.log 2>&1; echo "coll_fit rc=$?" >> $OUT/status.txt
  python tools/coll_fit.py --fit $OUT/coll_fit.json >> $OUT/coll_fit.log 2>&1; cp paper_2401_05965_b200/collectives_b200.json $OUT/
fi
HAP_PARITY_VARIANTS=${PARITY_VARIANTS:-kernel:sfb,auto:all_reduce} trun 1800 tests/multi/nccl_parity.py > $OUT/parity.log 2>&1; echo "parity rc=$?" >> $OUT/status.txt
for w in moe vitmoe; do
  trun 900 bench.py --gpus $N --steps 20 --warmup 5 --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo "bench $w rc=$?" >> $OUT/status.txt
done
