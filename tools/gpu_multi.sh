#!/bin/bash
# One multi-GPU session under `gpurun --gpus N`: collective latency/bandwidth
# sweeps for the cost model, NVLink hardware byte counters (NVML) around the
# peer-memory kernels, bench lines (BERT, BERT-MoE with each gradient sync, ViT-MoE with
# each collective implementation) and the NCCL-group parity run.  Outputs in
# gpurun_out/m$N/.
N=${1:-2}
STEPS=${STEPS:-20}
OUT=gpurun_out/m$N
mkdir -p $OUT
port=29500
# trun SECONDS script args...: one process per GPU under torchrun, bounded
trun() { local t=$1; shift; port=$((port + 1)); timeout $t python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port "$@"; }
nvidia-smi topo -m > $OUT/topo.txt 2>&1
trun 900 tools/coll_fit.py --json $OUT/coll_fit.json > $OUT/coll_fit.log 2>&1; echo "coll_fit rc=$?" >> $OUT/status.txt
# this box's fitted lines drive gather="auto" in the bench runs below (merged with the other world sizes locally)
python tools/coll_fit.py --fit $OUT/coll_fit.json >> $OUT/coll_fit.log 2>&1; cp paper_2401_05965_b200/collectives_b200.json $OUT/ 2>/dev/null
trun 300 tools/nvlink_ncu.py --nvml --rows 16384,65536,262144 --json $OUT/nvl_counters.json > $OUT/nvl_counters.log 2>&1; echo "nvl_counters rc=$?" >> $OUT/status.txt
HAP_P2P_COOP=1 trun 900 bench.py --gpus $N --steps $STEPS --warmup 5 --workload moe --grad-sync sfb > $OUT/bench_workload_moe_gradsync_sfb_coop.json 2> $OUT/bench_coop.err
echo "bench moe sfb (cooperative peer launches) rc=$?" >> $OUT/status.txt
# NVLink counters under ncu: the peer kernels with their cross-rank flag waits
# disabled (HAP_P2P_NOSYNC=1, results undefined), so ncu's kernel serialisation
# cannot deadlock them; only p2p_* kernels are profiled
port=$((port + 1))
HAP_P2P_NOSYNC=1 timeout 900 ncu --target-processes all -k regex:p2p_ --clock-control none --csv \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
  --log-file $OUT/nvl_ncu.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $port tools/nvlink_ncu.py --calls 2 --rows 65536,262144 > $OUT/nvl_ncu.log 2>&1; echo "nvl_ncu rc=$?" >> $OUT/status.txt
for args in "--workload bert" "--workload moe" "--workload moe --grad-sync sfb" "--workload moe --grad-sync all_reduce" \
            "--workload vitmoe" "--workload vitmoe --collectives p2p" "--workload vitmoe --collectives nccl"; do
  tag=$(echo $args | tr -d '-' | tr ' ' '_')
  trun 900 bench.py --gpus $N --steps $STEPS --warmup 5 $args > $OUT/bench_$tag.json 2> $OUT/bench_$tag.err
  echo "bench $args rc=$?" >> $OUT/status.txt
done
if [ "${PARITY:-1}" = "1" ]; then
  HAP_PARITY_VARIANTS=${PARITY_VARIANTS:-kernel:sfb,auto:all_reduce} trun 1800 tests/multi/nccl_parity.py > $OUT/parity.log 2>&1; echo "parity rc=$?" >> $OUT/status.txt
fi
