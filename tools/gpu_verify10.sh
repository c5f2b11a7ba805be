# one 1-GPU session: in-process peer test, per-launch GEMM trace, bench lines,
# the bench command's ncu launch list, GEMM DRAM traffic of one step, and one
# ncu --set full capture of the top GEMM
O=gpurun_out/v10
mkdir -p $O
timeout 1500 python tests/multi/peer_ranks.py --rotate --stride 2 --skip bf16:sfb --verbose > $O/peer.log 2>&1; echo "peer rc=$?" >> $O/status.txt
timeout 300 python tools/gemm_trace.py --json $O/trace.json > $O/trace.log 2>&1; echo "trace rc=$?" >> $O/status.txt
for w in bert moe vitmoe; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?" >> $O/status.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_bert.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/status.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control all \
  --clock-control none --profile-from-start off --csv --log-file $O/hbm_bert.csv python tools/step_once.py 2 > $O/ncu_hbm.log 2>&1; echo "ncu hbm rc=$?" >> $O/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 --launch-skip 6 --launch-count 1 \
  --profile-from-start off -o $O/gemm_full python tools/step_once.py 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/status.txt
