O=gpurun_out/v11
mkdir -p $O
timeout 300 python tests/multi/peer_ranks.py matmul_unary.hetero2 --dtypes bf16 --variants all_reduce --world 2 --verbose > $O/peer_case.log 2>&1; echo "peer case rc=$?" >> $O/status.txt
timeout 1500 python tools/tune_table.py --out $O/tune_b200.txt > $O/tune.log 2>&1; echo "tune rc=$?" >> $O/status.txt
