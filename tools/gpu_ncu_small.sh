python tools/gemm_one.py 256 768 3072 0 0 bf16 5
ncu --set full --import-source on --clock-control none -k regex:gemm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/small_split -f python tools/gemm_one.py 256 768 3072 0 0 bf16 5 > /dev/null 2>&1
HAP_GEMM_SPLIT_BF16=0 ncu --set full --import-source on --clock-control none -k regex:gemm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/small_nosplit -f python tools/gemm_one.py 256 768 3072 0 0 bf16 5 > /dev/null 2>&1
ls -la gpurun_out
