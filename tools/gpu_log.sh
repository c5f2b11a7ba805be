HAP_GEMM_LOG=1 timeout 300 python tools/step_once.py 1 2>&1 | grep "hap gemm" | sort | uniq -c | sort -rn | head -40
