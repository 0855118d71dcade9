UM_GEMM_PAIRS=4 UM_GEMM_PAIRS_FIXED=1 timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog|rror" | head -5 | sed "s/^/[np4 fixed probe] /"
for E in "UM_GEMM_PAIRS=4 UM_GEMM_PAIRS_FIXED=1" "UM_GEMM_PAIRS=2 UM_GEMM_PAIRS_FIXED=1" "UM_GEMM_PAIRS=1"; do
env $E UM_GEMM_STALLS=1 timeout 90 python tools/profile_gemm.py --time --iters 12 2>&1 | grep -E "max resident|pairs|TFLOP" | sort | uniq -c | head -4 | sed "s/^/[$E] /"
done
for E in "UM_GEMM_PAIRS=4 UM_GEMM_PAIRS_FIXED=1" "UM_GEMM_PAIRS=1" "UM_GEMM_PAIRS=4 UM_GEMM_PAIRS_FIXED=1" "UM_GEMM_PAIRS=1"; do
env $E timeout 90 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | sed "s/^/[$E long] /"
done
