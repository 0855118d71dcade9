# NP=4 adaptive (preferred cluster 8 / regular 2, B multicast over 4 pairs) correctness + A/B against NP=1
UM_GEMM_PAIRS=4 timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog|rror" | head -5 | sed "s/^/[np4 probe] /"
UM_GEMM_PAIRS=4 timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py tests/test_fullsize_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -3 | sed "s/^/[np4 tests] /"
run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters $ITERS $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS $SHAPE] /"; }
for SHAPE in "" "--m 16384 --n 16384 --k 16384"; do
for ITERS in 12 100; do
  for ENVS in "UM_GEMM_PAIRS=1" "UM_GEMM_PAIRS=4" "UM_GEMM_PAIRS=1" "UM_GEMM_PAIRS=4"; do run; done
done; done
UM_GEMM_PAIRS=4 UM_GEMM_STALLS=1 timeout 90 python tools/profile_gemm.py --time --iters 12 2>&1 | tail -4 | sed "s/^/[np4 stalls] /"
UM_GEMM_PAIRS=1 UM_GEMM_STALLS=1 timeout 90 python tools/profile_gemm.py --time --iters 12 2>&1 | tail -4 | sed "s/^/[np1 stalls] /"
