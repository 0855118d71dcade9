# K1 epilogue warps A/B: EW=4 vs EW=8 (register-held accumulator share)
UM_GEMM_EPI_WARPS=8 timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[ew8 probe] /"
UM_GEMM_EPI_WARPS=8 timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 | sed "s/^/[ew8 tests] /"
run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters $ITERS $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS $SHAPE] /"; }
for SHAPE in "" "--m 16384 --n 16384 --k 16384" "--m 8192 --n 8192 --k 65536"; do
for ITERS in 30; do
  for ENVS in "UM_GEMM_EPI_WARPS=4" "UM_GEMM_EPI_WARPS=8" "UM_GEMM_EPI_WARPS=4" "UM_GEMM_EPI_WARPS=8" "UM_GEMM_EPI_WARPS=8 UM_GEMM_NT=256"; do run; done
done; done
