UM_GEMM_EPI_DEBUG=red timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[red probe] /"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters $ITERS $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS $SHAPE] /"; }
for SHAPE in "" "--m 16384 --n 16384 --k 16384"; do
for ITERS in 12 100; do
  for ENVS in "UM_GEMM_EPI_DEBUG=reduce" "UM_GEMM_EPI_DEBUG=red" "UM_GEMM_EPI_DEBUG=reduce" "UM_GEMM_EPI_DEBUG=red"; do run; done
done; done
