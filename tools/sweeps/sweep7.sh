for v in "UM_GEMM_NT=512" "UM_GEMM_NT=256" "UM_GEMM_CG=1" "UM_GEMM_NO_END_STAGGER=1"; do env $v timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[$v] /"; done
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters $ITERS $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS $SHAPE] /"; }
for SHAPE in "" "--m 16384 --n 16384 --k 16384"; do
for ITERS in 12 100; do
  for ENVS in "UM_GEMM_NO_END_STAGGER=1" "UM_GEMM_NO_END_STAGGER=0" "UM_GEMM_NO_END_STAGGER=1" "UM_GEMM_NO_END_STAGGER=0"; do run; done
done; done
