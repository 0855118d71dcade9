UM_GEMM_EPI_WARPS=8 UM_GEMM_NO_END_STAGGER=2 timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[ew8 nostagger probe] /"
for ENVS in "UM_GEMM_EPI_WARPS=4" "UM_GEMM_EPI_WARPS=8" "UM_GEMM_EPI_WARPS=8 UM_GEMM_NO_END_STAGGER=2" "UM_GEMM_EPI_WARPS=8 UM_GEMM_NO_END_STAGGER=1"; do
  env UM_GEMM_STALLS=1 $ENVS timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[$ENVS] /"
  env $ENVS timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1 | sed "s/^/[$ENVS] /"
done
for ENVS in "UM_GEMM_EPI_WARPS=4" "UM_GEMM_EPI_WARPS=8 UM_GEMM_NO_END_STAGGER=2"; do env $ENVS timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1 | sed "s/^/[$ENVS] /"; env $ENVS timeout 90 python tools/profile_gemm.py --time --iters 30 --m 16384 --n 16384 --k 16384 2>&1 | tail -1 | sed "s/^/[$ENVS] /"; done
