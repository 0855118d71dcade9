UM_GEMM_STAGGER=1 timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[stagger1 probe] /"
for SG in 0 1 2 0 1 2; do
  UM_GEMM_STALLS=1 UM_GEMM_STAGGER=$SG timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[sg=$SG] /"
  UM_GEMM_STAGGER=$SG timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1 | sed "s/^/[sg=$SG] /"
done
