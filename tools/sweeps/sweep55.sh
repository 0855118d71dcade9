for H in 0 1 0 1; do
  UM_GEMM_STALLS=1 UM_GEMM_DEBUG_HALFB=$H timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[halfb=$H] /"
  UM_GEMM_DEBUG_HALFB=$H timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1 | sed "s/^/[halfb=$H] /"
done
