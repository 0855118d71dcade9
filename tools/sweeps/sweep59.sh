for P in 2 4; do UM_GEMM_PAIRS=$P UM_GEMM_STALLS=1 timeout 90 python tools/profile_gemm.py --time --iters 3 2>&1 | grep -E "max resident|pairs" | head -3 | sed "s/^/[pairs=$P] /"; done
