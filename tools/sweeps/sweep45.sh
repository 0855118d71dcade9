for E in reduce store none reduce store none; do UM_GEMM_EPI_DEBUG=$E timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1; done
for E in reduce store none; do UM_GEMM_EPI_DEBUG=$E timeout 90 python tools/profile_gemm.py --time --iters 30 --m 16384 --n 16384 --k 16384 2>&1 | tail -1; done
