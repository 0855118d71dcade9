timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
UM_GEMM_EPI_WARPS=8 timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for EW in 4 8 4 8; do UM_GEMM_STALLS=1 UM_GEMM_EPI_WARPS=$EW timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[ew=$EW] /"; done
for EW in 4 8 4 8; do UM_GEMM_EPI_WARPS=$EW timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1 | sed "s/^/[ew=$EW] /"; done
for EW in 4 8; do UM_GEMM_EPI_WARPS=$EW timeout 90 python tools/profile_gemm.py --time --iters 30 --m 16384 --n 16384 --k 16384 2>&1 | tail -1 | sed "s/^/[ew=$EW] /"; done
