run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters 30 $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS] /"; }
for SHAPE in "" "--m 8192 --n 8192 --k 65536" "--m 8192 --n 8192 --k 8192"; do
for ENVS in "UM_GEMM_EPI_WARPS=4" "UM_GEMM_EPI_WARPS=8" "UM_GEMM_EPI_WARPS=8 UM_GEMM_CPOL=1" "UM_GEMM_EPI_WARPS=8 UM_GEMM_CPOL=2" "UM_GEMM_EPI_WARPS=4" "UM_GEMM_EPI_WARPS=8"; do run; done; done
for ENVS in "UM_GEMM_EPI_WARPS=8 UM_GEMM_CPOL=1" "UM_GEMM_EPI_WARPS=8"; do UM_GEMM_STALLS=1 env $ENVS timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[$ENVS] /"; done
