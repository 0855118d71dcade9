for E in reduce none store; do UM_GEMM_STALLS=1 UM_GEMM_EPI_DEBUG=$E timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[$E cfg2] /"; done
UM_GEMM_STALLS=1 timeout 90 python tools/profile_gemm.py --iters 3 --m 16384 --n 16384 --k 16384 2>&1 | grep stalls | tail -1 | sed "s/^/[16384^3] /"
UM_GEMM_STALLS=1 timeout 90 python tools/profile_gemm.py --iters 3 --m 8192 --n 8192 --k 65536 2>&1 | grep stalls | tail -1 | sed "s/^/[cfg3] /"
UM_GEMM_STALLS=1 UM_GEMM_NT=256 timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[nt256 cfg2] /"
UM_GEMM_STALLS=1 UM_GEMM_NO_END_STAGGER=1 timeout 90 python tools/profile_gemm.py --iters 3 2>&1 | grep stalls | tail -1 | sed "s/^/[no end stagger] /"
UM_GEMM_STALLS=1 timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep stalls | tail -2 | sed "s/^/[cfg5 p8 rank] /"
UM_GEMM_STALLS=1 UM_GET_GBPS=770 timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep stalls | tail -2 | sed "s/^/[cfg5 p8 rank paced] /"
