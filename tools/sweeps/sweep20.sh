timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -2
timeout 120 python tools/solo_probe.py cfg5 8 kernel same_device_gets=direct 2>&1 | grep -v CUDAEvent.h | tail -2
timeout 120 python tools/solo_probe.py cfg4 8 kernel same_device_gets=direct 2>&1 | grep -v CUDAEvent.h | tail -2
for G in -4 -8 -2 -16 8; do UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1; done
for G in -4 -8 -2 -16 8; do UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 30 --m 16384 --n 16384 --k 16384 2>&1 | tail -1; done
for G in -4 -8; do UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1; done
