for NT in 0 512 256; do echo "== UM_GEMM_NT=$NT"
UM_GEMM_NT=$NT timeout 120 python tools/solo_probe.py cfg5 8 kernel same_device_gets=direct 2>&1 | grep -v CUDAEvent.h | tail -1
UM_GEMM_NT=$NT timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -1
UM_GEMM_NT=$NT timeout 120 python tools/solo_probe.py cfg1 4 kernel 2>&1 | grep -v CUDAEvent.h | tail -1
UM_GEMM_NT=$NT timeout 120 python tools/profile_gemm.py --time --iters 30 --m 8192 --n 8192 --k 8192 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
