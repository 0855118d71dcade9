timeout 600 python -m pytest tests/test_runtime_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for X in "" "chain_order=0"; do echo "== $X"
timeout 120 python tools/solo_probe.py cfg5 8 kernel $X 2>&1 | grep -v CUDAEvent.h | tail -2
timeout 120 python tools/solo_probe.py cfg5 4 kernel $X 2>&1 | grep -v CUDAEvent.h | tail -2
done
echo "== chain off in kernel"; UM_GEMM_CHAIN=0 timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -2
UM_MATRIX_SOLO=0 timeout 300 python tools/bench_matrix.py --configs cfg1,cfg5 --ps 2,4,8 2>&1 | grep -v CUDAEvent.h
