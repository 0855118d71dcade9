timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t34.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t34.log
for X in 1 0; do echo "== chain=$X"
UM_GEMM_CHAIN=$X timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -2
UM_GEMM_CHAIN=$X timeout 120 python tools/solo_probe.py cfg5 8 kernel same_device_gets=direct 2>&1 | grep -v CUDAEvent.h | tail -2
UM_GEMM_CHAIN=$X timeout 120 python tools/solo_probe.py cfg5 4 kernel 2>&1 | grep -v CUDAEvent.h | tail -2
UM_GEMM_CHAIN=$X UM_MATRIX_SOLO=0 timeout 300 python tools/bench_matrix.py --configs cfg1,cfg5 --ps 4,8 2>&1 | grep -v CUDAEvent.h
done
