timeout 600 python -m pytest tests/test_runtime_gpu.py -k "captured" -x -q -p no:cacheprovider 2>&1 | tail -2
UM_MATRIX_SOLO=0 timeout 300 python tools/bench_matrix.py --configs cfg1 2>&1 | grep -v CUDAEvent
UM_MATRIX_SOLO=0 UM_MATRIX_GRAPH=1 timeout 300 python tools/bench_matrix.py --configs cfg1,cfg5 2>&1 | grep -v CUDAEvent
