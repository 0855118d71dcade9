timeout 900 python -m pytest tests/test_runtime_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for X in True False; do UM_MATRIX_SOLO=0 timeout 900 python tools/bench_matrix.py --configs cfg3,cfg4,cfg5 --ps 2,4,8 --set share_sms=$X 2>&1 | grep -v CUDAEvent.h | sed "s/^/[share=$X] /"; done
