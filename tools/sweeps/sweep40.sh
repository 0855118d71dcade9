UM_GET_GBPS=770 timeout 1500 python tools/bench_matrix.py --configs cfg2,cfg3,cfg4,cfg5 --ps 2,4,8 --json gpurun_out/matrix_paced.json 2>&1 | grep -v CUDAEvent.h | grep -v "^cfg"
