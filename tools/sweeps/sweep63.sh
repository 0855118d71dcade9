timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_fullsize_gpu.py tests/test_capi.py tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
run() { env UM_GET_GBPS=770 $E timeout 300 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 4,8 --steps 3 --warmup 1 $S 2>&1 | grep -A1 "st=c" | sed "s/^/[$E $S] /"; }
E=""; S=""; run
