timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 600 python tools/bench_matrix.py --configs cfg2,cfg3,cfg4,cfg5 --ps 1,8 --steps 3 --warmup 1 2>&1 | grep "st=c" | cut -c1-120
timeout 600 python bench.py 2>/dev/null | tail -1 | cut -c1-400
