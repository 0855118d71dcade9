timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_fullsize_gpu.py tests/test_multiprocess_gpu.py tests/test_gemm_variants_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
UM_GEMM_TAIL_SPLIT=1 timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_fullsize_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
