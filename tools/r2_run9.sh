timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gemm_variants_gpu.py -q -s -x > gpurun_out/r2_t9.log 2>&1
timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x -k "copy_engine_pulls" >> gpurun_out/r2_t9.log 2>&1
grep -E "passed|failed|same-device" gpurun_out/r2_t9.log
