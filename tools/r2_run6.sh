timeout 1200 python -m pytest tests/test_bounded_gpu.py tests/test_reduce_modes_gpu.py tests/test_execute_gpu.py tests/test_gemm_gpu.py -q -rs -s -k "not variant" > gpurun_out/r2_t6.log 2>&1
timeout 400 python -m pytest tests/test_runtime_gpu.py -q -k "copy_engine_pulls" >> gpurun_out/r2_t6.log 2>&1
tail -5 gpurun_out/r2_t6.log
