timeout 900 python -m pytest tests/test_bounded_gpu.py tests/test_reduce_modes_gpu.py tests/test_execute_gpu.py -q -rs -s > gpurun_out/r2_t5.log 2>&1
tail -5 gpurun_out/r2_t5.log
