timeout 900 python -m pytest tests/test_bounded_gpu.py tests/test_runtime_gpu.py -x -q -k "bounded or captured or balance" > gpurun_out/r2_t3.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -k "all_of_c or real_inputs" >> gpurun_out/r2_t3.log 2>&1
for mode in bf16 f32beta1; do
  timeout 300 ncu --set full --clock-control none -k regex:'nvjet|gemm|sm100|cutlass' -c 1 -o gpurun_out/r2_cublas_${mode}_8192 -f python tools/cublas_once.py 8192 8192 8192 $mode > gpurun_out/r2_ncu_cublas_$mode.log 2>&1
done
