for mode in bf16 f32beta1; do
  timeout 300 ncu --set full --clock-control none -s 2 -c 1 -o gpurun_out/r2_cublas_${mode}_8192 python tools/cublas_once.py 8192 8192 8192 $mode > gpurun_out/r2_ncu_cublas_$mode.log 2>&1
done
ls gpurun_out
