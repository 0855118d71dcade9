B=$PWD/tools/debug/lib_base.so
rm -f gpurun_out/s3_ab3.log
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py tests/test_gemm_variants_gpu.py -x -q 2>&1 | tail -3 >> gpurun_out/s3_ab3.log
for S in 8192x8192x8192 16384x16384x16384 4096x4096x4096 65536x8192x8192; do
 for r in 1 2; do
  UNIMUL_B200_LIB=$B timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1,lt 2>&1 | sed "s/^/base_$S /" >> gpurun_out/s3_ab3.log
  timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/new_$S /" >> gpurun_out/s3_ab3.log
 done
done
UM_GEMM_STALLS=1 timeout 300 python tools/k1_timeline.py 8192 8192 8192 2>&1 | grep -v timeline | tail -2 >> gpurun_out/s3_ab3.log
