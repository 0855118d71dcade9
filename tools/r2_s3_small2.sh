rm -f gpurun_out/s3_small2.log
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py tests/test_gemm_variants_gpu.py tests/test_execute_gpu.py -x -q 2>&1 | tail -3 >> gpurun_out/s3_small2.log
timeout 300 python tools/debug/launch_probe.py >> gpurun_out/s3_small2.log 2>&1
for s in 256 1024 2048; do
  UM_GEMM_STALLS=1 timeout 120 python tools/k1_timeline.py $s $s $s 2>&1 | grep "block 0 timeline" | tail -1 | sed "s/^/$s: /" >> gpurun_out/s3_small2.log
done
for S in 8192x8192x8192 4096x4096x4096 2048x2048x4096; do
  UNIMUL_B200_LIB=$PWD/tools/debug/lib_e2f.so timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1,lt 2>&1 | sed "s/^/e2f_$S /" >> gpurun_out/s3_small2.log
  timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/new_$S /" >> gpurun_out/s3_small2.log
done
