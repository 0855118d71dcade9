for shp in 8192x8192x8192 4096x4096x4096; do
  UM_GEMM_NT=256 timeout 300 python tools/k1_series.py --shape $shp --iters 30 --blocks 2 > gpurun_out/s3_nt256_$shp.log 2>&1
done
for nt in 512 256; do
  UM_GEMM_NT=$nt UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=/tmp/tl_$nt.csv timeout 300 python tools/k1_timeline.py 8192 8192 8192 > gpurun_out/s3_tl_$nt.log 2>&1
  UM_GEMM_NT=$nt UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=/tmp/tl4_$nt.csv timeout 300 python tools/k1_timeline.py 4096 4096 4096 > gpurun_out/s3_tl4_$nt.log 2>&1
done
