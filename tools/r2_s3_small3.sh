rm -f gpurun_out/s3_small3.log
for S in 4096x4096x4096 2048x2048x4096 8192x8192x8192; do
 for fs in 1 0; do for fd in 1 0; do
  UM_GEMM_FIRST_STATIC=$fs UM_GEMM_FAST_DRAIN=$fd timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/fs${fs}fd${fd}_$S /" >> gpurun_out/s3_small3.log
 done; done
done
for fs in 1 0; do for fd in 1 0; do
  echo "fs=$fs fd=$fd" >> gpurun_out/s3_small3.log
  UM_GEMM_FIRST_STATIC=$fs UM_GEMM_FAST_DRAIN=$fd timeout 300 python tools/debug/launch_probe.py >> gpurun_out/s3_small3.log 2>&1
done; done
