B=$PWD/tools/debug/lib_base.so
P=$PWD/paper_2510_08874_b200/_lib/libunimul_b200_prof.so
rm -f gpurun_out/s3_ab2.log
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2 >> gpurun_out/s3_ab2.log
for S in 8192x8192x8192 16384x16384x16384 4096x4096x4096; do
 for r in 1 2; do
  UNIMUL_B200_LIB=$B timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1,lt 2>&1 | sed "s/^/base_$S /" >> gpurun_out/s3_ab2.log
  timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/new_$S /" >> gpurun_out/s3_ab2.log
 done
done
UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=1 UM_GEMM_EPI_DEBUG=none timeout 300 python tools/k1_series.py --shape 8192x8192x8192 --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/mma1ne /" >> gpurun_out/s3_ab2.log
UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=1 timeout 300 python tools/k1_series.py --shape 8192x8192x8192 --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/mma1 /" >> gpurun_out/s3_ab2.log
UNIMUL_B200_LIB=$P timeout 300 python tools/k1_series.py --shape 8192x8192x8192 --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/prof /" >> gpurun_out/s3_ab2.log
UM_GEMM_STALLS=1 timeout 300 python tools/k1_timeline.py 8192 8192 8192 2>&1 | grep -v timeline | tail -2 >> gpurun_out/s3_ab2.log
