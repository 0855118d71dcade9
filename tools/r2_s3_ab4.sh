B=$PWD/tools/debug/lib_e2f.so
V=$PWD/paper_2510_08874_b200/_lib/libunimul_b200_var.so
rm -f gpurun_out/s3_ab4.log
for S in 8192x8192x8192 4096x4096x4096 16384x16384x16384; do
 for r in 1 2; do
  UNIMUL_B200_LIB=$B timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1,lt 2>&1 | sed "s/^/e2f_$S /" >> gpurun_out/s3_ab4.log
  timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/epi_$S /" >> gpurun_out/s3_ab4.log
  UNIMUL_B200_LIB=$V UM_GEMM_EPI_WARPS=8 timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/ew8_$S /" >> gpurun_out/s3_ab4.log
  UM_GEMM_NT=256 timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/nt256_$S /" >> gpurun_out/s3_ab4.log
 done
done
