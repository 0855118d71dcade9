P=$PWD/paper_2510_08874_b200/_lib/libunimul_b200_prof.so
S=8192x8192x8192
run() { tag=$1; shift; env "$@" timeout 300 python tools/k1_series.py --shape $S --iters 20 --blocks 1 --impls k1 2>&1 | sed "s/^/$tag /" >> gpurun_out/s3_mma.log; }
rm -f gpurun_out/s3_mma.log
run prof UNIMUL_B200_LIB=$P
run mma1 UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=1
run mma2 UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=2
run mma1ne UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=1 UM_GEMM_EPI_DEBUG=none
run mma2ne UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=2 UM_GEMM_EPI_DEBUG=none
run mma1nt256 UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=1 UM_GEMM_NT=256
run mma2nt256 UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_MMA=2 UM_GEMM_NT=256
for e in 1 2; do
 echo "== stalls mma=$e" >> gpurun_out/s3_mma.log
 UM_GEMM_DEBUG_MMA=$e UM_GEMM_STALLS=1 timeout 300 python tools/k1_timeline.py 8192 8192 8192 2>&1 | grep -v timeline | tail -3 >> gpurun_out/s3_mma.log
done
