P=$PWD/paper_2510_08874_b200/_lib/libunimul_b200_prof.so
S=8192x8192x8192
run() { tag=$1; shift; env "$@" timeout 300 python tools/k1_series.py --shape $S --iters 30 --blocks 2 --impls k1 2>&1 | sed "s/^/$tag /" >> gpurun_out/s3_ab.log; }
rm -f gpurun_out/s3_ab.log
timeout 300 python tools/k1_series.py --shape $S --iters 30 --blocks 2 2>&1 | sed "s/^/base /" >> gpurun_out/s3_ab.log
run prof UNIMUL_B200_LIB=$P
run noepi UNIMUL_B200_LIB=$P UM_GEMM_EPI_DEBUG=none
run store UNIMUL_B200_LIB=$P UM_GEMM_EPI_DEBUG=store
run nohint UM_GEMM_APOL=0 UM_GEMM_BPOL=0
run gm8 UM_GEMM_GROUP=-8
run g8 UM_GEMM_GROUP=8
run g2 UM_GEMM_GROUP=2
run nt256 UM_GEMM_NT=256
run static UM_GEMM_STATIC=1
run halfb UNIMUL_B200_LIB=$P UM_GEMM_DEBUG_HALFB=1
