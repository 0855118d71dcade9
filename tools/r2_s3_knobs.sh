rm -f gpurun_out/s3_knobs.log
for S in 8192x8192x8192 16384x16384x16384 65536x8192x8192; do
 for r in 1 2; do
 for kv in "X=0" "UM_GEMM_APOL=0,UM_GEMM_BPOL=0" "UM_GEMM_GROUP=-8" "UM_GEMM_GROUP=-2" "UM_GEMM_GROUP=8" "UM_GEMM_STAGGER=2" "UM_GEMM_CPOL=1"; do
  env $(echo $kv | tr ',' ' ') timeout 300 python tools/k1_series.py --shape $S --iters 15 --blocks 1 --impls k1 2>&1 | sed "s/^/${kv}_$S /" >> gpurun_out/s3_knobs.log
 done
 done
done
