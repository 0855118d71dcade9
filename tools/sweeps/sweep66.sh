# L2 policy combos across shapes: short + long timing
for SHAPE in "" "--m 16384 --n 16384 --k 16384" "--m 8192 --n 8192 --k 65536"; do
for R in 1 2; do
for E in "UM_GEMM_APOL=0" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2 UM_GEMM_CPOL=1"; do
  env $E timeout 90 python tools/profile_gemm.py --time --iters 12 $SHAPE 2>&1 | tail -1 | sed "s/^/[$E short] /"
done; done
for E in "UM_GEMM_APOL=0" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2 UM_GEMM_CPOL=1"; do
  env $E timeout 90 python tools/profile_gemm.py --time --iters 100 $SHAPE 2>&1 | tail -1 | sed "s/^/[$E long] /"
done; done
