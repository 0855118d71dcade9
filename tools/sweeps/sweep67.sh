for R in 1 2; do
for E in "UM_GEMM_APOL=0 UM_GEMM_BPOL=0" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2" "UM_GEMM_APOL=0 UM_GEMM_BPOL=2"; do
  env $E timeout 300 python tools/bench_matrix.py --configs cfg5,cfg4 --ps 8 --steps 3 --warmup 1 2>&1 | grep -A1 "st=c" | sed "s/^/[$E] /" | cut -c1-160
done; done
