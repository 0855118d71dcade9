# raster / L2-policy sweep for K1 (NT=512): short (burst) and sustained runs
run() { env "$@" timeout 60 python tools/profile_gemm.py --time --iters $ITERS 2>&1 | tail -1 | sed "s/^/[$*] /"; }
for ITERS in 12 150; do
  echo "== iters $ITERS"
  run UM_GEMM_GROUP=16
  run UM_GEMM_GROUP=8
  run UM_GEMM_GROUP=-4
  run UM_GEMM_GROUP=-8
  run UM_GEMM_GROUP=-8 UM_GEMM_APOL=1 UM_GEMM_BPOL=2
  run UM_GEMM_GROUP=-8 UM_GEMM_APOL=1 UM_GEMM_BPOL=2 UM_GEMM_CPOL=1
  run UM_GEMM_GROUP=-4 UM_GEMM_APOL=1 UM_GEMM_BPOL=2 UM_GEMM_CPOL=1
  run UM_GEMM_GROUP=8 UM_GEMM_APOL=2 UM_GEMM_BPOL=1 UM_GEMM_CPOL=1
done
for g in -8 -4 16; do UM_GEMM_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:gemm_bf16 -c 1 python tools/profile_gemm.py --iters 1 2>/dev/null | grep -E "dram__|hit_rate" | sed "s/^/[G=$g] /"; done
