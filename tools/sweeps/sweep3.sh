run() { env "$@" timeout 60 python tools/profile_gemm.py --time --iters $ITERS 2>&1 | tail -1 | sed "s/^/[$*] /"; }
dram() { env "$@" timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_ltcfabric.sum -k regex:gemm_bf16 -c 1 python tools/profile_gemm.py --iters 1 2>/dev/null | grep -E "dram__|hit_rate|fabric" | tr -s ' ' | sed "s/^/[$*] /"; }
for p in 0 2 3; do dram UM_GEMM_PROMO=$p UM_GEMM_GROUP=16; done
dram UM_GEMM_PROMO=0 UM_GEMM_GROUP=-4
dram UM_GEMM_PROMO=0 UM_GEMM_GROUP=4
for ITERS in 12 150; do for p in 0 2 3; do run UM_GEMM_PROMO=$p UM_GEMM_GROUP=16; done; done
