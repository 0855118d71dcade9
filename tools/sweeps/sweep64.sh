# DRAM traffic of K1 vs rasterisation group (cfg2 shape), plus timing
for G in -4 -8 -2 -16 8; do
  UM_GEMM_GROUP=$G timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_bf16 -s 2 -c 1 --csv python tools/profile_gemm.py --iters 3 2>/dev/null | grep -E '"dram__|"gpu__time|"lts__' | awk -F'","' -v g=$G '{print "[group " g "] " $(NF-2) " " $(NF-1) " " $NF}'
done
for G in -4 -8 -2 -4 -8 -2; do
  UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 12 2>&1 | tail -1 | sed "s/^/[group $G short] /"
done
for G in -4 -8 -4 -8; do
  UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | sed "s/^/[group $G long] /"
done
