# raster group x L2 hints (hints now default for single-work launches): DRAM traffic + timing
for G in -4 -8 -6; do
  UM_GEMM_GROUP=$G timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 -s 2 -c 1 --csv python tools/profile_gemm.py --iters 3 2>/dev/null | grep -E '"dram__|"gpu__time' | awk -F'","' -v g=$G '{print "[group " g "] " $(NF-2) " " $(NF-1) " " $NF}'
done
for R in 1 2; do for G in -4 -8 -6; do
  UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 12 2>&1 | tail -1 | sed "s/^/[group $G short] /" | cut -c1-150
done; done
for G in -4 -8 -4 -8; do
  UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | sed "s/^/[group $G long] /" | cut -c1-150
done
for G in -4 -8; do
  UM_GEMM_GROUP=$G timeout 90 python tools/profile_gemm.py --time --iters 12 --m 16384 --n 16384 --k 16384 2>&1 | tail -1 | sed "s/^/[group $G 16k short] /" | cut -c1-150
done
