# DRAM traffic of K1 vs L2 eviction policies (cfg2 shape): pol 0 normal, 1 evict_first, 2 evict_last
for E in "UM_GEMM_BPOL=2" "UM_GEMM_APOL=1" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2 UM_GEMM_CPOL=1" "UM_GEMM_CPOL=1"; do
  env $E timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 -s 2 -c 1 --csv python tools/profile_gemm.py --iters 3 2>/dev/null | grep -E '"dram__|"gpu__time' | awk -F'","' -v g="$E" '{print "[" g "] " $(NF-2) " " $(NF-1) " " $NF}'
done
for E in "UM_GEMM_APOL=1 UM_GEMM_BPOL=2" "UM_GEMM_APOL=0" "UM_GEMM_APOL=1 UM_GEMM_BPOL=2" "UM_GEMM_APOL=0"; do
  env $E timeout 90 python tools/profile_gemm.py --time --iters 12 2>&1 | tail -1 | sed "s/^/[$E short] /"
  env $E timeout 90 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | sed "s/^/[$E long] /"
done
