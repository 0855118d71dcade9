run() { env "$@" timeout 60 python tools/profile_gemm.py --time --iters $ITERS 2>&1 | tail -1 | sed "s/^/[$*] /"; }
UM_GEMM_PF=4 timeout 300 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error"
for ITERS in 12 150; do
  echo "== iters $ITERS"
  for pf in 0 2 4 8 16; do run UM_GEMM_PF=$pf UM_GEMM_PROMO=0 UM_GEMM_GROUP=16; done
  run UM_GEMM_PF=0 UM_GEMM_PROMO=0 UM_GEMM_GROUP=16 UM_GEMM_NT=256
done
timeout 60 python tools/profile_gemm.py --time --iters 12 --cublas
for pf in 0 4 8; do UM_GEMM_PF=$pf UM_GEMM_PROMO=0 timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:gemm_bf16 -c 1 python tools/profile_gemm.py --iters 1 2>/dev/null | grep -E "dram__|hit_rate|tensor|cycles_elapsed" | tr -s ' ' | sed "s/^/[pf=$pf] /"; done
