for v in "UM_GEMM_NT=512" "UM_GEMM_NT=256" "UM_GEMM_CG=1"; do env $v timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[$v] /"; done
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
run() { env "$@" timeout 60 python tools/profile_gemm.py --time --iters $ITERS 2>&1 | tail -1 | sed "s/^/[$*] /"; }
for ITERS in 12 150; do
  echo "== iters $ITERS"; run UM_GEMM_GROUP=16; run UM_GEMM_GROUP=8; run UM_GEMM_GROUP=32
  run UM_GEMM_GROUP=16 --m 16384 --n 16384 --k 16384 ; run UM_GEMM_GROUP=8 --m 16384 --n 16384 --k 16384
done
for g in 16 8; do UM_GEMM_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second -k regex:gemm_bf16 -c 1 python tools/profile_gemm.py --iters 1 2>/dev/null | grep -E "dram__|hit_rate|fabric|cycles_elapsed" | tr -s ' ' | sed "s/^/[G=$g] /"; done
timeout 300 python bench.py --steps 10 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
