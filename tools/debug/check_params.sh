for v in "UM_GEMM_NT=512" "UM_GEMM_NT=256" "UM_GEMM_CG=1" "UM_GEMM_STATIC=1"; do env $v timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog|PERF" | sed "s/^/[$v] /"; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do timeout 90 python tools/profile_gemm.py --time --iters 12; done
for i in 1 2 3; do timeout 90 python tools/profile_gemm.py --time --iters 12 --m 16384 --n 16384 --k 16384; done
timeout 300 python bench.py --steps 10 --no-cpu 2>&1 | tail -1 | cut -c1-180
