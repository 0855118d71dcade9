UM_GEMM_EPI_DEBUG=rmw timeout 120 python tools/gemm_probe.py 2>&1 | grep -E "ALL_OK|FAIL|Error|watchdog" | sed "s/^/[rmw probe] /"
for E in reduce rmw reduce rmw; do UM_GEMM_EPI_DEBUG=$E timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1; done
for E in reduce rmw; do UM_GEMM_EPI_WARPS=8 UM_GEMM_EPI_DEBUG=$E timeout 90 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1 | sed "s/^/[ew8] /"; done
for E in reduce rmw; do UM_GEMM_EPI_DEBUG=$E timeout 90 python tools/profile_gemm.py --time --iters 30 --m 16384 --n 16384 --k 16384 2>&1 | tail -1; done
