set -x
UM_GEMM_NT=512 timeout 300 python tools/gemm_probe.py 2>&1 | grep -E "OK|FAIL|PERF|Error" | head -20
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -2
for g in 8 16 32; do for p in "2 1" "0 0"; do set -- $p; UM_GEMM_NT=512 UM_GEMM_GROUP=$g UM_GEMM_APOL=$1 UM_GEMM_BPOL=$2 timeout 60 python tools/profile_gemm.py --time --iters 150 2>&1 | tail -1 | sed "s/^/nt512 pol=$1$2 /"; done; done
UM_GEMM_NT=256 timeout 60 python tools/profile_gemm.py --time --iters 150 | sed "s/^/nt256 /"
timeout 60 python tools/profile_gemm.py --time --iters 150 --cublas
