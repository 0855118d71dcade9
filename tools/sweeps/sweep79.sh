timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for R in 1 2; do
  for S in "--m 4096 --n 4096 --k 4096" "" "--m 16384 --n 16384 --k 16384"; do
  UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so timeout 60 python tools/profile_gemm.py --time --iters 20 $S 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[HEAD] /"
  timeout 60 python tools/profile_gemm.py --time --iters 20 $S 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[work] /"
done; done
for R in 1 2; do
  UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so timeout 60 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | cut -c1-110 | sed "s/^/[HEAD long] /"
  timeout 60 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | cut -c1-110 | sed "s/^/[work long] /"
done
UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[HEAD] /"
python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[work] /"
UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 2>&1 | grep -E "pairs" | tail -1
UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 --m 1024 --n 1024 --k 1024 2>&1 | grep -E "timeline" | tail -1
UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so timeout 300 python tools/bench_matrix.py --configs cfg5 --ps 8 --steps 3 --warmup 1 2>&1 | grep -A1 "st=c" | cut -c1-120 | sed "s/^/[HEAD] /"
timeout 300 python tools/bench_matrix.py --configs cfg5 --ps 8 --steps 3 --warmup 1 2>&1 | grep -A1 "st=c" | cut -c1-120 | sed "s/^/[work] /"
