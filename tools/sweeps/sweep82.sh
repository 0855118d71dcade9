# paired TMA epilogue: default (2 boxes/warp) and v4 (4 boxes/warp, 5 stages at NT=256)
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
UNIMUL_B200_LIB=tools/debug/v4/libunimul_b200.so timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for L in v4 default; do
  if [ $L = v4 ]; then P=tools/debug/v4/libunimul_b200_prof.so; N=tools/debug/v4/libunimul_b200.so; else P=paper_2510_08874_b200/_lib/libunimul_b200_prof.so; N=paper_2510_08874_b200/_lib/libunimul_b200.so; fi
  UNIMUL_B200_LIB=$P UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 --m 1024 --n 1024 --k 1024 2>&1 | grep timeline | tail -1 | sed "s/^/[$L] /" | sed 's/\[um_gemm stalls\] block 0 timeline (us after entry)://'
  UNIMUL_B200_LIB=$P UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 2>&1 | grep "pairs" | tail -1 | sed "s/^/[$L cfg2] /"
  UNIMUL_B200_LIB=$N python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[$L] /"
  for S in "--m 4096 --n 4096 --k 4096" "" "--m 16384 --n 16384 --k 16384"; do
    UNIMUL_B200_LIB=$N timeout 60 python tools/profile_gemm.py --time --iters 20 $S 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[$L] /"
  done
  UNIMUL_B200_LIB=$N timeout 60 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | cut -c1-110 | sed "s/^/[$L long] /"
done
