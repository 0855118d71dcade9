# same-box A/B: HEAD library vs default library without profiling code
for R in 1 2; do
  for S in "--m 4096 --n 4096 --k 4096" "" "--m 16384 --n 16384 --k 16384"; do
  UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so timeout 60 python tools/profile_gemm.py --time --iters 20 $S 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[HEAD] /"
  timeout 60 python tools/profile_gemm.py --time --iters 20 $S 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[work] /"
done; done
UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[HEAD] /"
python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[work] /"
UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 --m 1024 --n 1024 --k 1024 2>&1 | grep -E "timeline|pairs" | tail -2
