# same-box A/B: HEAD library vs working tree (stamps compiled out, tensormap prefetch kept)
for R in 1 2; do
  UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so timeout 60 python tools/profile_gemm.py --time --iters 20 --m 4096 --n 4096 --k 4096 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[HEAD] /"
  timeout 60 python tools/profile_gemm.py --time --iters 20 --m 4096 --n 4096 --k 4096 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[work] /"
done
UNIMUL_B200_LIB=tools/debug/alt/libunimul_b200.so python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[HEAD] /"
python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[work] /"
