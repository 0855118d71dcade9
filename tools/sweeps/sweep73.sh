timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for E in 4 8; do for S in 256 1024 2048; do
UM_GEMM_EPI_WARPS=$E UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 5 --m $S --n $S --k $S 2>&1 | grep timeline | tail -1 | sed "s/^/[ew$E $S] /" | sed 's/\[um_gemm stalls\] block 0 timeline (us after entry)://'
done; done
for E in 4 8; do UM_GEMM_EPI_WARPS=$E python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[ew$E] /"; done
