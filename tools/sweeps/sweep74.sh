timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for E in reduce red; do for S in 256 2048; do
UM_GEMM_EPI_DEBUG=$E UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 5 --m $S --n $S --k $S 2>&1 | grep timeline | tail -1 | sed "s/^/[$E $S] /" | sed 's/\[um_gemm stalls\] block 0 timeline (us after entry)://'
done; done
for E in reduce red; do UM_GEMM_EPI_DEBUG=$E python tools/debug/launch_probe.py 2>&1 | grep "us/launch" | sed "s/^/[$E] /"; done
for E in reduce red; do UM_GEMM_EPI_DEBUG=$E timeout 60 python tools/profile_gemm.py --time --iters 20 --m 4096 --n 4096 --k 4096 2>&1 | tail -1 | cut -c1-100 | sed "s/^/[$E] /"; done
