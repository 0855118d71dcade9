for E in reduce store none; do for S in 1024; do
UM_GEMM_EPI_DEBUG=$E UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 --m $S --n $S --k $S 2>&1 | grep timeline | tail -1 | sed "s/^/[$E $S] /" | sed 's/\[um_gemm stalls\] block 0 timeline (us after entry)://'
done; done
