for S in 256 1024 2048; do
UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 5 --m $S --n $S --k $S 2>&1 | grep timeline | tail -2 | sed "s/^/[$S] /"
done
