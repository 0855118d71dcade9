run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters $ITERS $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS $SHAPE] /"; }
for SHAPE in "" "--m 16384 --n 16384 --k 16384" "--m 8192 --n 8192 --k 65536"; do
for ITERS in 12 100; do
  for ENVS in "UM_GEMM_STATIC=1 UM_GEMM_GROUP=16" "UM_GEMM_GROUP=8" "UM_GEMM_GROUP=16" "UM_GEMM_GROUP=4" "UM_GEMM_GROUP=-4"; do run; done
done; done
timeout 90 python tools/profile_gemm.py --time --iters 12 --m 16384 --n 16384 --k 16384 --cublas
