run() { env $ENVS timeout 90 python tools/profile_gemm.py --time --iters $ITERS $SHAPE 2>&1 | tail -1 | sed "s/^/[$ENVS $SHAPE] /"; }
for SHAPE in "" "--m 8192 --n 8192 --k 65536"; do
for ITERS in 12 100; do
  for ENVS in "UM_GEMM_EPI_DEBUG=reduce" "UM_GEMM_EPI_DEBUG=none" "UM_GEMM_EPI_DEBUG=store" "UM_GEMM_EPI_DEBUG=reduce" "UM_GEMM_EPI_DEBUG=none"; do run; done
done; done
