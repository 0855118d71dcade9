timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for R in 1 2; do
for W in 0 6 12; do
  UM_GEMM_CHAIN_WAVES=$W timeout 300 python tools/bench_matrix.py --configs cfg5,cfg1 --ps 4,8 --steps 3 --warmup 1 2>&1 | grep -A1 "st=c" | sed "s/^/[waves $W] /" | cut -c1-150
  UM_GET_GBPS=770 UM_GEMM_CHAIN_WAVES=$W timeout 300 python tools/bench_matrix.py --configs cfg5 --ps 8 --steps 3 --warmup 1 2>&1 | grep "solo" | sed "s/^/[waves $W paced] /" | cut -c1-150
done; done
