# paced (NVLink-like) pulls: k-chains vs per-slab order for ranks that pull before computing
run() { env UM_GET_GBPS=770 $E timeout 300 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 4,8 --steps 3 --warmup 1 $S 2>&1 | grep "solo ranks" | sed "s/^/[$E $S] /"; }
E=""; S=""; run
E="UM_GEMM_CHAIN=0"; S=""; run
E="UM_GEMM_CHAIN=0"; S="--set chain_order=False"; run
E="UM_GEMM_CHAIN=0"; S="--set k_split=8"; run
E=""; S="--set k_split=8"; run
