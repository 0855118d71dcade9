# cfg4: 2D sub-op grid for ops pulling both A and B, paced pulls
run() { env UM_GET_GBPS=770 $E timeout 300 python tools/bench_matrix.py --configs cfg4 --ps 2,4,8 --steps 3 --warmup 1 $S 2>&1 | grep -B1 "solo ranks" | sed "s/^/[$E $S] /"; }
E=""; S=""; run
E=""; S="--set mn_split=2"; run
E=""; S="--set mn_split=8"; run
E="UM_GET_GBPS=0"; S=""; run
