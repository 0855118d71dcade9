timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_fullsize_gpu.py tests/test_multiprocess_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
for R in 1 2; do for T in 0 1; do
UM_GEMM_TAIL_SPLIT=$T UM_GET_GBPS=770 timeout 300 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 8 --steps 3 --warmup 1 2>&1 | grep "solo" | cut -c1-100 | sed "s/^/[tail $T paced] /"
UM_GEMM_TAIL_SPLIT=$T timeout 300 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 4,8 --steps 3 --warmup 1 2>&1 | grep "st=c" | cut -c1-80 | sed "s/^/[tail $T] /"
done; done
rm -f gpurun_out/tl_cfg5_tail.csv
UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=gpurun_out/tl_cfg5_tail.csv UM_GET_GBPS=770 timeout 300 python tools/solo_probe.py cfg5 8 kernel > /dev/null 2>&1
python tools/timeline_report.py gpurun_out/tl_cfg5_tail.csv 3,7,11
