timeout 300 python -m pytest tests/test_gemm_variants_gpu.py tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
rm -f gpurun_out/tl_cfg5_paced2.csv
UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=gpurun_out/tl_cfg5_paced2.csv UM_GET_GBPS=770 timeout 300 python tools/solo_probe.py cfg5 8 kernel > /dev/null 2>&1
python tools/timeline_report.py gpurun_out/tl_cfg5_paced2.csv 3,7,11,15
for R in 1 2; do
UM_GET_GBPS=770 timeout 300 python tools/bench_matrix.py --configs cfg5 --ps 4,8 --steps 3 --warmup 1 2>&1 | grep "solo" | cut -c1-110
timeout 300 python tools/bench_matrix.py --configs cfg5,cfg1 --ps 8 --steps 3 --warmup 1 2>&1 | grep -A1 "st=c" | cut -c1-110
done
