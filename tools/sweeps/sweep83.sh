rm -f gpurun_out/tl_cfg5_paced.csv gpurun_out/tl_cfg4_paced.csv
UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=gpurun_out/tl_cfg5_paced.csv UM_GET_GBPS=770 timeout 300 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep "rank" | head -8
python tools/timeline_report.py gpurun_out/tl_cfg5_paced.csv 3,7,11,15,19,23,27,31
UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=gpurun_out/tl_cfg4_paced.csv UM_GET_GBPS=770 timeout 300 python tools/solo_probe.py cfg4 8 kernel 2>&1 | grep "rank" | head -8
python tools/timeline_report.py gpurun_out/tl_cfg4_paced.csv 3,7,11,15,19,23,27,31
