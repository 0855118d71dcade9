timeout 1200 python tools/bench_matrix.py --json gpurun_out/r1_engine_matrix.json > gpurun_out/matrix.log 2>&1; echo "[matrix rc=$?]"
UM_GET_GBPS=770 timeout 1200 python tools/bench_matrix.py --configs cfg2,cfg3,cfg4,cfg5 --ps 2,4,8 --json gpurun_out/r1_engine_matrix_paced770.json > gpurun_out/matrix_paced.log 2>&1; echo "[paced rc=$?]"
cat gpurun_out/matrix.log gpurun_out/matrix_paced.log | grep -v Warning | cut -c1-220
