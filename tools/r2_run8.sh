# full GPU suite, then the solo-rank projection with SM-free copy-engine pulls vs in-kernel pulls
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu_suite.log 2>&1
tail -3 gpurun_out/r2_gpu_suite.log
for eng in kernel ce; do
  timeout 900 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 8 --set get_engine=$eng --json gpurun_out/r2_matrix_p8_$eng.json > gpurun_out/r2_matrix_p8_$eng.log 2>&1
  UM_GET_GBPS=770 timeout 900 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 8 --set get_engine=$eng --json gpurun_out/r2_matrix_p8_${eng}_paced.json > gpurun_out/r2_matrix_p8_${eng}_paced.log 2>&1
done
grep -h "solo" gpurun_out/r2_matrix_p8_*.log
