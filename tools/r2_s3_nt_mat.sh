rm -f gpurun_out/s3_ntmat.log
for r in 1 2; do
 for nt in 0 256; do
  echo "== NT=$nt" >> gpurun_out/s3_ntmat.log
  UM_GEMM_NT=$nt timeout 600 python tools/bench_matrix.py --configs cfg5,cfg4,cfg3 --ps 8 --steps 5 2>&1 | grep -A1 "p=8" >> gpurun_out/s3_ntmat.log
 done
done
echo "== paced 770 (NT auto)" >> gpurun_out/s3_ntmat.log
UM_GET_GBPS=770 timeout 900 python tools/bench_matrix.py --configs cfg2,cfg3,cfg4,cfg5 --ps 2,4,8 --steps 5 --json gpurun_out/s3_paced770.json 2>&1 | grep -A1 "p=" >> gpurun_out/s3_ntmat.log
