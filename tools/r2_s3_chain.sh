rm -f gpurun_out/s3_chain.log
for cw in 6 12 3; do for tsplit in 0 1; do
  echo "== chain_waves=$cw tail_split=$tsplit" >> gpurun_out/s3_chain.log
  UM_GEMM_CHAIN_WAVES=$cw UM_GEMM_TAIL_SPLIT=$tsplit UM_GET_GBPS=770 timeout 300 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -E "rank (0|3|5)" | sed 's/(host[^)]*)//g' | cut -c1-200 >> gpurun_out/s3_chain.log
done; done
