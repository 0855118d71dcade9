for nt in 512 256; do
 for shp in "8192 8192 8192" "16384 16384 16384" "4096 4096 4096"; do
  echo "== NT=$nt $shp" >> gpurun_out/s3_lat.log
  UM_GEMM_NT=$nt UM_GEMM_STALLS=1 timeout 300 python tools/k1_timeline.py $shp 2>&1 | grep -v timeline | tail -4 >> gpurun_out/s3_lat.log
 done
done
