timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x -k "multiply_from_host" > gpurun_out/r2_t12.log 2>&1
grep -E "passed|failed" gpurun_out/r2_t12.log
for shp in "8192 8192 8192" "16384 16384 16384" "4096 4096 4096"; do
  UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=/tmp/tl.csv timeout 300 python tools/k1_timeline.py $shp 2>&1 | grep -v "^\[um_gemm stalls\] block" | tail -6
  rm -f /tmp/tl.csv
done
timeout 900 python tools/k1_ab.py --env UM_GEMM_NT=512 --env UM_GEMM_NT=256 --shapes 8192x8192x8192,16384x16384x16384 --rounds 2
