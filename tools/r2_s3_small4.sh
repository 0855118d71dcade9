rm -f gpurun_out/s3_small4.log
for sk in 1 0; do
  echo "splitk=$sk" >> gpurun_out/s3_small4.log
  UM_GEMM_SPLITK=$sk timeout 300 python tools/debug/launch_probe.py >> gpurun_out/s3_small4.log 2>&1
  UM_GEMM_SPLITK=$sk UM_GEMM_STALLS=1 timeout 120 python tools/k1_timeline.py 1024 1024 1024 2>&1 | grep "block 0 timeline" | tail -1 >> gpurun_out/s3_small4.log
done
echo "plain store (wrong results)" >> gpurun_out/s3_small4.log
UM_GEMM_EPI_DEBUG=store UM_GEMM_STALLS=1 timeout 120 python tools/k1_timeline.py 1024 1024 1024 2>&1 | grep "block 0 timeline" | tail -1 >> gpurun_out/s3_small4.log
echo "no C write (wrong results)" >> gpurun_out/s3_small4.log
UM_GEMM_EPI_DEBUG=none UM_GEMM_STALLS=1 timeout 120 python tools/k1_timeline.py 1024 1024 1024 2>&1 | grep "block 0 timeline" | tail -1 >> gpurun_out/s3_small4.log
