rm -f gpurun_out/s3_small5.log
timeout 300 python tools/debug/launch_probe.py >> gpurun_out/s3_small5.log 2>&1
for s in 256 1024 2048; do
  UM_GEMM_STALLS=1 timeout 120 python tools/k1_timeline.py $s $s $s 2>&1 | grep "block 0 timeline" | tail -1 | sed "s/^/$s: /" >> gpurun_out/s3_small5.log
done
