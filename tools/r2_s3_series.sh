for shp in 8192x8192x8192 4096x4096x4096 16384x16384x16384; do
  timeout 300 python tools/k1_series.py --shape $shp --iters 40 --blocks 4 > gpurun_out/s3_series_$shp.log 2>&1
done
timeout 300 python tools/k1_series.py --shape 8192x8192x8192 --iters 200 --blocks 2 > gpurun_out/s3_series_long.log 2>&1
