for shp in 8192x8192x8192 16384x16384x16384 4096x4096x4096; do
  timeout 300 python tools/k1_series.py --shape $shp --iters 30 --blocks 2 > gpurun_out/s3_clk_$shp.log 2>&1
done
