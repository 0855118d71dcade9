for shp in "1024 1024 1024" "2048 2048 2048" "512 512 512"; do
  UM_GEMM_STALLS=1 timeout 120 python tools/k1_once.py $shp 3 2>&1 | grep -E "timeline|MMA thread" | tail -2
done
timeout 600 python tools/k1_ab.py --shapes 1024x1024x1024,2048x2048x2048,512x512x512,4096x4096x1024 --iters 20 --rounds 2
