timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_runtime_gpu.py -q -x -k "not copy_engine" > gpurun_out/r2_t16.log 2>&1
grep -E "passed|failed" gpurun_out/r2_t16.log
timeout 900 python tools/k1_ab.py --env "" --env UM_GEMM_SPLITK=0 --env UM_GEMM_EPI_DEBUG=red --shapes 1024x1024x1024,512x512x512,2048x2048x4096,1024x1024x4096,768x768x2048 --iters 20 --rounds 2
for shp in "1024 1024 1024" "1024 1024 4096"; do
  UM_GEMM_STALLS=1 timeout 120 python tools/k1_once.py $shp 3 2>&1 | grep -E "timeline|MMA thread" | tail -2
done
