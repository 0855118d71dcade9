timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gemm_variants_gpu.py -q -x > gpurun_out/r2_t7.log 2>&1
tail -3 gpurun_out/r2_t7.log
timeout 1200 python tools/k1_ab.py --env UM_GEMM_SKSTART=0 --env UM_GEMM_SKSTART=1 --shapes 8192x8192x8192,4096x4096x4096,16384x16384x16384,2048x2048x4096,65536x8192x8192,6144x6144x6144 --json gpurun_out/r2_ab_skstart.json > gpurun_out/r2_ab_skstart.log 2>&1
cat gpurun_out/r2_ab_skstart.log
