timeout 300 python tools/get_probe.py 2>&1 | grep -v CUDAEvent.h
timeout 600 python -m pytest tests/test_runtime_gpu.py tests/test_gemm_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for c in cfg5 cfg4; do
  timeout 300 python tools/bench_matrix.py --configs $c --ps 4,8 --json gpurun_out/m15_${c}.json 2>&1 | grep -v CUDAEvent.h | tail -4
done
