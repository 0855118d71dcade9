timeout 900 python tools/bench_matrix.py --json gpurun_out/matrix_r1.json 2>&1 | grep -v CUDAEvent.h
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json; cat gpurun_out/bench_r1.json | cut -c1-600
