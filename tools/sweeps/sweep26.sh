timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t26.log 2>&1; echo "[tests rc=$?]"; tail -2 gpurun_out/t26.log
timeout 900 python tools/bench_matrix.py --json gpurun_out/matrix_r1b.json 2>&1 | grep -v CUDAEvent.h
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1b.json; cut -c1-300 gpurun_out/bench_r1b.json
