# fused get->GEMM (device arrival flags) + K4 rewrite: correctness then the engine matrix
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t11.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t11.log
timeout 600 python tools/bench_matrix.py --json gpurun_out/matrix_fused.json 2>&1 | tail -25
timeout 300 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 4,8 --set fused_gets=False 2>&1 | tail -5 | sed 's/^/[unfused] /'
