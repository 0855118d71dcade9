timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t29.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t29.log
timeout 600 python tools/bench_matrix.py --configs cfg3,cfg4 --ps 2,4,8 2>&1 | grep -v CUDAEvent.h
timeout 600 python tools/bench_matrix.py --configs cfg3,cfg4 --ps 8 --set overlap_reduce=False 2>&1 | grep -v CUDAEvent.h
