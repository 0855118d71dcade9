timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t17.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t17.log
timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h
timeout 120 python tools/solo_probe.py cfg5 8 copy 2>&1 | grep -v CUDAEvent.h | tail -3
timeout 120 python tools/solo_probe.py cfg4 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -5
timeout 600 python tools/bench_matrix.py --configs cfg5,cfg4,cfg1 --ps 2,4,8 --json gpurun_out/m17.json 2>&1 | grep -v CUDAEvent.h
timeout 300 python bench.py --no-cpu 2>&1 | tail -1 | cut -c1-300
