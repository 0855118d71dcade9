timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t21.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t21.log
timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -3
timeout 120 python tools/solo_probe.py cfg5 4 kernel 2>&1 | grep -v CUDAEvent.h | tail -2
timeout 120 python tools/get_probe.py 2>&1 | grep -v CUDAEvent.h
