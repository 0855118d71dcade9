timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t24.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t24.log
timeout 120 python tools/solo_probe.py cfg4 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -6
timeout 120 python tools/solo_probe.py cfg4 8 kernel k_split=0 2>&1 | grep -v CUDAEvent.h | tail -6
timeout 120 python tools/solo_probe.py cfg4 4 kernel 2>&1 | grep -v CUDAEvent.h | tail -4
