timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_fullsize_gpu.py -x -q -p no:cacheprovider > gpurun_out/t28.log 2>&1; echo "[tests rc=$?]"; tail -2 gpurun_out/t28.log
for X in "" "mn_split=0"; do echo "== $X"; timeout 120 python tools/solo_probe.py cfg5 4 kernel $X 2>&1 | grep -v CUDAEvent.h; done
for X in "" "mn_split=0"; do echo "== $X"; timeout 120 python tools/solo_probe.py cfg4 8 kernel $X 2>&1 | grep -v CUDAEvent.h | grep "rank 3\|rank 5\|rank 7"; done
for X in "" "mn_split=0"; do echo "== $X"; timeout 120 python tools/solo_probe.py cfg5 8 kernel $X 2>&1 | grep -v CUDAEvent.h | tail -2; done
