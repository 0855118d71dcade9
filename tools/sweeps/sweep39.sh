timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t39.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t39.log
for X in "" "fine_waits=0"; do echo "== $X"
timeout 120 python tools/solo_probe.py cfg4 8 kernel $X 2>&1 | grep -v CUDAEvent.h | grep "rank 3\|rank 5"
UM_GET_GBPS=770 timeout 120 python tools/solo_probe.py cfg4 8 kernel $X 2>&1 | grep -v CUDAEvent.h | grep "rank 3\|rank 5"
timeout 120 python tools/solo_probe.py cfg5 8 kernel $X 2>&1 | grep -v CUDAEvent.h | tail -1
UM_GET_GBPS=770 timeout 120 python tools/solo_probe.py cfg5 8 kernel $X 2>&1 | grep -v CUDAEvent.h | tail -1
done
