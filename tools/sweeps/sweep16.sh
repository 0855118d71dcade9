timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h
timeout 120 python tools/solo_probe.py cfg5 8 copy 2>&1 | grep -v CUDAEvent.h
timeout 120 python tools/solo_probe.py cfg4 8 kernel 2>&1 | grep -v CUDAEvent.h
