for X in "" "mn_split=0"; do echo "== $X"; timeout 120 python tools/solo_probe.py cfg5 4 kernel $X 2>&1 | grep -v CUDAEvent.h; done
for X in "" "mn_split=0"; do echo "== p2 $X"; timeout 120 python tools/solo_probe.py cfg5 2 kernel $X 2>&1 | grep -v CUDAEvent.h; done
timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
