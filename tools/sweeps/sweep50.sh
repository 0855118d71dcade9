timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t50.log 2>&1; echo "[tests rc=$?]"; tail -2 gpurun_out/t50.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench50.json; python3 -c "import json; d=json.load(open('gpurun_out/bench50.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'])"
