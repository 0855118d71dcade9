timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t36.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t36.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench36.json; python3 -c "import json; d=json.load(open('gpurun_out/bench36.json')); print(d['value'], d['roofline'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'], d['gpu_launches'])"
