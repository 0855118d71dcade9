timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/t54.log 2>&1; echo "[tests rc=$?]"; tail -9 gpurun_out/t54.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench54.json; python3 -c "import json; d=json.load(open('gpurun_out/bench54.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'], d['gpu_launches'])"
timeout 900 python tools/bench_matrix.py --json gpurun_out/matrix_final2.json 2>&1 | grep -v CUDAEvent.h | grep -v solo
