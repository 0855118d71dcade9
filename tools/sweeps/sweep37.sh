timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t37.log 2>&1; echo "[tests rc=$?]"; tail -3 gpurun_out/t37.log
for P in 4 2; do timeout 300 python tools/bench_matrix.py --configs cfg3,cfg4 --ps 4,8 --set reduce_panels=$P 2>&1 | grep -v CUDAEvent.h | grep -v solo; done
timeout 300 python bench.py --steps 6 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"
