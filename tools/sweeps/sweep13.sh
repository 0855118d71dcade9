timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t13.log 2>&1; echo "[tests rc=$?]"; grep -v "^$" gpurun_out/t13.log | tail -15
for c in cfg4 cfg5 cfg3 cfg1; do
  timeout 300 python tools/bench_matrix.py --configs $c --json gpurun_out/m13_$c.json > gpurun_out/m13_$c.log 2>&1
  echo "[$c rc=$?]"; grep -v CUDAEvent.h gpurun_out/m13_$c.log | tail -6
done
timeout 200 python bench.py --no-cpu > gpurun_out/b13.log 2>&1; tail -1 gpurun_out/b13.log | cut -c1-400
