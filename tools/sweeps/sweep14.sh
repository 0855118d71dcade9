timeout 300 python tools/get_probe.py 2>&1 | grep -v CUDAEvent.h
for c in cfg5 cfg4 cfg1; do
for e in kernel copy; do
  timeout 300 python tools/bench_matrix.py --configs $c --ps 2,4,8 --set get_engine=$e --json gpurun_out/m14_${c}_$e.json > gpurun_out/m14_${c}_$e.log 2>&1
  echo "[$c $e rc=$?]"; grep -v CUDAEvent.h gpurun_out/m14_${c}_$e.log | tail -6
done; done
timeout 300 python tools/bench_matrix.py --configs cfg3 --ps 2,4,8 2>&1 | tail -6
