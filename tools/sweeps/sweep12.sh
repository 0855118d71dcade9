# fused gets at scale, one config at a time (a hang -> watchdog trap -> next config)
for c in cfg4 cfg5 cfg3 cfg2 cfg1; do
  timeout 300 python tools/bench_matrix.py --configs $c --json gpurun_out/m12_$c.json > gpurun_out/m12_$c.log 2>&1
  echo "[$c rc=$?]"; grep -v CUDAEvent.h gpurun_out/m12_$c.log | tail -8
done
