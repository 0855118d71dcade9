# multi-process (torchrun) bench path on one GPU + per-config single-rank runs
export OMP_NUM_THREADS=1
for cfg in cfg2 cfg5 cfg4 cfg3; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu --config $cfg > gpurun_out/mp_$cfg.log 2>&1; echo "torchrun2 $cfg rc=$?"; grep -E '"value"' gpurun_out/mp_$cfg.log | python3 -c "import sys,json; [print({k:(d[k] if k!='e2e' else d[k]['value']) for k in ('value','ms_per_step','gpu_launches','e2e')}) for d in map(json.loads,sys.stdin)]" ; grep -iE "error|Traceback" gpurun_out/mp_$cfg.log | head -5
done
for cfg in cfg3 cfg4 cfg5; do timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 5 2>&1 | python3 -c "import sys,json; [print('$cfg p=1', d['value'], d['ms_per_step']) for d in map(json.loads,[l for l in sys.stdin if l.startswith('{')])]"; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 --ref-step-s 2 2>&1 | tail -1 | cut -c1-300
