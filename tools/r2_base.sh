set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest.log
timeout 600 python bench.py > gpurun_out/r2_bench_cfg2.log 2>&1
timeout 600 python bench.py --config cfg5 --no-cpu > gpurun_out/r2_bench_cfg5.log 2>&1
timeout 900 python tools/bench_matrix.py > gpurun_out/r2_matrix.log 2>&1
tail -3 gpurun_out/*.log
