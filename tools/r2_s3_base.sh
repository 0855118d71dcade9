set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/s3_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s3_bench.log 2>&1
tail -3 gpurun_out/*.log
