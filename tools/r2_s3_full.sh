timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/s3f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3f_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s3f_bench.log 2>&1
timeout 600 python bench.py --config cfg2 --no-cpu > gpurun_out/s3f_bench_cfg2.log 2>&1
timeout 1200 python tools/bench_matrix.py > gpurun_out/s3f_matrix.log 2>&1
