set -x
timeout 600 python tools/cublas_bar.py --json gpurun_out/r2_cublas_bar.json > gpurun_out/r2_cublas_bar.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 -o gpurun_out/r2_k1_8192 python tools/k1_once.py 8192 8192 8192 > gpurun_out/r2_ncu_8192.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/r2_k1_bench_cfg5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2_ncu_cfg5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench_cfg5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2_ncu_launches.log 2>&1
ls -la gpurun_out
