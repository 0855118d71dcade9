timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1 -c 1 -o gpurun_out/prof_gemm_v3 python tools/profile_gemm.py --iters 2 > /dev/null 2>&1; echo "ncu rc=$?"
