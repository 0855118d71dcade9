# round-1 final profile set (L2 policy defaults): GPU suite, smoke, bench, launch list,
# ncu full of K1 (bench), fused K1 (cfg5 p=8 rank), K4 (cfg3 p=8)
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/tests_c.log 2>&1; echo "[tests rc=$?]"; tail -2 gpurun_out/tests_c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "[bench rc=$?]"; tail -1 gpurun_out/bench_c.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r1_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "[launches rc=$?]"
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/k1_cfg2 -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_k1.log 2>&1; echo "[k1 rc=$?]"
UM_MATRIX_SOLO=0 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/k1_fused_cfg5 -f \
    python tools/solo_probe.py cfg5 8 kernel > gpurun_out/ncu_fused.log 2>&1; echo "[fused rc=$?]"
UM_MATRIX_SOLO=0 ncu --set full --clock-control none -k regex:reduce_kernel -s 8 -c 1 -o gpurun_out/k4_cfg3 -f \
    python tools/bench_matrix.py --configs cfg3 --ps 8 --steps 1 --warmup 1 > gpurun_out/ncu_k4.log 2>&1; echo "[k4 rc=$?]"
ls -la gpurun_out/ | grep ncu-rep
