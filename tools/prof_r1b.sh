# refreshed round-1 profile set with the final kernels: bench K1 (cfg2), fused get->GEMM (cfg5 p=8 rank),
# get-only launch (in-kernel get warps), K4 slice; launch list of the bench; the engine matrix
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r1_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "[launches rc=$?]"
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 -o gpurun_out/k1_cfg2 -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_k1.log 2>&1; echo "[k1 rc=$?]"
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/k1_fused_cfg5 -f \
    python tools/solo_probe.py cfg5 8 kernel > gpurun_out/ncu_fused.log 2>&1; echo "[fused rc=$?]"
ncu --set full --clock-control none -k regex:gemm_bf16 -s 5 -c 1 -o gpurun_out/k2_getonly -f \
    python tools/get_probe.py > gpurun_out/ncu_get.log 2>&1; echo "[getonly rc=$?]"
UM_MATRIX_SOLO=0 ncu --set full --clock-control none -k regex:reduce_kernel -s 8 -c 1 -o gpurun_out/k4_cfg3 -f \
    python tools/bench_matrix.py --configs cfg3 --ps 8 --steps 1 --warmup 1 > gpurun_out/ncu_k4.log 2>&1; echo "[k4 rc=$?]"
timeout 900 python tools/bench_matrix.py --json gpurun_out/matrix_final.json 2>&1 | grep -v CUDAEvent.h | grep -v solo | tail -20
ls gpurun_out/*.ncu-rep
