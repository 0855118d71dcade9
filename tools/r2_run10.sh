timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x -k "copy_engine_pulls or multiply_from_host" > gpurun_out/r2_t10.log 2>&1
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -s -k "probe" >> gpurun_out/r2_t10.log 2>&1
grep -E "passed|failed|same-device|watchdog" gpurun_out/r2_t10.log | head
timeout 600 python bench.py --no-cpu --steps 6 > gpurun_out/r2_bench_blocks.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_bench_blocks.log").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e"]["roofline"]["frac"])
PY
timeout 900 python tools/bench_matrix.py --configs cfg4,cfg5 --ps 8 --set get_engine=ce > gpurun_out/r2_matrix_p8_ce2.log 2>&1
grep -E "solo|watchdog" gpurun_out/r2_matrix_p8_ce2.log | head -5
