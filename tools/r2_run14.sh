timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x -k "host" > gpurun_out/r2_t14.log 2>&1
grep -E "passed|failed" gpurun_out/r2_t14.log
for extra in "" "--panels 16" "--panels 4" "--e2e-eager --panels 4"; do
  timeout 600 python bench.py --no-cpu --steps 6 $extra > gpurun_out/r2_b14.log 2>&1
  python - "$extra" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/r2_b14.log").read().strip().splitlines()[-1])
e = d["e2e"]
print(sys.argv[1] or "default", "value", round(d["value"]), "e2e", round(e["value"]), "ms", round(e["ms_per_step"], 2), "floor frac", round(e["roofline"]["frac"], 3), e["api"])
PY
done
