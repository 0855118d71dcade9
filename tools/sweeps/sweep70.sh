# small-GEMM K1 kernel durations (ncu) vs event timing around the API call
for S in 1024 2048 4096; do
  timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_bf16 -s 3 -c 1 --csv python tools/profile_gemm.py --iters 3 --m $S --n $S --k $S 2>/dev/null | grep gpu__time | awk -F'","' -v s=$S '{print "[ncu " s "^3] " $(NF-1) " " $NF}'
  timeout 120 python tools/profile_gemm.py --time --iters 50 --m $S --n $S --k $S 2>&1 | tail -1 | sed "s/^/[events $S^3] /" | cut -c1-120
done
timeout 300 python - <<'PY'
import torch, time, sys
sys.path.insert(0, '.')
import bench
from paper_2510_08874_b200 import ExecConfig, execute_multiply
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.graphs import CapturedMultiply
m, n, k, ap, bp, cp, fa, fb, fc, desc = bench.CONFIGS["cfg1"]
fab, A, B, C, _, _ = build_problem(m, n, k, 1, ap, bp, cp, fa(1), fb(1), fc(1), seed=0, real=True, synthetic=True, devices=[0])
cfg = ExecConfig()
for _ in range(5): execute_multiply(A, B, C, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): execute_multiply(A, B, C, cfg)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"[cfg1 p=1 execute_multiply] host issue {1e3*(t1-t0)/200:.3f} ms/call, wall {1e3*(t2-t0)/200:.3f} ms/call")
cm = CapturedMultiply(A, B, C, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(200): cm.replay()
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"[cfg1 p=1 graph replay] wall {1e3*(t2-t0)/200:.3f} ms/replay")
PY
