"""Per-rank solo timing of run_direct for one config (engine debugging)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_08874_b200 import ExecConfig, run_direct  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 8
engine = sys.argv[3] if len(sys.argv) > 3 else "kernel"
extra = {k: (int(v) if v.isdigit() else v) for k, v in (kv.split("=", 1) for kv in sys.argv[4:])}
extra = {k: (bool(v) if k in ("chain_order", "overlap_reduce", "fused_accumulate", "fine_waits") else v) for k, v in extra.items()}
m, n, k, ap, bp, cp, fa, fb, fc, desc = bench.CONFIGS[name]
fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, fa(p), fb(p), fc(p), seed=0, real=True, synthetic=True,
                                   devices=[0])
cfg = ExecConfig(get_engine=engine, **extra)
torch.cuda.synchronize()
for r in range(p):
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = run_direct(A, B, C, cfg, r)
        e1.record()
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        h2 = time.perf_counter()
        ts.append(f"{e0.elapsed_time(e1):.3f}ms(host issue {1e3 * (h1 - h0):.2f}ms, total {1e3 * (h2 - h0):.2f}ms)")
    print(f"{name} p={p} {engine} rank {r}: launches={st.launches} gets={st.gets} ops={len(st.executed_ops)} :: "
          + "  ".join(ts), flush=True)
