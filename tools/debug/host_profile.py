"""cProfile of execute_multiply's host path on a small config (launch-bound)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_08874_b200 import ExecConfig, execute_multiply  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m, n, k, ap, bp, cp, fa, fb, fc, desc = bench.CONFIGS[name]
fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, fa(p), fb(p), fc(p), seed=0, real=True, synthetic=True,
                                   devices=[0])
cfg = ExecConfig(graph_replay=os.environ.get("UM_GRAPH_REPLAY", "0") == "1")   # eager issue by default
for _ in range(10):
    execute_multiply(A, B, C, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    execute_multiply(A, B, C, cfg)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
