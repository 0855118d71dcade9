"""Print the K1 work list and pulls of one rank's issue plan (cfg4 p=8 rank 3)."""
import sys; sys.path.insert(0, '.')
import torch, bench
from paper_2510_08874_b200 import ExecConfig
from paper_2510_08874_b200 import engine as eng
from paper_2510_08874_b200.schedule import lower_direct
from paper_2510_08874_b200.cli import build_problem
m, n, k, ap, bp, cp, fa, fb, fc, _ = bench.CONFIGS['cfg4']
p = 8
fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, fa(p), fb(p), fc(p), seed=0, real=True, synthetic=True, devices=[0])
cfg = ExecConfig()
orig = eng._capi.load().um_gemm_prepare
def spy(arr, n, garr, ng, dev, h):
    for i in range(n):
        g = arr[i]
        print(f"op{i}: a rows {g.a.row_lo}-{g.a.row_hi} cols {g.a.col_lo}-{g.a.col_hi} | b rows {g.b.row_lo}-{g.b.row_hi} cols {g.b.col_lo}-{g.b.col_hi} a_get={g.a_get} b_get={g.b_get} mask={g.get_mask:x}")
    for i in range(ng):
        d = garr[i]
        print(f"get{i}: src rows {d.src.row_lo}-{d.src.row_hi} cols {d.src.col_lo}-{d.src.col_hi}")
    return orig(arr, n, garr, ng, dev, h)
real_load = eng._capi.load
class L:
    def __getattr__(self, a):
        return spy if a == 'um_gemm_prepare' else getattr(real_load(), a)
eng._capi.load = lambda: L()
sched = lower_direct(A, B, C, cfg, 3)
run = eng._RankRun(A, B, C, cfg, sched, [])
run.plan()
