"""One rank's fused launch over time (profiling build): per 25 us bucket, the
share of pairs holding a tile, the tiles started, their median span, and the
pulled chunks landed.

    UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=/tmp/tl.csv UM_GET_GBPS=770 \
        python tools/debug/rank_profile.py cfg4 8 3 [key=value ExecConfig overrides]
"""
import csv
import os
import statistics
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_08874_b200 import ExecConfig, run_direct  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402

name, p, rank = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
extra = {k: (int(v) if v.isdigit() else v) for k, v in (kv.split("=", 1) for kv in sys.argv[4:])}
m, n, k, ap, bp, cp, fa, fb, fc, _ = bench.CONFIGS[name]
fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, fa(p), fb(p), fc(p), seed=0, real=True, synthetic=True,
                                   devices=[0])
cfg = ExecConfig(**extra)
for _ in range(3):
    run_direct(A, B, C, cfg, rank)
torch.cuda.synchronize()
path = os.environ["UM_GEMM_TIMELINE"]
tiles, chunks, kbs = defaultdict(list), defaultdict(list), defaultdict(list)
with open(path) as f:
    for r in csv.DictReader(f):
        {"tile": tiles, "chunk": chunks, "kb": kbs}[r["kind"]][int(r["launch"])].append(r)
L = max(tiles)
ts = [(int(r["pair"]), int(r["start_ns"]), int(r["end_ns"])) for r in tiles[L]]
ch = sorted(int(r["start_ns"]) for r in chunks[L])
pairs = len({pp for pp, _, _ in ts})
span = max(e for _, _, e in ts)
B_NS = 25000
print(f"{name} p={p} rank {rank} {extra}: span {span / 1e3:.1f} us, {len(ts)} tiles on {pairs} pairs, "
      f"{len(ch)} chunks (last {ch[-1] / 1e3 if ch else 0:.1f} us)")
for b0 in range(0, span, B_NS):
    b1 = b0 + B_NS
    busy = sum(max(0, min(e, b1) - max(s, b0)) for _, s, e in ts) / (pairs * B_NS)
    started = [(e - s) / 1e3 for _, s, e in ts if b0 <= s < b1]
    landed = sum(1 for c in ch if b0 <= c < b1)
    med = statistics.median(started) if started else 0.0
    print(f"  {b0 / 1e3:6.0f}-{b1 / 1e3:4.0f} us: pairs busy {busy:4.0%}, tiles started {len(started):3d} "
          f"(median span {med:6.1f} us), chunks landed {landed}")

# profiling build: CTAs 0 / 1, first unit: A rows landed, loads issued per k-block
for cta in (0, 1):
    rec = {int(r["index"]): int(r["start_ns"]) / 1e3 for r in kbs[L] if int(r["pair"]) == cta}
    if rec:
        ks = sorted(k for k in rec if k >= 0)
        marks = [k for k in ks if k in (0, 1, 2, 4, 8, 16, 32, 48, 64, 80, 96, 112) or k == ks[-1]]
        print(f"  CTA {cta} first unit: A rows landed {rec.get(-1, float('nan')):.1f} us; loads issued at kb "
              + ", ".join(f"{k}: {rec[k]:.1f}" for k in marks) + " us")
