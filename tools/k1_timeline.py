"""Per-tile timeline of ONE K1 launch (profiling build): tile durations on the
MMA thread (tile taken -> all its MMAs issued), the gaps between consecutive
tiles of a pair, and the stall breakdown.

    UM_GEMM_STALLS=1 UM_GEMM_TIMELINE=/tmp/tl.csv python tools/k1_timeline.py 8192 8192 8192
"""
import csv
import ctypes
import os
import statistics
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08874_b200 import _capi as C  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
lib = C.load()
a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
b = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
c = torch.zeros(m, n, device="cuda")
va = C.UmView(a.data_ptr(), 0, m, 0, k, a.stride(0), C.UM_BF16, 0)
vb = C.UmView(b.data_ptr(), 0, k, 0, n, b.stride(0), C.UM_BF16, 0)
vc = C.UmView(c.data_ptr(), 0, m, 0, n, c.stride(0), C.UM_F32, 0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    C.check(lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s), "um_gemm_acc")
torch.cuda.synchronize()
path = os.environ.get("UM_GEMM_TIMELINE")
if not path:
    sys.exit(0)
rows = [r for r in csv.DictReader(open(path)) if r["kind"] == "tile"]
last = max(int(r["launch"]) for r in rows)
per_pair = defaultdict(list)
for r in rows:
    if int(r["launch"]) == last:
        per_pair[int(r["pair"])].append((int(r["start_ns"]), int(r["end_ns"])))
durs, gaps, firsts, ends = [], [], [], []
for p, ts in per_pair.items():
    ts.sort()
    firsts.append(ts[0][0])
    ends.append(ts[-1][1])
    for i, (s0, e0) in enumerate(ts):
        if e0:
            durs.append(e0 - s0)
        if i + 1 < len(ts) and e0:
            gaps.append(ts[i + 1][0] - e0)
span = max(ends)
print(f"{m}x{n}x{k}: {sum(len(v) for v in per_pair.values())} tiles on {len(per_pair)} pairs, span {span/1e3:.1f} us")
print(f"tile (taken -> MMAs issued) us: median {statistics.median(durs)/1e3:.2f}, min {min(durs)/1e3:.2f}, "
      f"max {max(durs)/1e3:.2f}")
if gaps:
    print(f"gap to next tile us: median {statistics.median(gaps)/1e3:.2f}, max {max(gaps)/1e3:.2f}")
print(f"first tile taken us: median {statistics.median(firsts)/1e3:.2f}; pairs' last MMA issue us: "
      f"min {min(ends)/1e3:.1f} median {statistics.median(ends)/1e3:.1f} max {max(ends)/1e3:.1f}")
