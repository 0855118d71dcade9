"""Debug the overlapped replica reduction on a small case, with a host-side timeout."""
import ctypes
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08874_b200 import ExecConfig, execute_multiply  # noqa: E402
from paper_2510_08874_b200 import runtime as rt  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402


def watchdog(sec, what):
    def fire():
        print(f"WATCHDOG: {what} did not finish in {sec}s", flush=True)
        os._exit(3)
    t = threading.Timer(sec, fire)
    t.daemon = True
    t.start()
    return t


m, n, k, p, ap, bp, cp, ca, cb, cc = 512, 512, 2048, 8, "col", "row", "2d", 1, 1, 8
fab, A, B, C, a, b = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=17)
cfg = ExecConfig(overlap_reduce=True, reduce_panels=1)
ovl = rt._overlap_for(A, B, C, cfg)
print("subs", {str(t): v for t, v in ovl.subs.items()}, "expected", {str(k_): v for k_, v in ovl.expected.items()},
      flush=True)
w = watchdog(30, "run 1")
execute_multiply(A, B, C, cfg)
print("issued", flush=True)
# peek flags without synchronizing the streams that wait
time.sleep(2)
for r, seg in enumerate(ovl.flag_segs):
    buf = np.zeros(seg.cols, dtype=np.uint32)
    torch.cuda.cudart().cudaMemcpy(ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(seg.ptr), buf.nbytes, 2) \
        if False else None
print("flags (host view via separate stream)", flush=True)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    vals = [seg.storage.view(torch.int32).clone() for seg in ovl.flag_segs]
s.synchronize()
print([v.tolist() for v in vals], flush=True)
torch.cuda.synchronize()
w.cancel()
print("run 1 ok", np.array_equal(C.gather(0), a @ b), flush=True)
