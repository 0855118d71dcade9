"""Host<->device copy shapes for the host-streaming e2e path: contiguous vs
2-D strided (column panels of B, blocks of C), via um_get (cudaMemcpy2DAsync),
and multiply_from_host with row panels vs shell-ordered blocks."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08874_b200 import ExecConfig, _capi  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402
from paper_2510_08874_b200.hostio import multiply_from_host  # noqa: E402

lib = _capi.load()
n = 16384
h = torch.empty((n, n), dtype=torch.bfloat16, pin_memory=True)
d = torch.empty((n, n), dtype=torch.bfloat16, device="cuda")
s = torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for cols in (16384, 2048, 512):
    hv = _capi.UmView(h.data_ptr(), 0, n, 0, cols, n, _capi.UM_BF16, -1)
    dv = _capi.UmView(d.data_ptr(), 0, n, 0, cols, n, _capi.UM_BF16, 0)
    nb = n * cols * 2
    up = timed(lambda: lib.um_get(ctypes.byref(hv), ctypes.byref(dv), ctypes.c_void_p(s.cuda_stream)))
    dn = timed(lambda: lib.um_get(ctypes.byref(dv), ctypes.byref(hv), ctypes.c_void_p(s.cuda_stream)))
    print(f"2-D copy {n} rows x {cols * 2} B: H2D {nb / up / 1e6:.1f} GB/s, D2H {nb / dn / 1e6:.1f} GB/s", flush=True)
del h, d
torch.cuda.empty_cache()
fab, A, B, C, _, _ = build_problem(16384, 16384, 16384, 1, "2d", "col", "row", 1, 1, 1, seed=0, real=True,
                                   synthetic=True, devices=[0])
a_h = torch.empty((16384, 16384), dtype=torch.bfloat16, pin_memory=True)
b_h = torch.empty((16384, 16384), dtype=torch.bfloat16, pin_memory=True)
c_h = torch.empty((16384, 16384), dtype=torch.float32, pin_memory=True)
for P, Q in ((32, 1), (8, 8), (16, 4), (4, 4), (8, 2)):
    for _ in range(2):
        multiply_from_host(A, B, C, a_h, b_h, c_h, ExecConfig(), panels=P, col_panels=Q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        multiply_from_host(A, B, C, a_h, b_h, c_h, ExecConfig(), panels=P, col_panels=Q)
    e1.record()
    torch.cuda.synchronize()
    host = (time.perf_counter() - t0) / 3 * 1e3
    dev = e0.elapsed_time(e1) / 3
    print(f"multiply_from_host P={P} Q={Q}: {dev:.1f} ms/step (host {host:.1f} ms) -> "
          f"{2 * 16384 ** 3 / (dev * 1e-3) / 1e12:.0f} TFLOP/s", flush=True)
