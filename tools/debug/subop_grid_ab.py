"""One 8192^3 C += A.B as a single K1 work vs as a 4x4 / 2x2 grid of sub-ops
(the split a rank that pulls both operands runs), operands resident: isolates
the cost of the sub-op structure from the pulls.

    python tools/debug/subop_grid_ab.py [reps]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2510_08874_b200 import _capi as C  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
N = 8192
lib = C.load()
a = (torch.rand(N, N, device="cuda") * 2 - 1).to(torch.bfloat16)
b = (torch.rand(N, N, device="cuda") * 2 - 1).to(torch.bfloat16)
c = torch.zeros(N, N, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def view(t, r0, r1, c0, c1, dt):
    return C.UmView(t.data_ptr(), r0, r1, c0, c1, t.stride(0), dt, 0)


def ops_for(g):
    q = N // g
    return [C.UmGemmOp(view(a, i * q, (i + 1) * q, 0, N, C.UM_BF16), view(b, 0, N, j * q, (j + 1) * q, C.UM_BF16),
                       view(c, i * q, (i + 1) * q, j * q, (j + 1) * q, C.UM_F32), 0)
            for i in range(g) for j in range(g)]


for rnd in range(2):
    for g in (1, 2, 4):
        ops = ops_for(g)
        arr = (C.UmGemmOp * len(ops))(*ops)
        h = ctypes.c_void_p()
        C.check(lib.um_gemm_prepare(arr, len(ops), None, 0, 0, ctypes.byref(h)), "prepare")
        for _ in range(3):
            C.check(lib.um_gemm_launch(h, s), "launch")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            C.check(lib.um_gemm_launch(h, s), "launch")
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"round {rnd} grid {g}x{g}: {ms:.3f} ms per launch = {2 * N ** 3 / ms / 1e9:.0f} TFLOP/s", flush=True)
        lib.um_gemm_destroy(h)
