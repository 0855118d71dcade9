"""K2 get-engine probe: copy-engine pull (um_get) vs in-kernel get warps
(um_gemm_acc_fused with no ops / alongside a GEMM), same-device slices."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08874_b200 import _capi  # noqa: E402

lib = _capi.load()
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
sp = ctypes.c_void_p(s.cuda_stream)


def view(t, r0, r1, c0, c1, dt=_capi.UM_BF16):
    return _capi.UmView(t.data_ptr(), r0, r1, c0, c1, t.stride(0), dt, 0)


def timed(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for rows, cols in ((16384, 2048), (8192, 4096), (16384, 16384)):
    src = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    dst = torch.empty_like(src)
    nbytes = src.numel() * 2
    sv, dv = view(src, 0, rows, 0, cols), view(dst, 0, rows, 0, cols)

    def ce():
        _capi.check(lib.um_get(ctypes.byref(sv), ctypes.byref(dv), sp), "um_get")

    g = _capi.UmGetDesc(sv, dv)

    def kern():
        _capi.check(lib.um_gemm_acc_fused(None, 0, ctypes.byref(g), 1, 0, sp), "fused")

    for name, fn in (("um_get (driver copy)", ce), ("in-kernel get warps", kern)):
        dst.zero_()
        ms = timed(fn)
        assert torch.equal(dst, src), name
        print(f"{rows}x{cols} bf16 ({nbytes / 2**20:.0f} MiB) {name:22s}: {ms:.3f} ms "
              f"{nbytes / ms / 1e6:.0f} GB/s copied ({2 * nbytes / ms / 1e6:.0f} GB/s HBM r+w)", flush=True)

# get + an independent GEMM in the same launch (interference)
m = n = 4096
k = 8192
A = torch.randn(m, k, device="cuda").to(torch.bfloat16)
B = torch.randn(k, n, device="cuda").to(torch.bfloat16)
C = torch.zeros(m, n, device="cuda")
op = _capi.UmGemmOp(view(A, 0, m, 0, k), view(B, 0, k, 0, n), view(C, 0, m, 0, n, _capi.UM_F32), 0)
src = torch.randn(16384, 16384, device="cuda").to(torch.bfloat16)
dst = torch.empty_like(src)
g = _capi.UmGetDesc(view(src, 0, 16384, 0, 16384), view(dst, 0, 16384, 0, 16384))
t_gemm = timed(lambda: lib.um_gemm_acc_fused(ctypes.byref(op), 1, None, 0, 0, sp))
t_get = timed(lambda: lib.um_gemm_acc_fused(None, 0, ctypes.byref(g), 1, 0, sp))
t_both = timed(lambda: lib.um_gemm_acc_fused(ctypes.byref(op), 1, ctypes.byref(g), 1, 0, sp))
print(f"GEMM {m}x{n}x{k} alone {t_gemm:.3f} ms ({2 * m * n * k / t_gemm / 1e9:.0f} TFLOP/s); get 512 MiB alone "
      f"{t_get:.3f} ms; both in one launch {t_both:.3f} ms (sum {t_gemm + t_get:.3f})")
