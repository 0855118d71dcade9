"""Host cost of one prepared K1 launch (um_gemm_launch) vs the GPU time, small GEMMs."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2510_08874_b200 import _capi as C  # noqa: E402

lib = C.load()
torch.cuda.set_device(0)


def v(t, dt):
    return C.UmView(t.data_ptr(), 0, t.shape[0], 0, t.shape[1], t.stride(0), dt, 0)


SIZES = [int(x) for x in os.environ.get("UM_PROBE_SIZES", "256,1024,2048,4096").split(",")]
for s in SIZES:
    a = torch.randn(s, s, device="cuda").to(torch.bfloat16)
    b = torch.randn(s, s, device="cuda").to(torch.bfloat16)
    c = torch.zeros(s, s, device="cuda")
    op = C.UmGemmOp(v(a, C.UM_BF16), v(b, C.UM_BF16), v(c, C.UM_F32), 0)
    h = ctypes.c_void_p()
    C.check(lib.um_gemm_prepare(ctypes.byref(op), 1, None, 0, 0, ctypes.byref(h)), "prepare")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(20):
        lib.um_gemm_launch(h, st)
    torch.cuda.synchronize()
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(n):
        lib.um_gemm_launch(h, st)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    gpu = e0.elapsed_time(e1) / n * 1e3
    # GPU time when the host is far ahead: a graph of 50 launches
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    lib.um_gemm_launch(h, ctypes.c_void_p(side.cuda_stream))   # per-stream counters allocated outside capture
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        for _ in range(50):
            lib.um_gemm_launch(h, ctypes.c_void_p(side.cuda_stream))
    g.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    ggpu = e0.elapsed_time(e1) / 500 * 1e3
    print(f"{s}^3: host {1e6 * (t1 - t0) / n:.1f} us/launch, stream {gpu:.1f} us/launch, "
          f"graph {ggpu:.1f} us/launch ({2 * s ** 3 / (ggpu * 1e-6) / 1e12:.0f} TFLOP/s)", flush=True)
    lib.um_gemm_destroy(h)
