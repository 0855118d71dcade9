"""Standalone K1 probe: correctness on edge cases + throughput (dev tool)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_08874_b200 import _capi as C

lib = C.load()
dev = 0
torch.cuda.set_device(dev)

def v(t, r0, r1, c0, c1, dt):
    return C.UmView(t.data_ptr(), r0, r1, c0, c1, t.stride(0), dt, dev)

def run(m, n, k, off=(0, 0, 0, 0, 0, 0), pad=(0, 0, 0), real=False):
    ar0, ac0, br0, bc0, cr0, cc0 = off
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    def mk(rows, cols, dt):
        pitch = ((cols + 7) // 8) * 8 + 8 * pad[0]
        if real:
            t = torch.rand(rows, pitch, device="cuda", generator=g) * 2 - 1
        else:
            t = torch.randint(-8, 9, (rows, pitch), device="cuda", generator=g).float()
        return t.to(dt)
    A = mk(ar0 + m, ac0 + k, torch.bfloat16)
    B = mk(br0 + k, bc0 + n, torch.bfloat16)
    Cm = mk(cr0 + m, cc0 + n, torch.float32)
    ref = Cm.clone()
    ref[cr0:cr0 + m, cc0:cc0 + n] += A[ar0:ar0 + m, ac0:ac0 + k].float() @ B[br0:br0 + k, bc0:bc0 + n].float()
    va, vb, vc = v(A, ar0, ar0 + m, ac0, ac0 + k, 0), v(B, br0, br0 + k, bc0, bc0 + n, 0), v(Cm, cr0, cr0 + m, cc0, cc0 + n, 1)
    rc = lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc:
        print("ERR", C.last_error()); return False
    torch.cuda.synchronize()
    if real:
        err = ((Cm - ref).abs().max() / (ref.abs().max() + 1e-6)).item()
        ok = err < 1e-5
    else:
        ok = torch.equal(Cm, ref)
        err = (Cm - ref).abs().max().item()
    print(f"m={m} n={n} k={k} off={off} real={real}: {'OK' if ok else 'FAIL'} maxerr={err}", flush=True)
    if not ok:
        d = (Cm - ref).abs() > 1e-3
        idx = d.nonzero()
        print("  bad count", d.sum().item(), "first", idx[:8].tolist())
    return ok

def perf(m, n, k, iters=10):
    A = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    B = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
    Cm = torch.zeros(m, n, device="cuda")
    va, vb, vc = v(A, 0, m, 0, k, 0), v(B, 0, k, 0, n, 0), v(Cm, 0, m, 0, n, 1)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2 * m * n * k / ms / 1e9
    # cuBLAS reference for context
    A2 = A; B2 = B
    for _ in range(3): torch.matmul(A2, B2)
    torch.cuda.synchronize(); e0.record()
    for _ in range(iters): torch.matmul(A2, B2)
    e1.record(); torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / iters
    print(f"PERF m={m} n={n} k={k}: {ms:.3f} ms {tf:.1f} TFLOP/s | cuBLAS bf16-out {ms2:.3f} ms {2*m*n*k/ms2/1e9:.1f} TFLOP/s", flush=True)

if __name__ == "__main__":
    cg = os.environ.get("UM_GEMM_CG", "2")
    print("CG", cg, C.load().um_version().decode())
    ok = True
    ok &= run(128, 256, 64)
    ok &= run(256, 256, 64)
    ok &= run(256, 512, 128)
    ok &= run(7, 9, 5)
    ok &= run(1000, 1000, 1000)
    ok &= run(300, 200, 100, off=(5, 3, 7, 11, 2, 1))
    ok &= run(1024, 1024, 4096, real=True)
    ok &= run(2048, 4096, 2048, off=(2048, 0, 0, 0, 0, 0))
    print("ALL_OK" if ok else "SOME_FAIL", flush=True)
    if ok:
        perf(4096, 4096, 4096)
        perf(8192, 8192, 8192)
        perf(65536, 8192, 8192, iters=5)
