"""The fair cuBLAS bar for K1 (VERDICT r1 "next" 3): on the same box and shapes,
time (a) torch.matmul bf16 x bf16 -> bf16 (MEASURED_PEAKS' denominator),
(b) torch.addmm(C, A, B, out_dtype=fp32): cuBLASLt bf16 x bf16 -> fp32 with
beta = 1, i.e. exactly the fp32 `C += A @ B` K1 does, and (c) K1 itself
(um_gemm_acc).  Runs interleaved rounds and reports best and median TFLOP/s.

    python tools/cublas_bar.py [--shapes 8192x8192x8192,...] [--iters 20] [--rounds 3] [--json out]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08874_b200 import _capi as C  # noqa: E402

SHAPES = "8192x8192x8192,65536x8192x8192,16384x16384x16384,8192x8192x65536,4096x4096x4096,2048x2048x4096"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=SHAPES)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    lib = C.load()
    torch.cuda.set_device(0)
    out = {}
    for shp in args.shapes.split(","):
        m, n, k = (int(x) for x in shp.split("x"))
        a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
        b = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
        c = torch.zeros(m, n, device="cuda")
        cb = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        va = C.UmView(a.data_ptr(), 0, m, 0, k, a.stride(0), C.UM_BF16, 0)
        vb = C.UmView(b.data_ptr(), 0, k, 0, n, b.stride(0), C.UM_BF16, 0)
        vc = C.UmView(c.data_ptr(), 0, m, 0, n, c.stride(0), C.UM_F32, 0)

        def k1():
            s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            C.check(lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s), "um_gemm_acc")

        impls = {
            "cublas_bf16_out": lambda: torch.matmul(a, b, out=cb),
            "cublaslt_f32_beta1": lambda: torch.addmm(c, a, b, out_dtype=torch.float32, out=c),
            "k1": k1,
        }
        res = {name: [] for name in impls}
        flops = 2.0 * m * n * k
        for _ in range(args.rounds):
            for name, fn in impls.items():
                try:
                    for _ in range(3):
                        fn()
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(args.iters):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        fn()
                        e1.record()
                        ts.append((e0, e1))
                    torch.cuda.synchronize()
                    res[name] += [flops / (x.elapsed_time(y) * 1e-3) / 1e12 for x, y in ts]
                except Exception as e:  # noqa: BLE001
                    res[name] = [f"error: {e}"]
        row = {}
        for name, v in res.items():
            if v and isinstance(v[0], float):
                row[name] = {"best": max(v), "median": statistics.median(v)}
            else:
                row[name] = v[:1]
        out[shp] = row
        print(shp, json.dumps(row), flush=True)
        del a, b, c, cb
        torch.cuda.empty_cache()
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
