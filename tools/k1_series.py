"""Per-launch time series of K1 vs cuBLASLt (bf16 x bf16 -> fp32, beta = 1) on
one shape, with the SM clock the kernels actually ran at (a one-warp
clock64 / globaltimer sampler co-resident with the GEMM: `kernel_mhz`) and
NVML's view (`sm_mhz`, `watts`).  TFLOP/s per GHz separates kernel
efficiency from the power cap.

    python tools/k1_series.py [--shape 8192x8192x8192] [--iters 40] [--blocks 4] [--impls k1,lt]

(the clock probe is tools/debug/clk_probe.so: make -C tools/debug)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="8192x8192x8192")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--json", default=None)
    ap.add_argument("--impls", default="k1,lt")
    args = ap.parse_args()
    import threading
    import time
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        clk = lambda: (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),  # noqa: E731
                       pynvml.nvmlDeviceGetPowerUsage(h) // 1000)
    except Exception:  # noqa: BLE001
        clk = lambda: (-1, -1)  # noqa: E731
    samples, stop = [], threading.Event()

    def sampler():
        while True:
            samples.append(clk())
            if stop.wait(0.002):
                return
    lib = C.load()
    torch.cuda.set_device(0)
    # in-kernel SM clock: a one-warp sampler co-resident with the GEMMs
    probe = None
    so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "debug", "clk_probe.so")
    if os.path.exists(so):
        probe = ctypes.CDLL(so)
        pbuf = torch.zeros(2 * 65536, dtype=torch.int64, device="cuda")
        pcnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        pstop = torch.zeros(1, dtype=torch.int32).pin_memory()
        pstream = torch.cuda.Stream()

    def probe_start():
        if probe is None:
            return
        pstop.zero_()
        probe.clk_probe_launch(ctypes.c_void_p(pbuf.data_ptr()), 65536, 20000, ctypes.c_void_p(pstop.data_ptr()),
                               ctypes.c_void_p(pcnt.data_ptr()), ctypes.c_void_p(pstream.cuda_stream))

    def probe_stop():
        if probe is None:
            return None
        pstop.fill_(1)
        pstream.synchronize()
        n = int(pcnt.item())
        v = pbuf[: 2 * n].view(n, 2).cpu().tolist()
        f = [(c1 - c0) / (t1 - t0) * 1e3 for (t0, c0), (t1, c1) in zip(v, v[1:]) if t1 > t0]
        return round(statistics.median(f)) if f else None
    m, n, k = (int(x) for x in args.shape.split("x"))
    a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
    c = torch.zeros(m, n, device="cuda")
    va = C.UmView(a.data_ptr(), 0, m, 0, k, a.stride(0), C.UM_BF16, 0)
    vb = C.UmView(b.data_ptr(), 0, k, 0, n, b.stride(0), C.UM_BF16, 0)
    vc = C.UmView(c.data_ptr(), 0, m, 0, n, c.stride(0), C.UM_F32, 0)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    impls = {
        "k1": lambda: lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s),
        "lt": lambda: torch.addmm(c, a, b, out_dtype=torch.float32, out=c),
    }
    flops = 2.0 * m * n * k
    out = {"shape": args.shape, "blocks": []}
    order = args.impls.split(",")
    for blk in range(args.blocks):
        for name in (order if blk % 2 == 0 else order[::-1]):
            fn = impls[name]
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            samples.clear()
            stop.clear()
            th = threading.Thread(target=sampler)
            th.start()
            probe_start()
            evs = []
            for _ in range(args.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                evs.append((e0, e1))
            torch.cuda.current_stream().synchronize()
            kmhz = probe_stop()
            stop.set()
            th.join()
            time.sleep(0.2)
            tf = [flops / (x.elapsed_time(y) * 1e-3) / 1e12 for x, y in evs]
            rec = {"impl": name, "kernel_mhz": kmhz, "sm_mhz": statistics.median([x[0] for x in samples]) if samples else None,
                   "watts": max([x[1] for x in samples]) if samples else None, "median": statistics.median(tf), "best": max(tf),
                   "tflops": [round(v) for v in tf]}
            out["blocks"].append(rec)
            print(json.dumps(rec), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
