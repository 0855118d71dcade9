"""A/B of K1 launch-time knobs: each (env setting) runs in its own process
(knobs are read once per process), interleaved over rounds; prints best and
median TFLOP/s per shape.

    python tools/k1_ab.py --env "UM_GEMM_SKSTART=0" --env "UM_GEMM_SKSTART=1" [--shapes 8192x8192x8192,...]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import ctypes, json, sys, torch
sys.path.insert(0, %r)
from paper_2510_08874_b200 import _capi as C
lib = C.load()
out = {}
for shp in %r.split(","):
    m, n, k = (int(x) for x in shp.split("x"))
    a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
    c = torch.zeros(m, n, device="cuda")
    va = C.UmView(a.data_ptr(), 0, m, 0, k, a.stride(0), C.UM_BF16, 0)
    vb = C.UmView(b.data_ptr(), 0, k, 0, n, b.stride(0), C.UM_BF16, 0)
    vc = C.UmView(c.data_ptr(), 0, m, 0, n, c.stride(0), C.UM_F32, 0)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(%d):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    out[shp] = [2.0 * m * n * k / (x.elapsed_time(y) * 1e-3) / 1e12 for x, y in ts]
    del a, b, c
    torch.cuda.empty_cache()
print(json.dumps(out))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", action="append", default=[])
    ap.add_argument("--shapes", default="8192x8192x8192,4096x4096x4096,16384x16384x16384,2048x2048x4096")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    envs = args.env or [""]
    res = {e: {} for e in envs}
    for _ in range(args.rounds):
        for e in envs:
            env = dict(os.environ)
            for kv in filter(None, e.split(",")):
                k, v = kv.split("=")
                env[k] = v
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, args.shapes, args.iters)], env=env,
                                 capture_output=True, text=True, timeout=600)
            if out.returncode:
                print(e, "FAILED", out.stderr[-2000:])
                continue
            for shp, v in json.loads(out.stdout.strip().splitlines()[-1]).items():
                res[e].setdefault(shp, []).extend(v)
    summary = {}
    for e, d in res.items():
        for shp, v in d.items():
            summary.setdefault(shp, {})[e or "default"] = {"best": max(v), "median": statistics.median(v)}
    for shp, d in summary.items():
        print(shp, "  ".join(f"{e}: best {x['best']:.0f} med {x['median']:.0f}" for e, x in d.items()), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
