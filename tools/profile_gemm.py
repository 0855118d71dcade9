"""Run the K1 GEMM on a cfg2-sized op (for ncu captures and raster/clock sweeps)."""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08874_b200 import kernels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=65536)
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=8192)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--time", action="store_true")
ap.add_argument("--cublas", action="store_true")
a = ap.parse_args()
A = (torch.rand(a.m, a.k, device="cuda") * 2 - 1).to(torch.bfloat16)
B = (torch.rand(a.k, a.n, device="cuda") * 2 - 1).to(torch.bfloat16)
C = torch.zeros(a.m, a.n, device="cuda")
fn = (lambda: torch.matmul(A, B)) if a.cublas else (lambda: kernels.gemm_accumulate(A, B, C))
for _ in range(3 if a.time else a.iters):
    fn()
torch.cuda.synchronize()
if a.time:
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    clk = sorted(float(x.split(",")[0]) for x in out if "," in x)
    pw = sorted(float(x.split(",")[1]) for x in out if "," in x)
    reasons = sorted({x.split(",")[2].strip() for x in out if x.count(",") >= 2})
    ms = e0.elapsed_time(e1) / a.iters
    print(f"{os.environ.get('UM_GEMM_GROUP', 'default'):>8} {'cublas' if a.cublas else 'k1':6} "
          f"{a.m}x{a.n}x{a.k}: {ms:.3f} ms {2 * a.m * a.n * a.k / ms / 1e9:.1f} TFLOP/s "
          f"sm_clk_med={clk[len(clk) // 2] if clk else 0:.0f} power_med={pw[len(pw) // 2] if pw else 0:.0f}W "
          f"n={len(clk)} reasons={reasons} epi={os.environ.get('UM_GEMM_EPI_DEBUG', 'reduce')}", flush=True)
else:
    print("done")
