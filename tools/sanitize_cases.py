"""Small representative device paths for compute-sanitizer (memcheck /
racecheck / synccheck): K1 edge shapes, the fused get -> GEMM launch with
chunk-level waits, copy-engine pulls + arrival flags, fused remote
accumulates (Stationary A), the overlapped and the barrier replica
reduction (K4), bounded staging, and K3 / K2' / K5 through the C-ABI.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08874_b200 import ExecConfig, Stationarity, execute_multiply, kernels  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402


def check(tag, got, ref):
    ok = np.array_equal(got, ref)
    print(f"{tag}: {'OK' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


def main():
    g = torch.Generator(device="cuda").manual_seed(3)
    for m, n, k in ((7, 9, 5), (256, 256, 256), (300, 520, 200)):
        a = torch.randint(-8, 9, (m, k), generator=g, device="cuda").to(torch.bfloat16)
        b = torch.randint(-8, 9, (k, n), generator=g, device="cuda").to(torch.bfloat16)
        c = torch.zeros(m, n, device="cuda")
        kernels.gemm_accumulate(a, b, c)
        check(f"K1 {m}x{n}x{k}", c.cpu().numpy(), (a.double() @ b.double()).cpu().numpy())
    cases = [
        ("fused gets cfg1-class p=4", (512, 512, 512, 4, "2d", "2d", "2d", 1, 1, 1), {}),
        ("copy-engine pulls + flags", (512, 512, 512, 4, "2d", "2d", "2d", 1, 1, 1), dict(get_engine="ce")),
        ("mismatched p=8 (chains, bands)", (512, 512, 512, 8, "2d", "col", "row", 1, 1, 1), {}),
        ("stationary A (fused peer accumulate)", (384, 320, 512, 4, "2d", "col", "2d", 1, 1, 1),
         dict(stationarity=Stationarity.STATIONARY_A)),
        ("replicated C, overlapped K4", (512, 512, 512, 4, "2d", "2d", "2d", 1, 1, 2), {}),
        ("replicated C, barrier K4", (512, 512, 512, 4, "2d", "2d", "2d", 1, 1, 2), dict(overlap_reduce=False)),
        ("bounded staging", (512, 512, 512, 8, "2d", "col", "row", 1, 1, 1), dict(pool_capacity=3)),
    ]
    for tag, case, kw in cases:
        fab, A, B, C, a, b = build_problem(*case, seed=5)
        execute_multiply(A, B, C, ExecConfig(**kw))
        check(tag, C.gather(0), a @ b)
    print("ALL OK", flush=True)


if __name__ == "__main__":
    main()
