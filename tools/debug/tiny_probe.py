import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_08874_b200 import kernels
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
def t(label, m, n, k, pa, pb, pc):
    A = torch.randint(-8, 9, (m, k + pa), device="cuda").to(torch.bfloat16)[:, :k]
    B = torch.randint(-8, 9, (k, n + pb), device="cuda").to(torch.bfloat16)[:, :n]
    C = torch.zeros(m, n + pc, device="cuda")[:, :n]
    torch.cuda.synchronize()
    t0 = time.perf_counter(); kernels.gemm_accumulate(A, B, C); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    ok = torch.equal(C, (A.double() @ B.double()).float())
    print(f"{label}: launch {1e3*(t1-t0):.1f} ms, sync {1e3*(t2-t1):.1f} ms ok={ok}", flush=True)
for i in range(2):
    t("aligned 128x256x64", 128, 256, 64, 0, 0, 0)
    t("tiny 7x9x5 unpadded", 7, 9, 5, 0, 0, 0)
    t("tiny 7x9x5 staged A", 7, 9, 5, 5, 7, 7)
    t("1x1x1 staged", 1, 1, 1, 5, 3, 7)
    t("300x200x100 staged", 300, 200, 100, 5, 3, 7)
