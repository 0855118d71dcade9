"""One cuBLAS launch at a shape after warm-up, for ncu (kernel name = tile config):
    python tools/cublas_once.py M N K bf16|f32beta1"""
import sys

import torch

m, n, k = (int(x) for x in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "bf16"
a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
b = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
c = torch.zeros(m, n, device="cuda")
for _ in range(3):
    if mode == "bf16":
        torch.matmul(a, b)
    else:
        torch.addmm(c, a, b, out_dtype=torch.float32, out=c)
torch.cuda.synchronize()
print("done", mode)
