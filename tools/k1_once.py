"""One K1 launch (after warm-up) at a shape, for ncu captures:
    python tools/k1_once.py 8192 8192 8192 [launches]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_08874_b200 import _capi as C  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
lib = C.load()
a = (torch.rand(m, k, device="cuda") * 2 - 1).to(torch.bfloat16)
b = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
c = torch.zeros(m, n, device="cuda")
va = C.UmView(a.data_ptr(), 0, m, 0, k, a.stride(0), C.UM_BF16, 0)
vb = C.UmView(b.data_ptr(), 0, k, 0, n, b.stride(0), C.UM_BF16, 0)
vc = C.UmView(c.data_ptr(), 0, m, 0, n, c.stride(0), C.UM_F32, 0)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(reps):
    C.check(lib.um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc), s), "um_gemm_acc")
torch.cuda.synchronize()
print("done", m, n, k)
