"""K1 compile-time / launch-time variants selected by library knobs give the
same exact results as the default (integer inputs, C += A.B).

Each variant runs in a subprocess (the knobs are read once per process):
one large single op (NT=512 pair tiles, L2 hints), a ragged op, and a batch
of k-chunk ops sharing one C region (k-chains, capped by UM_GEMM_CHAIN_WAVES).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import ctypes, sys, torch
sys.path.insert(0, '.')
from paper_2510_08874_b200 import _capi as C, kernels
lib = C.load()
g = torch.Generator(device='cuda').manual_seed(11)
def ints(r, c):
    return torch.randint(-8, 9, (r, c), generator=g, device='cuda').to(torch.bfloat16)
def view(t, r0, r1, c0, c1, dt):
    return C.UmView(t.data_ptr(), r0, r1, c0, c1, t.stride(0), dt, 0)
for m, n, k in ((8192, 4096, 512), (1000, 1000, 1000)):
    a, b = ints(m, k), ints(k, n)
    c = torch.randint(-8, 9, (m, n), generator=g, device='cuda').float()
    ref = c.double() + a.double() @ b.double()
    kernels.gemm_accumulate(a, b, c)
    assert torch.equal(c.double(), ref), (m, n, k)
# 8 ops accumulating k-chunks of one product into the same C (one launch)
m, n, k, parts = 2048, 2048, 4096, 8
a, b = ints(m, k), ints(k, n)
c = torch.zeros(m, n, device='cuda')
kc = k // parts
ops = (C.UmGemmOp * parts)(*[C.UmGemmOp(view(a, 0, m, i * kc, (i + 1) * kc, C.UM_BF16),
                                        view(b, i * kc, (i + 1) * kc, 0, n, C.UM_BF16),
                                        view(c, 0, m, 0, n, C.UM_F32), 0) for i in range(parts)])
C.check(lib.um_gemm_acc_batch(ops, parts, 0, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), 'batch')
torch.cuda.synchronize()
assert torch.equal(c.double(), a.double() @ b.double())
# a fused launch with in-kernel gets (tail split acts on these), k-chains and bands
import numpy as np
from paper_2510_08874_b200 import ExecConfig, execute_multiply
from paper_2510_08874_b200.cli import build_problem
for case in ((2048, 2048, 2048, 8, "2d", "col", "row", 1, 1, 1), (1536, 1024, 2048, 8, "2d", "2d", "2d", 2, 2, 2)):
    fab, A, B, C_, a_, b_ = build_problem(*case, seed=71)
    for _ in range(2):
        C_.zero_()
        execute_multiply(A, B, C_, ExecConfig(get_engine="kernel"))
        assert np.array_equal(C_.gather(0), a_ @ b_), case
print('OK')
"""

PROF_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_08874_b200", "_lib",
                        "libunimul_b200_prof.so")
# variants measured and rejected in round 1 exist only in the profiling build
PROF_ONLY = ("UM_GEMM_PAIRS", "UM_GEMM_EPI_WARPS", "UM_GEMM_CG", "UM_GEMM_EPI_DEBUG")


@pytest.mark.parametrize("env", [
    {},
    {"UM_GEMM_PAIRS": "2"},                              # clusters of 2 pairs, B multicast (preferred 4)
    {"UM_GEMM_PAIRS": "4"},                              # preferred clusters of 8
    {"UM_GEMM_PAIRS": "4", "UM_GEMM_PAIRS_FIXED": "1"},  # clusters of 8 only
    {"UM_GEMM_NT": "256"},
    {"UM_GEMM_NT": "128"},                               # narrow tiles everywhere (default: few-tile launches)
    {"UM_GEMM_EPI_WARPS": "8"},
    {"UM_GEMM_CHAIN_WAVES": "0"},                        # uncapped k-chains
    {"UM_GEMM_CHAIN": "0"},
    {"UM_GEMM_EPI_DEBUG": "red"},                        # red.global epilogue for local C
    {"UM_GEMM_APOL": "0", "UM_GEMM_BPOL": "0", "UM_GEMM_CPOL": "1"},
    {"UM_GEMM_TAIL_SPLIT": "1"},                         # last wave split along k (fused launches, gets)
    {"UM_GEMM_SKSTART": "0"},                            # no staggered start
    {"UM_GEMM_CG": "1"},                                 # cta_group::1 (profiling build)
    {"UM_GEMM_PDL": "0"},                                # without programmatic dependent launch
    {"UM_GEMM_SPLITK": "0"},                             # small launches without split-k
    {"UM_RASTER_N": "0"},                                # row-sliced ops walked row-major
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_variant_exact(env):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(env)
    if any(k in env for k in PROF_ONLY):
        env["UNIMUL_B200_LIB"] = PROF_LIB
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=dict(os.environ, **env), cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "OK" in out.stdout, (out.stdout[-1000:], out.stderr[-2000:])
