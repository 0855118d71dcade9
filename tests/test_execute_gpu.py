"""Whole multiplies through the C-ABI entry alone (um_execute / um_sync_all):
the serialised plans of every rank plus the replica-reduction steps, issued
by ONE C call per multiply (runtime.py:339-387 at the C boundary)."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2510_08874_b200 import ExecConfig, Stationarity, _capi
from paper_2510_08874_b200.cexec import CompiledMultiply
from paper_2510_08874_b200.cli import build_problem

pytestmark = pytest.mark.gpu

CASES = {
    "cfg1": (1024, 1024, 1024, 4, "2d", "2d", "2d", 1, 1, 1),          # BASELINE configs[0]: 2D x 3, p = 4
    "cfg1-replicated": (1024, 1024, 1024, 4, "2d", "2d", "2d", 1, 1, 2),
    "mismatched": (768, 640, 1024, 8, "2d", "col", "row", 1, 1, 1),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_c_entry_alone_replays_exactly(cuda, name):
    m, n, k, p, ap, bp, cp, ca, cb, cc = CASES[name]
    fab, A, B, C, a, b = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=59)
    cm = CompiledMultiply(A, B, C, ExecConfig())
    lib = _capi.load()
    for _ in range(3):
        C.zero_()
        torch.cuda.synchronize()                 # the C caller's own ordering: inputs ready
        # the whole multiply: one C call, then the C host barrier
        assert lib.um_execute(cm.plans, cm.nplans, cm.steps, cm.nsteps, ctypes.byref(cm.cfg_c)) == 0, \
            _capi.last_error()
        assert lib.um_sync_all() == 0
        assert np.array_equal(C.gather(0), a @ b)


def test_compiled_multiply_stream_ordered(cuda):
    """execute() joins torch's current stream: no host sync between zeroing,
    the multiply and the read-back."""
    fab, A, B, C, a, b = build_problem(*CASES["cfg1-replicated"], seed=61)
    cm = CompiledMultiply(A, B, C, ExecConfig(stationarity=Stationarity.STATIONARY_C))
    for _ in range(2):
        C.zero_()
        cm.execute()
        assert np.array_equal(C.gather(0), a @ b)
