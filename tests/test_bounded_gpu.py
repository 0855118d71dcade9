"""Bounded staging (ExecConfig.pool_capacity / prefetch_depth /
max_inflight_gemms): the reference's bounded-asynchrony discipline
(runtime.py:43-73,186-231) on the device — results exact, staging memory and
ops in flight bounded, evicted slices pulled again."""

import numpy as np
import pytest
import torch

from paper_2510_08874_b200 import ExecConfig, Stationarity, execute_multiply
from paper_2510_08874_b200.cli import build_problem

pytestmark = pytest.mark.gpu

# cfg5-class (A 2D 2x4, B col, C row) scaled to 2048^3, and cfg4-class (2.5D c=2)
CASES = [(2048, 2048, 2048, 8, "2d", "col", "row", 1, 1, 1),
         (1536, 1024, 2048, 8, "2d", "2d", "2d", 2, 2, 2)]


@pytest.mark.parametrize("case", CASES, ids=["cfg5-class", "cfg4-class"])
@pytest.mark.parametrize("cap,depth,inflight", [(3, 2, 4), (4, 1, 1), (11, 2, 4)])
def test_bounded_pool_exact_and_bounded(cuda, case, cap, depth, inflight):
    m, n, k, p, ap, bp, cp, ca, cb, cc = case
    fab, A, B, C, a, b = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=41)
    free = execute_multiply(A, B, C, ExecConfig())
    assert np.array_equal(C.gather(0), a @ b)
    C.zero_()
    cfg = ExecConfig(pool_capacity=cap, prefetch_depth=depth, max_inflight_gemms=inflight)
    for _ in range(2):                      # the plan is built once and replayed
        C.zero_()
        stats = execute_multiply(A, B, C, cfg)
        torch.cuda.synchronize()
        assert np.array_equal(C.gather(0), a @ b)
    for r, st in stats.items():
        assert st.pool_peak <= cap
        assert st.peak_ops_per_launch <= min(inflight, depth + 1)
        # every slot is one op's largest operand slice: staging bounded by the pool
        max_slice = max(max(len(op.m_bound) * len(op.k_bound), len(op.k_bound) * len(op.n_bound))
                        for op in st.executed_ops) if st.executed_ops else 0
        assert st.staged_bytes <= cap * max(1, max_slice) * 2 + cap * 1024 * 16     # + pitch padding
        if free[r].gets:
            assert st.gets >= free[r].gets               # evicted slices are pulled again
        assert [o.a_tile for o in st.executed_ops] == [o.a_tile for o in free[r].executed_ops]


def test_bounded_pool_bounds_staging_below_fetch_once(cuda):
    """cfg5-class at p = 8: fetch-once staging holds every remote slice of a rank
    (3 A slices + 7 B tiles); a 3-slot pool holds three op-sized slices."""
    fab, A, B, C, a, b = build_problem(2048, 2048, 2048, 8, "2d", "col", "row", seed=43)
    free = execute_multiply(A, B, C, ExecConfig())
    C.zero_()
    bounded = execute_multiply(A, B, C, ExecConfig(pool_capacity=3))
    assert np.array_equal(C.gather(0), a @ b)
    for r in range(8):
        assert bounded[r].staged_bytes < free[r].staged_bytes
        assert bounded[r].pool_peak <= 3


def test_bounded_pool_stationary_a(cuda):
    """Remote C (Stationary A: fused peer accumulates) under a bounded pool."""
    fab, A, B, C, a, b = build_problem(768, 640, 1024, 4, "2d", "col", "2d", seed=47)
    execute_multiply(A, B, C, ExecConfig(stationarity=Stationarity.STATIONARY_A, pool_capacity=3))
    assert np.array_equal(C.gather(0), a @ b)
