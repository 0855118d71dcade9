"""ExecConfig.graph_replay: small multiplies repeated on the same (A, B, C,
config) switch to one CUDA-graph replay on their third call.

Integer inputs: every call must give exactly a @ b (C zeroed before each,
since a replicated C keeps partials in its non-origin replicas),
and the reference-model counters must grow by one multiply per call, as for
the eager path (runtime.py:339-387)."""

import dataclasses

import numpy as np
import pytest
import torch

from paper_2510_08874_b200 import ExecConfig, execute_multiply
from paper_2510_08874_b200 import engine as eng
from paper_2510_08874_b200 import runtime as rt
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.graphs import CapturedMultiply
from paper_2510_08874_b200.schedule import schedule_cache

pytestmark = pytest.mark.gpu


def _graphs(A, B, C):
    return [v for v in schedule_cache(A, B, C).values() if isinstance(v, CapturedMultiply)]


@pytest.mark.parametrize("case", [
    (1024, 1024, 1024, 4, "2d", "2d", "2d", 1, 1, 1),      # cfg1 (BASELINE configs[0]) on the device
    (384, 320, 512, 4, "2d", "col", "2d", 1, 1, 2),        # replicated C (K4 inside the graph)
    (512, 384, 640, 8, "2d", "col", "row", 1, 1, 1),       # mismatched partitionings, 8 ranks
])
def test_repeated_small_multiply_replays_exactly(cuda, case):
    m, n, k, p, ap, bp, cp, ca, cb, cc = case
    fab, A, B, C, a, b = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=41)
    cfg = ExecConfig()
    ref = a @ b
    execute_multiply(A, B, C, cfg)
    torch.cuda.synchronize()
    bytes1, flops1 = fab.counters.bytes.copy(), fab.counters.flops.copy()
    stats1 = None
    for call in range(2, 7):
        C.zero_()
        stats = execute_multiply(A, B, C, cfg)
        assert np.array_equal(C.gather(0), ref), f"call {call}"
        assert len(_graphs(A, B, C)) == (1 if call > rt.GRAPH_AFTER else 0)
        stats1 = stats1 or stats
        assert [s.executed_ops for s in stats.values()] == [s.executed_ops for s in stats1.values()]
        assert all(stats[r].flops == int(fab.counters.flops[r]) for r in stats)
    assert np.array_equal(fab.counters.bytes, 6 * bytes1)
    assert np.array_equal(fab.counters.flops, 6 * flops1)


def test_graph_replay_off_and_size_limit(cuda, monkeypatch):
    fab, A, B, C, a, b = build_problem(384, 320, 512, 4, "2d", "col", "2d", 1, 1, 1, seed=43)
    off = ExecConfig(graph_replay=False)
    for _ in range(4):
        execute_multiply(A, B, C, off)
    assert not _graphs(A, B, C)
    monkeypatch.setattr(rt, "GRAPH_MAX_FLOPS", 2 * 384 * 320 * 512 - 1)
    for _ in range(4):
        execute_multiply(A, B, C, ExecConfig())
    assert not _graphs(A, B, C)
    monkeypatch.setattr(rt, "GRAPH_MAX_FLOPS", 2 * 384 * 320 * 512)
    C.zero_()
    for _ in range(4):
        execute_multiply(A, B, C, ExecConfig())
    assert len(_graphs(A, B, C)) == 1
    assert np.array_equal(C.gather(0), 4 * (a @ b))


def test_graph_replay_skipped_while_tracing_and_per_config(cuda):
    """Launch tracing (per-launch events) needs the eager path; a different
    config is a different graph."""
    fab, A, B, C, a, b = build_problem(384, 320, 512, 4, "2d", "col", "2d", 1, 1, 1, seed=47)
    eng.TRACE_ENABLED = True
    try:
        for _ in range(4):
            execute_multiply(A, B, C, ExecConfig())
    finally:
        eng.TRACE_ENABLED = False
        eng.TRACE.clear()
    assert not _graphs(A, B, C)
    cfg_b = dataclasses.replace(ExecConfig(), chain_order=False)
    for _ in range(3):
        execute_multiply(A, B, C, ExecConfig())
        execute_multiply(A, B, C, cfg_b)
    assert len(_graphs(A, B, C)) == 2
    torch.cuda.synchronize()
    assert np.array_equal(C.gather(0), 10 * (a @ b))


def test_failed_capture_stays_eager(cuda, monkeypatch):
    """A multiply whose capture fails keeps running eagerly, exactly, with
    counters of one multiply per call (the failed capture's host-side
    counting is rolled back)."""
    fab, A, B, C, a, b = build_problem(384, 320, 512, 4, "2d", "col", "2d", 1, 1, 2, seed=53)

    def boom(self, A_, *args, **kwargs):
        A_.fabric.counters.add_traffic(0, 1, 12345)        # host-side counting ran, then the capture failed
        raise RuntimeError("capture refused")

    monkeypatch.setattr(CapturedMultiply, "__init__", boom)
    execute_multiply(A, B, C, ExecConfig())
    torch.cuda.synchronize()
    bytes1 = fab.counters.bytes.copy()
    for _ in range(4):
        C.zero_()
        execute_multiply(A, B, C, ExecConfig())
        assert np.array_equal(C.gather(0), a @ b)
    assert not _graphs(A, B, C)
    assert np.array_equal(fab.counters.bytes, 5 * bytes1)
