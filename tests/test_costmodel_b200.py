"""B200 path cost model (costmodel.ingress_bytes / pick_stationarity_b200), on CPU.

SURVEY.md §8(d, f-1) computed, with the reference planner, the max per-rank
ingress of each stationarity on the B200 path (fetch-once bf16 slices, fp32
accumulates, pull-to-origin reduction): cfg4 A/B/C = 640/640/512 MiB, cfg5
496/896/496 MiB — Stationary C best or tied in every BASELINE config."""

import pytest

from paper_2510_08874_b200 import costmodel
from paper_2510_08874_b200.cli import RunConfig, _build_problem_cfg, _resolve_stationarity
from paper_2510_08874_b200.opgen import Stationarity
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.fabric import Fabric, LinkTable

MiB = 1 << 20
ST = {"a": Stationarity.STATIONARY_A, "b": Stationarity.STATIONARY_B, "c": Stationarity.STATIONARY_C}


def problem(m, n, k, p, ap, bp, cp, ca=1, cb=1, cc=1):
    fab = Fabric(p, LinkTable.uniform(p, 1e9), devices=[])
    _, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, synthetic=True, fabric=fab)
    return A, B, C


@pytest.mark.parametrize("args,expect", [
    ((16384, 16384, 16384, 8, "2d", "2d", "2d", 2, 2, 2), {"a": 640, "b": 640, "c": 512}),   # cfg4
    ((16384, 16384, 16384, 8, "2d", "col", "row"), {"a": 496, "b": 896, "c": 496}),          # cfg5
    ((65536, 8192, 8192, 8, "row", "2d", "row", 1, 8, 1), {"a": 0, "b": 0, "c": 0}),         # cfg2
])
def test_max_ingress_matches_survey(args, expect):
    A, B, C = problem(*args)
    for s, mib in expect.items():
        assert max(costmodel.ingress_bytes(A, B, C, ST[s], distributed_reduce=False)) == mib * MiB
    assert costmodel.pick_stationarity_b200(A, B, C) is Stationarity.STATIONARY_C


def test_distributed_reduction_spreads_ingress():
    A, B, C = problem(8192, 8192, 65536, 8, "col", "row", "2d", 1, 1, 8)                        # cfg3
    naive = costmodel.ingress_bytes(A, B, C, ST["c"], distributed_reduce=False)
    dist = costmodel.ingress_bytes(A, B, C, ST["c"])
    assert max(naive) == 7 * 256 * MiB and sum(naive) == sum(dist)
    assert max(dist) == 7 * 256 * MiB // 8
    assert costmodel.modeled_time(A, B, C, ST["c"]) < costmodel.modeled_time(A, B, C, ST["a"]) + 1e-12


def test_auto_b200_in_the_cli_grammar():
    cfg = RunConfig(p=8, m=16384, n=16384, k=16384, a_part="2d", b_part="col", c_part="row",
                    stationarity="auto-b200")
    cfg.validate()
    _, machine, A, B, C, _, _ = _build_problem_cfg(cfg, placement_only=True)
    assert _resolve_stationarity(cfg, A, B, C, machine) is Stationarity.STATIONARY_C
