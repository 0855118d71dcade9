"""C++ planner (um_plan via the C-ABI) is bit-exact with the reference's opgen.

CPU only: the planner needs no GPU.  Golden rows come from the real
reference (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2510_08874_b200 import Fabric, Stationarity, opgen
from paper_2510_08874_b200.cli import resolve_partition
from paper_2510_08874_b200.distmatrix import DistributedMatrix
from paper_2510_08874_b200.errors import ConfigError, ContractError
from paper_2510_08874_b200.tiling import Bounds2D, PartitionSpec, Range, Shape2D, TileIdx, col_block

STAT = {"a": Stationarity.STATIONARY_A, "b": Stationarity.STATIONARY_B, "c": Stationarity.STATIONARY_C}


def placement(cfg):
    fab = Fabric(cfg["p"], devices=[])
    out = {}
    for name, shape, desc, c in (("A", (cfg["m"], cfg["k"]), cfg["a_part"], cfg["c_a"]),
                                 ("B", (cfg["k"], cfg["n"]), cfg["b_part"], cfg["c_b"]),
                                 ("C", (cfg["m"], cfg["n"]), cfg["c_part"], cfg["c_c"])):
        out[name] = DistributedMatrix(fab, name, Shape2D(*shape),
                                      resolve_partition(desc, Shape2D(*shape), cfg["p"] // c), c)
    return out


def plan(cfg):
    M = placement(cfg)
    return [opgen.plan_rows(M["A"].desc(), M["B"].desc(), M["C"].desc(), cfg["p"], STAT[cfg["stat"]], r).tolist()
            for r in range(cfg["p"])]


def digest(per_rank):
    h = hashlib.sha256()
    for r, rows in enumerate(per_rank):
        for row in rows:
            h.update((f"{r}:" + ",".join(map(str, row)) + "\n").encode())
    return h.hexdigest()[:16]


def test_sweep_matches_reference(oplists):
    for e in oplists["sweep"]:
        rows = plan(e["cfg"])
        assert [len(r) for r in rows] == e["nops"], e["cfg"]
        assert digest(rows) == e["digest"], e["cfg"]


def test_baseline_configs_match_reference(oplists):
    for e in oplists["baseline"]:
        assert plan(e["cfg"]) == e["rows"], e["cfg"]


def test_baseline_format_digests(oplists):
    for e in oplists["baseline"]:
        cfg = e["cfg"]
        M = placement(cfg)
        lines = [f"rank {r}: {opgen.format_op(op)}" for r in range(cfg["p"])
                 for op in opgen.generate(STAT[cfg["stat"]], M["A"], M["B"], M["C"], r)]
        assert hashlib.sha256(("\n".join(lines) + "\n").encode()).hexdigest()[:16] == e["format_digest"]


def test_random_configs_match_reference(oplists):
    for e in oplists["random"]:
        if "error" in e:
            with pytest.raises((ConfigError, ValueError)):
                plan(e["cfg"])
            continue
        assert plan(e["cfg"]) == e["rows"], e["cfg"]


def triples(ops):
    return [(i, l, j) for op in ops for i in range(op.m_bound.lo, op.m_bound.hi)
            for l in range(op.k_bound.lo, op.k_bound.hi) for j in range(op.n_bound.lo, op.n_bound.hi)]


@given(data=st.data())
@settings(max_examples=60, deadline=None)
def test_exact_cover_property(data):
    """Every (i,l,j) triple computed exactly once (test_opgen.py:221-249 property)."""
    p = data.draw(st.sampled_from([1, 2, 4, 6, 8, 12]))
    m, n, k = (data.draw(st.integers(1, 14)) for _ in range(3))
    stat = data.draw(st.sampled_from(list(Stationarity)))
    cs = {"A": 1, "B": 1, "C": 1}
    cs[stat.value.upper()] = data.draw(st.sampled_from([d for d in range(1, p + 1) if p % d == 0]))
    fab = Fabric(p, devices=[])
    mats = {}
    for name, shape in (("A", (m, k)), ("B", (k, n)), ("C", (m, n))):
        desc = data.draw(st.sampled_from(["row", "col", "2d", "misaligned"]))
        mats[name] = DistributedMatrix(fab, name, Shape2D(*shape),
                                       resolve_partition(desc, Shape2D(*shape), p // cs[name]), cs[name])
    cover = []
    for r in range(p):
        cover += triples(opgen.generate(stat, mats["A"], mats["B"], mats["C"], r))
    assert len(cover) == len(set(cover)) == m * n * k


def test_known_answers_from_reference_tests():
    # test_opgen.py:103-115 (aligned 4x4, Stationary C, rank 0)
    fab = Fabric(4, devices=[])
    part = PartitionSpec(Shape2D(2, 2), Shape2D(2, 2))
    A, B, C = (DistributedMatrix(fab, n, Shape2D(4, 4), part) for n in "ABC")
    ops = opgen.generate_stationary_c(A, B, C, 0)
    assert [(o.a_tile, o.b_tile, o.c_tile, (o.k_bound.lo, o.k_bound.hi)) for o in ops] == [
        (TileIdx(0, 0), TileIdx(0, 0), TileIdx(0, 0), (0, 2)),
        (TileIdx(0, 1), TileIdx(1, 0), TileIdx(0, 0), (2, 4))]
    assert all(o.a_local == Bounds2D(Range(0, 2), Range(0, 2)) for o in ops)
    # test_opgen.py:192-206: replicated A splits the inner work
    fab = Fabric(4, devices=[])
    A = DistributedMatrix(fab, "A", Shape2D(4, 4), PartitionSpec(Shape2D(4, 4), Shape2D(1, 1)), c=4)
    B = DistributedMatrix(fab, "B", Shape2D(4, 8), col_block(Shape2D(4, 8), 4))
    C = DistributedMatrix(fab, "C", Shape2D(4, 8), col_block(Shape2D(4, 8), 4))
    for r in range(4):
        assert sum(op.flops for op in opgen.generate_stationary_a(A, B, C, r)) == 2 * 4 * 4 * 8 // 4
    assert opgen.format_op(opgen.generate_stationary_c(
        *[DistributedMatrix(Fabric(1, devices=[]), n, Shape2D(1, 1), PartitionSpec(Shape2D(1, 1), Shape2D(1, 1)))
          for n in "ABC"], 0)[0]) == "a=(0,0) b=(0,0) c=(0,0) m=[0,1) k=[0,1) n=[0,1)"


def test_errors_map_to_reference_exceptions():
    fab = Fabric(1, devices=[])
    p1 = PartitionSpec(Shape2D(4, 4), Shape2D(1, 1))
    A = DistributedMatrix(fab, "A", Shape2D(4, 4), p1)
    B = DistributedMatrix(fab, "B", Shape2D(3, 4), PartitionSpec(Shape2D(3, 4), Shape2D(1, 1)))
    C = DistributedMatrix(fab, "C", Shape2D(4, 4), p1)
    with pytest.raises(ConfigError):
        opgen.generate_stationary_c(A, B, C, 0)
    with pytest.raises(ContractError):
        opgen.global_to_local(Bounds2D(Range(3, 4), Range(0, 1)), Bounds2D(Range(0, 3), Range(0, 4)))
    with pytest.raises(ValueError):
        opgen.restrict_for_replication(Range(0, 4), 2, 2)
    from paper_2510_08874_b200.runtime import iteration_offset

    with pytest.raises(ValueError):
        iteration_offset(TileIdx(0, 0), 0)
    assert iteration_offset(TileIdx(1, 2), 4) == 3 and iteration_offset(TileIdx(3, 3), 4) == 2


def test_plan_is_cached_and_deterministic():
    fab = Fabric(4, devices=[])
    part = PartitionSpec(Shape2D(2, 2), Shape2D(2, 2))
    A, B, C = (DistributedMatrix(fab, n, Shape2D(4, 4), part) for n in "ABC")
    for s in Stationarity:
        assert opgen.generate(s, A, B, C, 1) == opgen.generate(s, A, B, C, 1)
