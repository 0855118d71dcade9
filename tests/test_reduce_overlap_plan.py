"""Host-side plan of the overlapped replica reduction (runtime._ReduceOverlap), on CPU.

Each C tile is cut into c * panels row sub-slices on 256-row boundaries; the
reducer of sub-slice k is the owner of replica k mod c; every rank's ops are
split exactly at the sub-slice rows and signal the sub-slice's flag; the
reducer waits for `expected` ops — which must equal the number of items that
will signal it (the pieces of one op along n count once), or the reduction
would start early or never."""

import pytest

from paper_2510_08874_b200 import ExecConfig
from paper_2510_08874_b200 import runtime as rt
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.fabric import Fabric, LinkTable


def problem(m, n, k, p, ap, bp, cp, ca, cb, cc):
    fab = Fabric(p, LinkTable.uniform(p, 1e9), devices=[])
    _, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, synthetic=True, fabric=fab)
    return A, B, C


@pytest.mark.parametrize("case,panels", [
    ((8192, 8192, 65536, 8, "col", "row", "2d", 1, 1, 8), 2),        # cfg3 at p=8
    ((16384, 16384, 16384, 8, "2d", "2d", "2d", 2, 2, 2), 2),        # cfg4 at p=8
    ((16384, 16384, 16384, 4, "2d", "2d", "2d", 2, 2, 2), 3),
    ((600, 520, 900, 4, "misaligned", "col", "row", 1, 1, 2), 1),
    ((3000, 700, 900, 6, "row", "2d", "custom:500:700", 1, 1, 3), 2),
])
def test_sub_slices_reducers_and_expected_signals(case, panels):
    A, B, C = problem(*case)
    cfg = ExecConfig(reduce_panels=panels)
    ovl = rt._ReduceOverlap(A, B, C, cfg)
    for t, subs in ovl.subs.items():
        rows = len(C.tile_bounds(t).rows)
        assert subs[0][0] == 0 and subs[-1][1] == rows
        for (r0, r1, rep), nxt in zip(subs, subs[1:] + [None]):
            assert r0 < r1 and (r0 % 256 == 0)
            if nxt:
                assert nxt[0] == r1
            assert 0 <= rep < C.c
    # count the items that will signal each sub-slice, over every rank's plan
    signalled = {}
    for r in range(C.p):
        sched = rt.lower_direct(A, B, C, cfg, r)
        sig = ovl.signals_for(sched)
        items, _, _ = rt.plan_bands(sched, [True] * len(sched.fetches), cfg, {i: c for i, (c, _) in sig.items()})
        # n-pieces of one (op, sub-slice) count once (um_gemm_op.done_piece)
        last = {(i, m0, m1): it for it, (i, _, m0, m1, *_) in enumerate(items)}
        for it, (i, t_, m0, m1, n0, n1, k0, k1) in enumerate(items):
            if last[(i, m0, m1)] != it:
                continue
            op = sched.ops[i]
            lo = op.c_local.rows.lo
            key = (op.c_tile, ovl.sub_slice_of(op.c_tile, lo + m0))
            r0, r1, _ = ovl.subs[op.c_tile][key[1]]
            assert r0 <= lo + m0 and lo + m1 <= r1            # an item never straddles two sub-slices
            signalled[key] = signalled.get(key, 0) + 1
    assert signalled == {k_: v for k_, v in ovl.expected.items() if v}


def test_row_sliced_op_raster_order():
    """cfg3 at p = 8: each rank's 8192^3 op, cut at the reducers' row
    sub-slices, is also cut into 2048-column pieces and walked piece-major
    inside four groups of row slices: the pieces tile the op exactly once,
    and the row-slice groups complete one after the other."""
    from paper_2510_08874_b200 import schedule as sch

    A, B, C = problem(8192, 8192, 65536, 8, "col", "row", "2d", 1, 1, 8)
    cfg = ExecConfig(reduce_panels=4)
    ovl = rt._ReduceOverlap(A, B, C, cfg)
    sched = rt.lower_direct(A, B, C, cfg, 0)
    sig = ovl.signals_for(sched)
    items, _, _ = rt.plan_bands(sched, [True] * len(sched.fetches), cfg, {i: c for i, (c, _) in sig.items()})
    op = sched.ops[0]
    mlen, nlen = len(op.m_bound), len(op.n_bound)
    cells = [(m0, m1, n0, n1) for (_, _, m0, m1, n0, n1, _, _) in items]
    assert sum((m1 - m0) * (n1 - n0) for m0, m1, n0, n1 in cells) == mlen * nlen
    assert len(set(cells)) == len(cells)
    assert {n1 - n0 for _, _, n0, n1 in cells} == {sch._RASTER_N}
    rows = sorted({(m0, m1) for m0, m1, _, _ in cells})
    group = {r: g * 4 // len(rows) for g, r in enumerate(rows)}       # quarter of the row slices
    seq = [group[(m0, m1)] for m0, m1, _, _ in cells]
    assert seq == sorted(seq)                                          # groups in order
    first = cells[: len(rows) // 4]
    assert len({(n0, n1) for _, _, n0, n1 in first}) == 1              # piece-major inside a group
