"""Host-side planning of the in-kernel pulls (runtime.plan_bands), on CPU.

The fused get -> GEMM launch lets every (sub-)op wait only for the bands of
the staged slices it reads; these tests pin the band/sub-op structure on the
BASELINE configurations and check, for random configurations, that the bands
are disjoint and cover every slice an op reads (so no op can start on data
that has not landed)."""

import random

import pytest

from paper_2510_08874_b200 import ExecConfig, Stationarity
from paper_2510_08874_b200 import runtime as rt
from paper_2510_08874_b200 import schedule as sch
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.fabric import Fabric, LinkTable


def problem(m, n, k, p, ap, bp, cp, ca=1, cb=1, cc=1):
    fab = Fabric(p, LinkTable.uniform(p, 1e9), devices=[])       # placement only: no device
    _, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, synthetic=True, fabric=fab)
    return A, B, C


def plan(A, B, C, r, **kw):
    cfg = ExecConfig(**kw)
    sched = rt.lower_direct(A, B, C, cfg, r)
    items, bands, need = rt.plan_bands(sched, [True] * len(sched.fetches), cfg)
    return sched, items, bands, need


def slice_of(sched, item):
    i, t, m0, m1, n0, n1, k0, k1 = item
    op = sched.ops[i]
    a, b = op.a_local, op.b_local
    return {sched.a_src[i]: (a.rows.lo + m0, a.rows.lo + m1, a.cols.lo + k0, a.cols.lo + k1),
            sched.b_src[i]: (b.rows.lo + k0, b.rows.lo + k1, b.cols.lo + n0, b.cols.lo + n1)}


def check_cover(sched, items, bands, need):
    for j, bl in enumerate(bands):
        for x in range(len(bl)):
            for y in range(x + 1, len(bl)):
                p, q = bl[x], bl[y]
                assert p[1] <= q[0] or q[1] <= p[0] or p[3] <= q[2] or q[3] <= p[2], "overlapping bands"
    for it, item in enumerate(items):
        for j, (r0, r1, c0, c1) in slice_of(sched, item).items():
            if j < 0:
                continue
            f = sched.fetches[j]
            r0, r1, c0, c1 = r0 - f.r0, r1 - f.r0, c0 - f.c0, c1 - f.c0
            got = [bands[j][k] for k in need[(it, j)]]
            area = sum((min(r1, b[1]) - max(r0, b[0])) * (min(c1, b[3]) - max(c0, b[2])) for b in got)
            assert area == (r1 - r0) * (c1 - c0), (item, j)          # the needed bands cover the slice
    # every sub-op of an op together covers the op exactly once
    per_op = {}
    for i, t, m0, m1, n0, n1, k0, k1 in items:
        per_op[i] = per_op.get(i, 0) + (m1 - m0) * (n1 - n0) * (k1 - k0)
    for i, op in enumerate(sched.ops):
        assert per_op[i] == len(op.m_bound) * len(op.n_bound) * len(op.k_bound)


def test_cfg5_p8_b_tiles_banded_into_k_slabs():
    A, B, C = problem(16384, 16384, 16384, 8, "2d", "col", "row")
    for r in range(8):
        sched, items, bands, need = plan(A, B, C, r)
        assert len(sched.fetches) == 10 and len(items) == 32
        for j, f in enumerate(sched.fetches):
            if f.mat == "B":
                assert bands[j] == [(4096 * q, 4096 * (q + 1), 0, 2048) for q in range(4)]   # 16 MiB k-slabs
            else:
                assert len(bands[j]) == 1
        assert all(len(need[(it, sched.b_src[i])]) == 1 for it, (i, *_rest) in enumerate(items)
                   if sched.b_src[i] >= 0)
        check_cover(sched, items, bands, need)


def test_cfg4_p8_whole_tile_op_split_into_a_grid():
    A, B, C = problem(16384, 16384, 16384, 8, "2d", "2d", "2d", 2, 2, 2)
    sched, items, bands, need = plan(A, B, C, 3)          # rank 3 pulls one A and one B tile (128 MiB each)
    assert len(sched.ops) == 1 and len(sched.fetches) == 2
    # both operands pulled: 4 x 4 sub-ops, row by row; each waits for one A row
    # band and one B column band (32 MiB each), the first for 1/4 of each pull
    q = [(0, 2048), (2048, 4096), (4096, 6144), (6144, 8192)]
    assert [(m0, m1, n0, n1) for _, _, m0, m1, n0, n1, _, _ in items] == [(*a, *b) for a in q for b in q]
    ja, jb = sched.a_src[0], sched.b_src[0]
    assert bands[ja] == [(r0, r1, 0, 8192) for r0, r1 in q] and bands[jb] == [(0, 8192, c0, c1) for c0, c1 in q]
    assert [need[(it, ja)] for it in range(16)] == [[it // 4] for it in range(16)]
    assert [need[(it, jb)] for it in range(16)] == [[it % 4] for it in range(16)]
    check_cover(sched, items, bands, need)
    # mn_split = 2: a 2 x 2 grid
    sched, items, bands, need = plan(A, B, C, 3, mn_split=2)
    assert len(items) == 4
    check_cover(sched, items, bands, need)
    # overlapped replica reduction: the op is cut at the reduction rows, and a
    # large pulled B along n as well
    cuts = [1024 * t for t in range(1, 8)]
    cfg = ExecConfig()
    items, bands, need = rt.plan_bands(sched, [True] * len(sched.fetches), cfg, {0: cuts})
    assert len(items) == 8 * 4
    assert [(m0, m1) for _, _, m0, m1, *_ in items[:5]] == [(0, 1024)] * 4 + [(1024, 2048)]
    assert bands[jb] == [(0, 8192, c0, c1) for c0, c1 in q]
    check_cover(sched, items, bands, need)
    # k split instead: A banded by columns, B by rows, one slab each
    sched, items, bands, need = plan(A, B, C, 3, k_split=4)
    assert [(k0, k1) for *_, k0, k1 in items] == [(0, 2048), (2048, 4096), (4096, 6144), (6144, 8192)]
    assert bands[sched.a_src[0]] == [(0, 8192, 2048 * q, 2048 * (q + 1)) for q in range(4)]
    assert bands[sched.b_src[0]] == [(2048 * q, 2048 * (q + 1), 0, 8192) for q in range(4)]
    check_cover(sched, items, bands, need)


@pytest.mark.parametrize("seed", range(16))
def test_random_configs_bands_cover_slices(seed, monkeypatch):
    monkeypatch.setattr(sch, "_SPLIT_BYTES", 1 << 10)
    monkeypatch.setattr(sch, "_SPLIT_MIN", 16)
    rnd = random.Random(seed)
    p = rnd.choice([2, 4, 6, 8, 12])
    m, n, k = (rnd.randint(8, 300) for _ in range(3))
    descs = ["row", "col", "2d", "misaligned", "custom:40:24", "custom:16:16:2:2:cyclic" if p % 4 == 0 else "2d"]
    reps = [c for c in (1, 2) if p % c == 0]
    ca, cb, cc = (rnd.choice(reps) for _ in range(3))

    def fits(d, c):
        return not d.startswith("custom:16:16:2:2") or (p // c) == 4

    ap, bp, cp = (rnd.choice([d for d in descs if fits(d, c)]) for c in (ca, cb, cc))
    A, B, C = problem(m, n, k, p, ap, bp, cp, ca, cb, cc)
    kw = rnd.choice([dict(), dict(k_split=3), dict(mn_split=0), dict(staging="tile")])
    for st in Stationarity:
        for r in range(p):
            sched, items, bands, need = plan(A, B, C, r, stationarity=st, **kw)
            check_cover(sched, items, bands, need)


def test_device_order_keeps_rotation_balance():
    """cfg5 at p = 8: the reference's rotation makes every schedule position a
    permutation of B owners (each rank pulls from a different peer,
    SURVEY §8(e)); the device order (k-chains grouped, plan_bands) keeps it."""
    A, B, C = problem(16384, 16384, 16384, 8, "2d", "col", "row")
    dev, ref = {}, {}
    for r in range(8):
        s, items, _, _ = plan(A, B, C, r)
        dev[r] = [B.owner_rank(s.ops[i].b_tile, 0) for i in dict.fromkeys(it[0] for it in items)]
        ref[r] = [B.owner_rank(op.b_tile, 0) for op in s.ops]
        assert sorted(dev[r]) == sorted(ref[r])
    for order in (dev, ref):
        for pos in range(len(order[0])):
            assert len({order[r][pos] for r in range(8)}) == 8, pos
