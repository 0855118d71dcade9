"""Generate the golden fixtures by running the REAL reference (unimul).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only, not
copied) and records its outputs for the hot path:

  oplists.json   opgen.generate op rows (all LocalMatMulOp fields) for the
                 acceptance-sweep configs (digests), the BASELINE configs and
                 random configs (full rows), plus Appendix-C format_op digests
  numeric.npz    execute_multiply / run_direct results (per replica) on
                 integer and bf16-rounded real inputs
  runtime.json   RunStats request orders, FabricCounters bytes/msgs/flops,
                 lower_greedy IR programs and validate() verdicts

The fixtures are committed; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from unimul import kernels, lowering, opgen, runtime  # noqa: E402
from unimul.cli import RunConfig, build_problem, resolve_partition  # noqa: E402
from unimul.distmatrix import DistributedMatrix  # noqa: E402
from unimul.fabric import AccumulateMode, Fabric  # noqa: E402
from unimul.opgen import Stationarity  # noqa: E402
from unimul.tiling import Shape2D  # noqa: E402

# numpy GEMM backend: identical results on integer inputs, fast on big ones
kernels.gemm_accumulate = kernels.gemm_accumulate_numpy

STATS = {"a": Stationarity.STATIONARY_A, "b": Stationarity.STATIONARY_B, "c": Stationarity.STATIONARY_C}


def op_row(op):
    return [op.a_tile.i, op.a_tile.j, op.b_tile.i, op.b_tile.j, op.c_tile.i, op.c_tile.j,
            op.m_bound.lo, op.m_bound.hi, op.k_bound.lo, op.k_bound.hi, op.n_bound.lo, op.n_bound.hi,
            op.a_local.rows.lo, op.a_local.rows.hi, op.a_local.cols.lo, op.a_local.cols.hi,
            op.b_local.rows.lo, op.b_local.rows.hi, op.b_local.cols.lo, op.b_local.cols.hi,
            op.c_local.rows.lo, op.c_local.rows.hi, op.c_local.cols.lo, op.c_local.cols.hi]


def rows_digest(per_rank_rows):
    h = hashlib.sha256()
    for r, rows in enumerate(per_rank_rows):
        for row in rows:
            h.update((f"{r}:" + ",".join(map(str, row)) + "\n").encode())
    return h.hexdigest()[:16]


def mats_for(cfg: dict):
    """Placement-only matrices (no init) for an op-list config."""
    p = cfg["p"]
    fab = Fabric(p)
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    out = {}
    for name, shape, desc, c in (("A", (m, k), cfg["a_part"], cfg["c_a"]),
                                 ("B", (k, n), cfg["b_part"], cfg["c_b"]),
                                 ("C", (m, n), cfg["c_part"], cfg["c_c"])):
        part = resolve_partition(desc, Shape2D(*shape), p // c)
        out[name] = DistributedMatrix(fab, name, Shape2D(*shape), part, c)
    return out


def plan_all(cfg: dict):
    mats = mats_for(cfg)
    stat = STATS[cfg["stat"]]
    return [[op_row(op) for op in opgen.generate(stat, mats["A"], mats["B"], mats["C"], r)]
            for r in range(cfg["p"])]


def divisors(p):
    return [d for d in range(1, p + 1) if p % d == 0]


def sweep_configs():
    """test_acceptance.sweep_configs (tests/test_acceptance.py:40-68) minus the
    execution axis (it does not change op lists)."""
    shapes = [(12, 12, 12), (7, 9, 5), (16, 8, 24)]
    combos = [("row", "col", "2d"), ("misaligned",) * 3, ("2d", "row", "col")]
    which = {"a": "c_a", "b": "c_b", "c": "c_c"}
    for p in (4, 12):
        for m, n, k in shapes:
            for parts in combos:
                for stat in ("a", "b", "c"):
                    reps = []
                    for c in divisors(p):
                        r = {"c_a": 1, "c_b": 1, "c_c": 1}
                        r[which[stat]] = c
                        reps.append(r)
                    reps.append({"c_a": 2, "c_b": 2, "c_c": 2})
                    for r in reps:
                        yield dict(p=p, m=m, n=n, k=k, a_part=parts[0], b_part=parts[1], c_part=parts[2],
                                   stat=stat, **r)


def baseline_configs():
    """BASELINE.json configs resolved for p (SURVEY.md §8(d) 'Scaling')."""
    out = []
    for stat in ("a", "b", "c"):
        out.append(dict(name="cfg1", p=4, m=1024, n=1024, k=1024, a_part="2d", b_part="2d", c_part="2d",
                        c_a=1, c_b=1, c_c=1, stat=stat))
        for p in (1, 2, 4, 8):
            out.append(dict(name="cfg2", p=p, m=65536, n=8192, k=8192, a_part="row", b_part="2d", c_part="row",
                            c_a=1, c_b=p, c_c=1, stat=stat))
            out.append(dict(name="cfg3", p=p, m=8192, n=8192, k=65536, a_part="col", b_part="row", c_part="2d",
                            c_a=1, c_b=1, c_c=p, stat=stat))
            c = min(2, p)
            out.append(dict(name="cfg4", p=p, m=16384, n=16384, k=16384, a_part="2d", b_part="2d", c_part="2d",
                            c_a=c, c_b=c, c_c=c, stat=stat))
            out.append(dict(name="cfg5", p=p, m=16384, n=16384, k=16384, a_part="2d", b_part="col", c_part="row",
                            c_a=1, c_b=1, c_c=1, stat=stat))
    return out


def random_configs(n=100, seed=7):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        p = rng.choice([1, 2, 3, 4, 6, 8, 12])
        m, nn, k = (rng.randint(1, 20) for _ in range(3))
        stat = rng.choice("abc")
        cs = {"c_a": 1, "c_b": 1, "c_c": 1}
        if rng.random() < 0.6:
            cs[rng.choice(list(cs))] = rng.choice(divisors(p))
        parts = []
        for name, (r, c) in (("A", (m, k)), ("B", (k, nn)), ("C", (m, nn))):
            ck = {"A": "c_a", "B": "c_b", "C": "c_c"}[name]
            ranks = p // cs[ck]
            desc = rng.choice(["row", "col", "2d", "misaligned", "custom"])
            if desc == "custom":
                gr = rng.choice([d for d in divisors(ranks)])
                gc = ranks // gr
                desc = f"custom:{rng.randint(1, 9)}:{rng.randint(1, 9)}:{gr}:{gc}"
                if rng.random() < 0.5:
                    desc += ":cyclic"
            parts.append(desc)
        out.append(dict(p=p, m=m, n=nn, k=k, a_part=parts[0], b_part=parts[1], c_part=parts[2], stat=stat, **cs))
    return out


def appendix_c_digest(cfg):
    mats = mats_for(cfg)
    stat = STATS[cfg["stat"]]
    lines = []
    for r in range(cfg["p"]):
        for op in opgen.generate(stat, mats["A"], mats["B"], mats["C"], r):
            lines.append(f"rank {r}: {opgen.format_op(op)}")
    text = "\n".join(lines) + "\n"
    return len(lines), hashlib.sha256(text.encode()).hexdigest()[:16]


def make_oplists():
    sweep = []
    for cfg in sweep_configs():
        rows = plan_all(cfg)
        sweep.append(dict(cfg=cfg, nops=[len(r) for r in rows], digest=rows_digest(rows)))
    baseline = []
    for cfg in baseline_configs():
        rows = plan_all(cfg)
        nops, fmt_digest = appendix_c_digest(cfg)
        baseline.append(dict(cfg=cfg, rows=rows, format_digest=fmt_digest, nops_total=nops))
    rnd = []
    for cfg in random_configs():
        try:
            rows = plan_all(cfg)
        except Exception as e:  # noqa: BLE001 - record the reference's verdict
            rnd.append(dict(cfg=cfg, error=type(e).__name__))
            continue
        rnd.append(dict(cfg=cfg, rows=rows))
    with open(os.path.join(OUT, "oplists.json"), "w") as f:
        json.dump(dict(sweep=sweep, baseline=baseline, random=rnd), f, separators=(",", ":"))
    print(f"oplists: {len(sweep)} sweep, {len(baseline)} baseline, {len(rnd)} random")


# ---------------------------------------------------------------- numeric

NUMERIC_CASES = [
    # (p, m, n, k, a_part, b_part, c_part, c_a, c_b, c_c, stat, real)
    (4, 12, 12, 12, "2d", "2d", "2d", 1, 1, 1, "c", False),
    (4, 7, 9, 5, "row", "col", "2d", 1, 1, 1, "a", False),
    (4, 7, 9, 5, "row", "col", "2d", 1, 1, 1, "b", False),
    (12, 16, 8, 24, "misaligned", "misaligned", "misaligned", 1, 1, 1, "c", False),
    (12, 16, 8, 24, "2d", "row", "col", 2, 2, 2, "b", False),
    (4, 4, 4, 8, "row", "row", "row", 1, 1, 4, "c", False),
    (8, 64, 48, 80, "2d", "col", "row", 1, 1, 1, "c", False),
    (8, 64, 64, 64, "2d", "2d", "2d", 2, 2, 2, "c", False),
    (4, 33, 17, 65, "custom:5:7:2:2:cyclic", "custom:9:4:1:4", "custom:6:6:4:1", 1, 1, 1, "c", False),
    (4, 12, 12, 12, "2d", "2d", "2d", 1, 1, 1, "c", True),
    (8, 64, 48, 80, "2d", "col", "row", 1, 1, 1, "b", True),
    (8, 96, 64, 128, "col", "row", "2d", 1, 1, 8, "c", True),
]


def bf16_round(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def run_numeric(case, seed):
    p, m, n, k, ap, bp, cp, ca, cb, cc, stat, real = case
    rng = np.random.default_rng(seed)
    if real:
        a = bf16_round(rng.uniform(-8.0, 8.0, size=(m, k)))
        b = bf16_round(rng.uniform(-8.0, 8.0, size=(k, n)))
    else:
        a = rng.integers(-8, 9, size=(m, k)).astype(float)
        b = rng.integers(-8, 9, size=(k, n)).astype(float)
    fab = Fabric(p)

    def make(name, dense, shape, desc, c):
        part = resolve_partition(desc, Shape2D(*shape), p // c)
        init = None if dense is None else (lambda r, cc_, d=dense: d[r, cc_])
        return DistributedMatrix(fab, name, Shape2D(*shape), part, c, init)

    A = make("A", a, (m, k), ap, ca)
    B = make("B", b, (k, n), bp, cb)
    C = make("C", None, (m, n), cp, cc)
    cfg = runtime.ExecConfig(stationarity=STATS[stat])
    stats = {r: runtime.run_direct(A, B, C, cfg, r) for r in range(p)}
    partials = np.stack([C.gather(replica=r) for r in range(C.c)])
    if C.c > 1:
        C.reduce_replicas(0)
    final = np.stack([C.gather(replica=r) for r in range(C.c)])
    return a, b, partials, final, fab, stats


def make_numeric():
    arrays = {}
    meta = []
    for i, case in enumerate(NUMERIC_CASES):
        a, b, partials, final, fab, _ = run_numeric(case, seed=100 + i)
        arrays[f"a{i}"] = a
        arrays[f"b{i}"] = b
        arrays[f"partials{i}"] = partials
        arrays[f"final{i}"] = final
        meta.append(dict(case=list(case), comm_bytes=fab.counters.comm_bytes(),
                         flops=fab.counters.flops.tolist()))
    np.savez_compressed(os.path.join(OUT, "numeric.npz"), **arrays)
    return meta


# ---------------------------------------------------------------- runtime / lowering / counters

def make_runtime(numeric_meta):
    out = dict(numeric=numeric_meta)
    # request orders (RunStats.a_requests / b_requests, runtime.py:238-243)
    req = []
    for case in [(9, 12, 12, 12, "2d", "2d", "2d", 1, 1, 1, "c", False),
                 (4, 7, 9, 5, "row", "col", "2d", 1, 1, 1, "a", False),
                 (12, 16, 8, 24, "misaligned", "misaligned", "misaligned", 1, 1, 1, "b", False),
                 (8, 64, 48, 80, "2d", "col", "row", 1, 1, 1, "c", False)]:
        _, _, _, _, fab, stats = run_numeric(case, seed=1)
        req.append(dict(case=list(case),
                        a=[[[t.i, t.j] for t in stats[r].a_requests] for r in range(case[0])],
                        b=[[[t.i, t.j] for t in stats[r].b_requests] for r in range(case[0])],
                        bytes=fab.counters.bytes.tolist(), msgs=fab.counters.msgs.tolist()))
    out["requests"] = req
    # comm bytes of full execute_multiply runs (cli.build_problem conventions)
    vol = []
    for kw in [dict(m=64, n=384, k=96, p=12, stationarity="c", a_part="custom:64:96:1:1", c_a=12,
                    b_part="col", c_part="col"),
               dict(m=64, n=384, k=96, p=12, stationarity="c", a_part="2d", b_part="2d", c_part="2d"),
               dict(m=64, n=96, k=384, p=12, stationarity="b", a_part="col", b_part="row", c_part="2d"),
               dict(m=64, n=96, k=384, p=12, stationarity="c", a_part="row", b_part="row", c_part="row"),
               dict(m=12, n=12, k=12, p=4, stationarity="a", a_part="2d", b_part="2d", c_part="2d"),
               dict(m=12, n=12, k=12, p=4, stationarity="b", a_part="2d", b_part="2d", c_part="2d",
                    accumulate_mode="lockgetput"),
               dict(m=16, n=8, k=24, p=12, stationarity="c", a_part="misaligned", b_part="misaligned",
                    c_part="misaligned", c_c=3)]:
        cfg = RunConfig(**kw)
        fabric, _, A, B, C, a, b = build_problem(cfg)
        mode = AccumulateMode.LOCK_GET_PUT if cfg.accumulate_mode == "lockgetput" else AccumulateMode.PEER_ATOMIC
        runtime.execute_multiply(A, B, C, runtime.ExecConfig(stationarity=STATS[cfg.stationarity],
                                                             accumulate_mode=mode))
        assert np.array_equal(C.gather(0), a @ b)
        vol.append(dict(kw=kw, comm_bytes=fabric.counters.comm_bytes()))
    out["volume"] = vol
    # lowering: greedy IR programs + validation verdicts
    low = []
    for case, limits in [((4, 12, 12, 12, "2d", "2d", "2d", 1, 1, 1, "c"), (4, 4)),
                         ((4, 12, 12, 12, "row", "col", "2d", 1, 1, 1, "b"), (1, 1)),
                         ((12, 16, 8, 24, "misaligned", "misaligned", "misaligned", 1, 1, 1, "a"), (2, 3)),
                         ((4, 8, 8, 8, "2d", "2d", "2d", 1, 1, 1, "b"), (None, None))]:
        p, m, n, k, ap, bp, cp, ca, cb, cc, stat = case
        mats = mats_for(dict(p=p, m=m, n=n, k=k, a_part=ap, b_part=bp, c_part=cp, c_a=ca, c_b=cb, c_c=cc,
                             stat=stat))
        progs = []
        for r in range(p):
            ops = opgen.generate(STATS[stat], mats["A"], mats["B"], mats["C"], r)
            g = lowering.build_graph(ops, mats, r)
            prog = lowering.lower_greedy(g, *limits)
            assert lowering.validate(prog, {r: g}) is None
            progs.append(lowering.format_program(prog, r))
        low.append(dict(case=list(case), limits=list(limits), programs=progs))
    out["lowering"] = low
    with open(os.path.join(OUT, "runtime.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"runtime: {len(req)} request orders, {len(vol)} volumes, {len(low)} lowering cases")


if __name__ == "__main__":
    make_oplists()
    meta = make_numeric()
    make_runtime(meta)
