"""Pin the CPU oracle to the REAL reference's outputs (tests/golden/, made by
tests/golden/make_golden.py importing /root/reference).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import um_oracle as O


def mats(cfg):
    p = cfg["p"]
    out = {}
    for name, (r, c), desc, rep in (("A", (cfg["m"], cfg["k"]), cfg["a_part"], cfg["c_a"]),
                                    ("B", (cfg["k"], cfg["n"]), cfg["b_part"], cfg["c_b"]),
                                    ("C", (cfg["m"], cfg["n"]), cfg["c_part"], cfg["c_c"])):
        out[name] = O.Mat(name, r, c, O.resolve_partition(desc, r, c, p // rep), rep, p)
    return out


def rows_digest(per_rank):
    h = hashlib.sha256()
    for r, rows in enumerate(per_rank):
        for row in rows:
            h.update((f"{r}:" + ",".join(map(str, row)) + "\n").encode())
    return h.hexdigest()[:16]


def oracle_rows(cfg):
    M = mats(cfg)
    return [[list(op.row()) for op in O.generate(cfg["stat"], M["A"], M["B"], M["C"], r)] for r in range(cfg["p"])]


def test_sweep_op_lists_match_reference(oplists):
    for entry in oplists["sweep"]:
        rows = oracle_rows(entry["cfg"])
        assert [len(r) for r in rows] == entry["nops"], entry["cfg"]
        assert rows_digest(rows) == entry["digest"], entry["cfg"]


def test_baseline_op_lists_match_reference(oplists):
    for entry in oplists["baseline"]:
        cfg = entry["cfg"]
        assert oracle_rows(cfg) == entry["rows"], cfg
        M = mats(cfg)
        lines = [f"rank {r}: {O.format_op(op)}" for r in range(cfg["p"])
                 for op in O.generate(cfg["stat"], M["A"], M["B"], M["C"], r)]
        text = "\n".join(lines) + "\n"
        assert hashlib.sha256(text.encode()).hexdigest()[:16] == entry["format_digest"]


def test_baseline_digests_match_survey_appendix_c(oplists):
    # SURVEY.md Appendix C, Stationary C column, p=8
    want = {"cfg2": "3ee56c26affcba7b", "cfg3": "09b0edae1846ec8a", "cfg4": "0b32a5d41b93b504",
            "cfg5": "1fe2df38daa49249"}
    got = {e["cfg"]["name"]: e["format_digest"] for e in oplists["baseline"]
           if e["cfg"]["p"] == 8 and e["cfg"]["stat"] == "c"}
    assert got == want
    cfg1 = [e for e in oplists["baseline"] if e["cfg"]["name"] == "cfg1" and e["cfg"]["stat"] == "c"][0]
    assert cfg1["format_digest"] == "e364e11d02f1d363"


def test_random_op_lists_match_reference(oplists):
    for entry in oplists["random"]:
        if "error" in entry:
            with pytest.raises(Exception):
                oracle_rows(entry["cfg"])
            continue
        assert oracle_rows(entry["cfg"]) == entry["rows"], entry["cfg"]


def _numeric_case(runtime_golden, i):
    return runtime_golden["numeric"][i]["case"]


def test_numeric_results_match_reference(runtime_golden, numeric_golden):
    for i, meta in enumerate(runtime_golden["numeric"]):
        p, m, n, k, ap, bp, cp, ca, cb, cc, stat, real = meta["case"]
        cfg = dict(p=p, m=m, n=n, k=k, a_part=ap, b_part=bp, c_part=cp, c_a=ca, c_b=cb, c_c=cc)
        M = mats(cfg)
        a, b = numeric_golden[f"a{i}"], numeric_golden[f"b{i}"]
        partial = O.execute(stat, M["A"], M["B"], M["C"], a, b, reduce=False)
        final = O.execute(stat, M["A"], M["B"], M["C"], a, b, reduce=True)
        ref_partial, ref_final = numeric_golden[f"partials{i}"], numeric_golden[f"final{i}"]
        if real:
            np.testing.assert_allclose(np.stack(partial), ref_partial, rtol=0, atol=1e-9)
            np.testing.assert_allclose(np.stack(final), ref_final, rtol=0, atol=1e-9)
        else:
            assert np.array_equal(np.stack(partial), ref_partial), meta["case"]
            assert np.array_equal(np.stack(final), ref_final), meta["case"]
        assert np.array_equal(final[0], np.asarray(ref_final[0]))  or real


def test_request_orders_match_reference(runtime_golden):
    for entry in runtime_golden["requests"]:
        p, m, n, k, ap, bp, cp, ca, cb, cc, stat, _ = entry["case"]
        M = mats(dict(p=p, m=m, n=n, k=k, a_part=ap, b_part=bp, c_part=cp, c_a=ca, c_b=cb, c_c=cc))
        for r in range(p):
            a_req, b_req = O.request_order(stat, M["A"], M["B"], M["C"], r)
            assert [list(t) for t in a_req] == entry["a"][r]
            assert [list(t) for t in b_req] == entry["b"][r]


def test_reference_model_bytes_match_reference(runtime_golden):
    for entry in runtime_golden["volume"]:
        kw = dict(entry["kw"])
        lgp = kw.pop("accumulate_mode", "peer") == "lockgetput"
        cfg = dict(p=kw["p"], m=kw["m"], n=kw["n"], k=kw["k"], a_part=kw["a_part"], b_part=kw["b_part"],
                   c_part=kw["c_part"], c_a=kw.get("c_a", 1), c_b=kw.get("c_b", 1), c_c=kw.get("c_c", 1))
        M = mats(cfg)
        assert O.reference_model_bytes(kw["stationarity"], M["A"], M["B"], M["C"], lgp) == entry["comm_bytes"], kw


def test_greedy_programs_match_reference(runtime_golden):
    for entry in runtime_golden["lowering"]:
        p, m, n, k, ap, bp, cp, ca, cb, cc, stat = entry["case"]
        M = mats(dict(p=p, m=m, n=n, k=k, a_part=ap, b_part=bp, c_part=cp, c_a=ca, c_b=cb, c_c=cc))
        for r in range(p):
            ops = O.generate(stat, M["A"], M["B"], M["C"], r)
            g = O.build_graph(ops, M, r)
            steps = O.lower_greedy(g, *entry["limits"])
            assert O.format_program(g, steps) == entry["programs"][r]


def test_fill_values_are_the_documented_sets():
    ints = O.fill_values(3, 0, 64, 0, 64, "int")
    assert set(np.unique(ints)).issubset(set(range(-8, 9))) and len(np.unique(ints)) == 17
    reals = O.fill_values(3, 0, 64, 0, 64, "real")
    assert reals.min() >= -1.0 and reals.max() < 1.0
    # global coordinates: a sub-block equals the same window of a bigger fill
    big = O.fill_values(9, 0, 40, 0, 40, "real")
    assert np.array_equal(big[7:19, 11:30], O.fill_values(9, 7, 19, 11, 30, "real"))


def test_round_bf16():
    x = np.array([1.0, 1.00390625, 1.0078125, -3.14159, 65504.0, 1e-20], dtype=np.float32)
    r = O.round_bf16(x)
    import torch

    assert np.array_equal(r, torch.tensor(x).to(torch.bfloat16).float().numpy())


def test_reference_compiled_kernel_agrees(runtime_golden, numeric_golden):
    """oracle/_ref (the reference's own _gemmcore, built from /root/reference) gives
    the same results as the numpy port on the golden integer cases."""
    try:
        O.gemm_kernel("reference")
    except ImportError:
        pytest.skip("oracle/_ref not built")
    for i, meta in enumerate(runtime_golden["numeric"][:6]):
        p, m, n, k, ap, bp, cp, ca, cb, cc, stat, real = meta["case"]
        M = mats(dict(p=p, m=m, n=n, k=k, a_part=ap, b_part=bp, c_part=cp, c_a=ca, c_b=cb, c_c=cc))
        a, b = numeric_golden[f"a{i}"], numeric_golden[f"b{i}"]
        got = O.execute(stat, M["A"], M["B"], M["C"], a, b, kernel="reference")
        assert np.array_equal(np.stack(got), numeric_golden[f"final{i}"])
