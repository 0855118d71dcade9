"""Host-side IR lowering (paper_2510_08874_b200.lowering) on a placement-only
fabric: the properties the reference's lowering suite pins
(/root/reference/pkg/tests/test_lowering.py), restated against this package.

Covered: data-node deduplication and pre-satisfied local edges
(lowering.py:108-132), every lowerer's output passing validate() under
compute/comm limits (:145-348), the exhaustive search being minimum-cost and
bounded (:269-348), each invariant validate() checks (:351-420), and the text
form (:423-429).  No GPU: the CLI's placement-only fabric plans and lowers
without device memory."""

import dataclasses

import pytest

from paper_2510_08874_b200 import Stationarity, costmodel, lowering, opgen
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.errors import ConfigError

# (m, n, k, p, A, B, C partitions, c_A, c_B, c_C)
CASES = [
    (64, 48, 80, 4, "2d", "2d", "2d", 1, 1, 1),
    (96, 64, 128, 4, "2d", "col", "row", 1, 1, 1),
    (72, 40, 56, 6, "row", "col", "2d", 1, 1, 1),
    (64, 64, 96, 4, "2d", "2d", "2d", 1, 1, 2),
    (50, 30, 70, 3, "misaligned", "row", "col", 1, 1, 1),
]
STATS = [Stationarity.STATIONARY_A, Stationarity.STATIONARY_B, Stationarity.STATIONARY_C]
LIMITS = [(None, None), (1, 1), (2, 1), (1, 2), (3, 3)]


def graphs_for(case, st):
    m, n, k, p, ap, bp, cp, ca, cb, cc = case
    fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=3)
    assert fab.placement_only
    mats = {"A": A, "B": B, "C": C}
    out = {}
    for r in range(p):
        ops = opgen.generate(st, A, B, C, r)
        out[r] = lowering.build_graph(ops, mats, r)
    return fab, out


def machine(p):
    return costmodel.MachineModel.b200(p)


def cost(prog, g, mach):
    return sum(costmodel.step_cost(s, g.caller, g.ops, mach) for s in prog.steps_by_rank[g.caller])


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("st", STATS)
def test_every_lowerer_is_valid_under_limits(case, st):
    _, graphs = graphs_for(case, st)
    mach = machine(case[3])
    for g in graphs.values():
        progs = [lowering.lower_naive(g)]
        for mc, mm in LIMITS:
            progs.append(lowering.lower_greedy(g, mc, mm))
            progs.append(lowering.lower_cost_greedy(g, mach, mc, mm))
        for prog in progs:
            assert lowering.validate(prog, {g.caller: g}) is None
            for step in prog.steps_by_rank[g.caller]:
                assert step.compute or step.comm


@pytest.mark.parametrize("case", CASES)
def test_data_nodes_deduplicated_and_local_edges_satisfied(case):
    _, graphs = graphs_for(case, Stationarity.STATIONARY_C)
    for g in graphs.values():
        keys = [(d.matrix, d.tile) for d in g.data_nodes]
        assert len(keys) == len(set(keys))
        for d in g.data_nodes:
            assert d.local == (d.owner == g.caller)
        # every remote input is fetched exactly once, in first-reference order
        order = g.fetch_order
        assert len(order) == len(set(order))
        assert all(not g.data_nodes[d].local for d in order)
        first = []
        for cn in g.compute_nodes:
            for d in (cn.a_data, cn.b_data):
                if not g.data_nodes[d].local and d not in first:
                    first.append(d)
        assert order == first


def test_single_rank_is_one_compute_step():
    _, graphs = graphs_for((64, 48, 80, 1, "2d", "2d", "2d", 1, 1, 1), Stationarity.STATIONARY_C)
    g = graphs[0]
    prog = lowering.lower_greedy(g)
    steps = prog.steps_by_rank[0]
    assert len(steps) == 1 and steps[0].compute == list(range(len(g.ops))) and not steps[0].comm


def test_empty_op_list():
    _, graphs = graphs_for(CASES[0], Stationarity.STATIONARY_C)
    g = dataclasses.replace(graphs[0], ops=[], compute_nodes=[],
                            data_nodes=[d for d in graphs[0].data_nodes if d.local])
    for prog in (lowering.lower_greedy(g), lowering.lower_naive(g)):
        assert prog.steps_by_rank[g.caller] == []
        assert lowering.validate(prog, {g.caller: g}) is None


@pytest.mark.parametrize("case", CASES[:3])
@pytest.mark.parametrize("st", STATS)
def test_exhaustive_is_minimum_cost(case, st):
    _, graphs = graphs_for(case, st)
    mach = machine(case[3])
    for g in graphs.values():
        if len(g.ops) > 4:
            continue
        for mc, mm in [(None, None), (1, 1), (2, 1)]:
            best = lowering.lower_exhaustive(g, mach, mc, mm)
            assert lowering.validate(best, {g.caller: g}) is None
            c_best = cost(best, g, mach)
            for other in (lowering.lower_greedy(g, mc, mm), lowering.lower_cost_greedy(g, mach, mc, mm)):
                assert c_best <= cost(other, g, mach) * (1 + 1e-12)
            assert c_best <= cost(lowering.lower_naive(g), g, mach) * (1 + 1e-12)


def test_exhaustive_refuses_large_instances():
    _, graphs = graphs_for((96, 64, 128, 4, "2d", "col", "row", 1, 1, 1), Stationarity.STATIONARY_C)
    g = max(graphs.values(), key=lambda g: len(g.ops))
    assert len(g.ops) > 2
    with pytest.raises(ConfigError):
        lowering.lower_exhaustive(g, machine(4), exhaustive_bound=2)


def _remote_c_graph():
    """A rank under Stationary A whose ops accumulate into a remote C tile."""
    for case in CASES:
        _, graphs = graphs_for(case, Stationarity.STATIONARY_A)
        for g in graphs.values():
            if any(g.accum_comm(i) is not None for i in range(len(g.ops))) and g.fetch_order:
                return g
    raise AssertionError("no rank with remote accumulates and fetches")


def test_validate_reports_each_violation():
    g = _remote_c_graph()
    G = {g.caller: g}
    prog = lowering.lower_naive(g)
    steps = prog.steps_by_rank[g.caller]
    assert lowering.validate(prog, G) is None

    def with_steps(new, mc=lowering.UNBOUNDED, mm=lowering.UNBOUNDED):
        return lowering.IrProgram({g.caller: new}, mc, mm)

    # dependency: a compute whose remote input has not been fetched yet
    first_fetch = next(s for s, st in enumerate(steps) if st.comm and st.comm[0].kind == "fetch")
    dep = [lowering.IrStep(list(st.compute), list(st.comm)) for st in steps]
    fetched = dep[first_fetch].comm[0].data
    user = next(cn.index for cn in g.compute_nodes if fetched in (cn.a_data, cn.b_data))
    for st in dep:
        if user in st.compute:
            st.compute.remove(user)
    dep.insert(0, lowering.IrStep([user], []))
    assert lowering.validate(with_steps(dep), G).kind == "dependency"
    # completeness: an op never scheduled
    last_compute = max(s for s, st in enumerate(steps) if st.compute)
    inc = [lowering.IrStep(list(st.compute), list(st.comm)) for st in steps]
    inc[last_compute].compute.pop()
    inc = [st for st in inc if st.compute or st.comm]
    v = lowering.validate(with_steps(inc), G)
    assert v is not None and v.kind in ("completeness", "accum")
    # duplicate fetch
    dup = [lowering.IrStep(list(st.compute), list(st.comm)) for st in steps]
    dup.append(lowering.IrStep([], [g.fetch_comm(fetched)]))
    assert lowering.validate(with_steps(dup), G).kind == "fetch"
    # limits: a step with more comm ops than the program allows
    packed = lowering.lower_greedy(g)
    wide = max(packed.steps_by_rank[g.caller], key=lambda st: len(st.comm) + len(st.compute))
    n = max(len(wide.comm), len(wide.compute))
    if n > 1:
        assert lowering.validate(with_steps(packed.steps_by_rank[g.caller], n - 1, n - 1), G).kind == "limits"
    # accumulate before its compute
    acc_op = next(i for i in range(len(g.ops)) if g.accum_comm(i) is not None)
    early = [lowering.IrStep(list(st.compute), [c for c in st.comm if not (c.kind == "accum"
                                                                            and c.op_index == acc_op)])
             for st in steps]
    early.insert(0, lowering.IrStep([], [g.accum_comm(acc_op)]))
    early = [st for st in early if st.compute or st.comm]
    assert lowering.validate(with_steps(early), G).kind == "accum"


def test_format_and_merge():
    _, graphs = graphs_for(CASES[1], Stationarity.STATIONARY_C)
    progs = [lowering.lower_greedy(g, 1, 1) for g in graphs.values()]
    merged = lowering.merge_programs(progs)
    assert sorted(merged.steps_by_rank) == sorted(graphs)
    assert lowering.validate(merged, graphs) is None
    for r, g in graphs.items():
        text = lowering.format_program(merged, r).splitlines()
        assert len(text) == len(merged.steps_by_rank[r])
        for s, line in enumerate(text):
            assert line.startswith(f"step {s}: compute=[") and "] comm=[" in line
        for st, line in zip(merged.steps_by_rank[r], text):
            for c in st.comm:
                assert str(c) in line
                assert str(c).startswith("fetch " if c.kind == "fetch" else "acc ")


def test_greedy_fills_compute_before_comm_each_step():
    """Greedy: every op whose inputs are satisfied at a step's start runs in that
    step (up to max_compute) -- lowering.py:145-177."""
    _, graphs = graphs_for(CASES[1], Stationarity.STATIONARY_C)
    for g in graphs.values():
        for mc in (None, 1, 2):
            prog = lowering.lower_greedy(g, mc, 1)
            satisfied = {i for i, d in enumerate(g.data_nodes) if d.local}
            done = set()
            cap = mc or lowering.UNBOUNDED
            for st in prog.steps_by_rank[g.caller]:
                ready = [cn.index for cn in g.compute_nodes if cn.index not in done
                         and cn.a_data in satisfied and cn.b_data in satisfied]
                assert st.compute == ready[:cap]
                done.update(st.compute)
                satisfied.update(c.data for c in st.comm if c.kind == "fetch")
            assert done == set(range(len(g.ops)))
