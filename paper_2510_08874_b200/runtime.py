"""Execution engine: op lists -> one-sided pulls + tcgen05 GEMMs on B200.

Drop-in for unimul.runtime (runtime.py:26-387): same ExecConfig, RunStats,
iteration_offset, local_gemm, run_direct, run_ir and execute_multiply
signatures.  What runs underneath is B200-native, in four modules:

* `schedule`: the caller's op list from the C++ planner, rotated by the
  reference's iteration offset (runtime.py:213-214); remote operand slices
  DEDUPLICATED into fetch-once pulls (the reference re-fetches the whole tile
  for every op: distmatrix.py:158, runtime.py:219-231); `plan_bands` cuts
  ops into sub-ops and pulls into bands so that each (sub-)op waits only for
  the data it reads.
* `engine`: per rank and knob set, an issue plan built once (persistent
  staging pool, prepared K1 launches carrying the in-kernel pulls) and
  replayed by every multiply — normally ONE launch per rank, in which get
  warps pull remote slices while the tensor cores run earlier ops.
* remote C (Stationary A/B): the K1 epilogue accumulates straight into the
  owner's tile (TMA reduce-add on the same GPU, red.global.add over NVLink to
  a peer GPU) — the reference's scratch + accumulate_tile round trip
  (runtime.py:152-166) disappears.
* `replicas`: replicated C is reduced into replica 0 by K4, distributed
  over the replica owners, either after a run-level barrier or — default
  under Stationary C — per row sub-slice as soon as every replica's K1 has
  signalled it.

Everything is stream-ordered: work starts after whatever is pending on the
devices' current streams and the current streams wait for completion on
return, so torch code sees the results without host synchronisation.
"""

from __future__ import annotations

import copy
import ctypes
import dataclasses

import torch

from paper_2510_08874_b200.trace import nvtx
from paper_2510_08874_b200 import _capi, engine, kernels, lowering, opgen
from paper_2510_08874_b200.config import BufferPool, ExecConfig, RunStats
from paper_2510_08874_b200.distmatrix import DistributedMatrix
from paper_2510_08874_b200.engine import TRACE, _current_events, _IssuePlan, _join_current, _RankRun  # noqa: F401
from paper_2510_08874_b200.errors import ContractError
from paper_2510_08874_b200.fabric import ELEM_BYTES, AccumulateMode, pitch_for, um_dtype
from paper_2510_08874_b200.opgen import LocalMatMulOp, Stationarity  # noqa: F401
from paper_2510_08874_b200.replicas import (  # noqa: F401
    _overlap_for, _ReduceOverlap, reduce_replicas, resolve_reduce_mode)
from paper_2510_08874_b200.schedule import (  # noqa: F401
    DirectSchedule, _Fetch, _in_place, _tma_ok, iteration_offset, lower_direct, plan_bands, rotated_ops,
    schedule_cache)
from paper_2510_08874_b200.tiling import TileIdx  # noqa: F401

__all__ = ["ExecConfig", "BufferPool", "RunStats", "iteration_offset", "local_gemm", "run_direct",
           "run_ir", "execute_multiply", "reduce_replicas", "lower_direct", "DirectSchedule", "plan_bands"]


def local_gemm(a, b, c, counters=None, rank: int = 0) -> None:
    """c += a @ b on K1, reporting flops (runtime.py:96-107)."""
    m, k = a.shape
    k2, n = b.shape
    if k != k2 or tuple(c.shape) != (m, n):
        raise ContractError(f"gemm shape mismatch: {tuple(a.shape)} x {tuple(b.shape)} -> {tuple(c.shape)}")
    kernels.gemm_accumulate(a, b, c)
    if counters is not None:
        counters.add_flops(rank, 2 * m * k * n)


def _count_reference_traffic(A, B, C, cfg: ExecConfig, sched: DirectSchedule):
    """FabricCounters exactly as the reference's run_direct would record them.

    Every remote A/B tile is a whole-tile get per op (runtime.py:219-231,
    distmatrix.py:158); every remote C update one accumulate_tile
    (runtime.py:126-135 -> distmatrix.py:170-209: one message if full-width, else one per row;
    2x bytes and messages in LOCK_GET_PUT, fabric.py:225-234).  The per-rank
    totals are computed once per schedule and accumulation mode and added in
    one step per run (the host issue path stays O(1) in the op count).
    """
    ctr = A.fabric.counters
    lgp = cfg.accumulate_mode is AccumulateMode.LOCK_GET_PUT
    memo = sched.__dict__.setdefault("traffic_memo", {})
    delta = memo.get(lgp)
    if delta is None:
        from paper_2510_08874_b200.fabric import FabricCounters

        tmp = FabricCounters(ctr.nprocs)
        _reference_traffic_into(tmp, A, B, C, lgp, sched)
        delta = memo[lgp] = tmp
    ctr.merge(delta)


def _reference_traffic_into(ctr, A, B, C, lgp: bool, sched: DirectSchedule):
    caller = sched.caller
    for i, op in enumerate(sched.ops):
        for M, t in ((A, op.a_tile), (B, op.b_tile)):
            owner = M.owner_rank(t, M.replica_of(caller))
            if owner != caller:
                ctr.add_traffic(caller, owner, ELEM_BYTES * M.tile_bounds(t).area, 1, 0)
        if sched.c_remote[i]:
            owner = C.owner_rank(op.c_tile, C.replica_of(caller))
            n = len(op.m_bound) * len(op.n_bound)
            full = len(op.c_local.cols) == len(C.tile_bounds(op.c_tile).cols)
            msgs = 1 if full else len(op.m_bound)
            ctr.add_traffic(caller, owner, (2 if lgp else 1) * ELEM_BYTES * n, (2 if lgp else 1) * msgs,
                            4 * n)
        ctr.add_flops(caller, op.flops)


def _check_operands(A, B, C):
    if A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise ContractError("A and B must be bfloat16 matrices (tensor-core inputs); "
                            "construct them with dtype=torch.bfloat16")
    if C.dtype != torch.float32:
        raise ContractError("C must be a float32 matrix (fp32 accumulation)")
    A.fabric._require_data()


@nvtx("um:run_direct")
def run_direct(A: DistributedMatrix, B: DistributedMatrix, C: DistributedMatrix, cfg: ExecConfig,
               caller: int) -> RunStats:
    """Direct execution of one rank's rotated op list (runtime.py:193-256).

    Asynchronous and stream-ordered; the driver (execute_multiply) owns the
    run-level barrier and the replica reduction, as in the reference.
    """
    _check_operands(A, B, C)
    fab = A.fabric
    if not fab.is_local(caller):
        raise ContractError(f"rank {caller} is hosted by process {fab.process_of(caller)}")
    fab.heap.exchange()
    sched = lower_direct(A, B, C, cfg, caller)
    _count_reference_traffic(A, B, C, cfg, sched)
    run = _RankRun(A, B, C, cfg, sched, _current_events(fab)).issue()
    _join_current(fab, [run.done])
    run.stats.flops = int(fab.counters.flops[caller])
    return run.stats


# ---------------------------------------------------------------------------
# IR replay (runtime.py:259-336)
# ---------------------------------------------------------------------------

@nvtx("um:run_ir")
def run_ir(prog, graph, A, B, C, cfg: ExecConfig, caller: int) -> RunStats:
    """Replay a validated single-rank IR program on the device.

    A step's computes run first (grouped K1 launch; remote-C ops into scratch),
    then its comm: fetches pull whole tiles into the tile cache on the copy
    stream (satisfying later steps), accumulates push scratch into remote C
    tiles with K3 after their compute (stream order).
    """
    v = lowering.validate(prog, {caller: graph})
    if v is not None:
        raise ContractError(f"refusing to run invalid IR: {v.kind}: {v.message}")
    _check_operands(A, B, C)
    fab = A.fabric
    fab.heap.exchange()
    lib = _capi.load()
    dev = fab.device_of(caller)
    gs, cs = fab.stream(caller, "get"), fab.stream(caller, "compute")
    for ev in _current_events(fab):
        gs.wait_event(ev)
        cs.wait_event(ev)
    mats = {"A": A, "B": B, "C": C}
    stats = RunStats()
    cache: dict[int, tuple] = {}          # data node -> (buffer, event)
    scratch: dict[int, torch.Tensor] = {}
    keep = []
    lgp = cfg.accumulate_mode is AccumulateMode.LOCK_GET_PUT
    ctr = fab.counters
    with torch.cuda.device(dev):
        for step in prog.steps_by_rank[caller]:
            batch = []
            for i in step.compute:
                op = graph.ops[i]
                cn = graph.compute_nodes[i]
                views = []
                for d, t, loc, M in ((cn.a_data, op.a_tile, op.a_local, A), (cn.b_data, op.b_tile, op.b_local, B)):
                    if d in cache:
                        buf, ev = cache[d]
                        cs.wait_event(ev)
                        views.append(_capi.UmView(buf.data_ptr(), loc.rows.lo, loc.rows.hi, loc.cols.lo, loc.cols.hi,
                                                  buf.stride(0), um_dtype(M.dtype), dev))
                    else:
                        seg = M.segment(t, M.replica_of(caller))
                        views.append(seg.um_view(loc.rows.lo, loc.rows.hi, loc.cols.lo, loc.cols.hi))
                if graph.data_nodes[cn.c_data].local:
                    cseg = C.segment(op.c_tile, C.replica_of(caller))
                    gc = cseg.um_view(op.c_local.rows.lo, op.c_local.rows.hi, op.c_local.cols.lo, op.c_local.cols.hi)
                else:
                    m, n = len(op.m_bound), len(op.n_bound)
                    with torch.cuda.stream(cs):
                        sc = torch.zeros((m, pitch_for(n, torch.float32)), dtype=torch.float32, device=f"cuda:{dev}")
                    scratch[i] = sc
                    gc = _capi.UmView(sc.data_ptr(), 0, m, 0, n, sc.stride(0), _capi.UM_F32, dev)
                batch.append(_capi.UmGemmOp(views[0], views[1], gc, 0, 0))
                ctr.add_flops(caller, op.flops)
                stats.executed_ops.append(op)
            if batch:
                arr = (_capi.UmGemmOp * len(batch))(*batch)
                _capi.check(lib.um_gemm_acc_batch(arr, len(batch), dev, ctypes.c_void_p(cs.cuda_stream)),
                            "um_gemm_acc_batch")
                stats.launches += 1
                stats.peak_ops_per_launch = max(stats.peak_ops_per_launch, len(batch))
            for cm in step.comm:
                M = mats[cm.matrix]
                if cm.kind == "fetch":
                    seg = M.segment(cm.tile, M.replica_of(caller))
                    with torch.cuda.stream(gs):
                        buf = torch.empty((seg.rows, seg.pitch), dtype=M.dtype, device=f"cuda:{dev}")
                    buf.record_stream(cs)
                    src = seg.um_view(0, seg.rows, 0, seg.cols)
                    dst = _capi.UmView(buf.data_ptr(), 0, seg.rows, 0, seg.cols, seg.pitch, um_dtype(M.dtype), dev)
                    _capi.check(lib.um_get(ctypes.byref(src), ctypes.byref(dst), ctypes.c_void_p(gs.cuda_stream)),
                                "um_get")
                    ev = torch.cuda.Event()
                    ev.record(gs)
                    cache[cm.data] = (buf, ev)
                    keep.append(buf)
                    ctr.add_traffic(caller, seg.owner, ELEM_BYTES * seg.length, 1, seg.length * buf.element_size())
                    stats.gets += 1
                    (stats.a_requests if cm.matrix == "A" else stats.b_requests).append(cm.tile)
                else:
                    op = graph.ops[cm.op_index]
                    sc = scratch.pop(cm.op_index)
                    keep.append(sc)
                    cseg = C.segment(op.c_tile, C.replica_of(caller))
                    m, n = len(op.m_bound), len(op.n_bound)
                    src = _capi.UmView(sc.data_ptr(), 0, m, 0, n, sc.stride(0), _capi.UM_F32, dev)
                    dst = cseg.um_view(op.c_local.rows.lo, op.c_local.rows.hi, op.c_local.cols.lo, op.c_local.cols.hi)
                    _capi.check(lib.um_accumulate(ctypes.byref(src), ctypes.byref(dst), ctypes.c_void_p(cs.cuda_stream)),
                                "um_accumulate")
                    full = len(op.c_local.cols) == len(C.tile_bounds(op.c_tile).cols)
                    msgs = 1 if full else m
                    ctr.add_traffic(caller, cseg.owner, (2 if lgp else 1) * ELEM_BYTES * m * n,
                                    (2 if lgp else 1) * msgs, 4 * m * n)
                    stats.peak_inflight_accums = max(stats.peak_inflight_accums, 1)
        for buf, ev in cache.values():
            cs.wait_event(ev)
        done = torch.cuda.Event()
        done.record(cs)
    _join_current(fab, [done])
    stats.pool_acquired = stats.pool_released = stats.pool_peak = stats.gets
    stats.peak_inflight_gemms = 1 if stats.executed_ops else 0
    stats.device_order = list(stats.executed_ops)     # IR steps launch in program order
    stats.flops = int(ctr.flops[caller])
    return stats


# ---------------------------------------------------------------------------
# whole-multiply driver (runtime.py:339-387)
# ---------------------------------------------------------------------------

def _cross_process(A, B, C, cfg: ExecConfig) -> bool:
    """Does any rank's schedule touch memory hosted by another process?

    Decided from the plans of ALL ranks (identical on every process), so every
    process takes the same barrier decision.  When nothing crosses a process
    boundary (e.g. cfg2: A/C row blocks, B replicated) the multiply runs with
    no host synchronisation at all.
    """
    fab = A.fabric
    if fab.world.size == 1:
        return False
    key = ("cross", cfg.stationarity, cfg.staging, cfg.same_device_gets)
    cache = schedule_cache(A, B, C)
    if key in cache:
        return cache[key]
    proc = fab.process_of
    cross = False
    for r in range(fab.nprocs):
        sched = lower_direct(A, B, C, cfg, r)
        if any(proc(f.owner) != proc(r) for f in sched.fetches):
            cross = True
        for i, op in enumerate(sched.ops):
            if sched.c_remote[i] and proc(C.owner_rank(op.c_tile, C.replica_of(r))) != proc(r):
                cross = True
    if C.c > 1:
        for t in C.grid.tiles():
            if len({proc(C.owner_rank(t, rep)) for rep in range(C.c)}) > 1:
                cross = True
    cache[key] = cross
    return cross


def _share_sms(fab, ranks) -> dict:
    """Ranks co-resident on one GPU split its SMs: each K1 launch gets an equal
    share of the persistent grid, so their launches (and the pulls inside
    them) overlap instead of queueing behind each other.  Returns the caps set."""
    per_dev: dict = {}
    for r in ranks:
        d = fab.device_of(r)
        per_dev[d] = per_dev.get(d, 0) + 1
    caps = {}
    lib = _capi.load()
    for d, nr in per_dev.items():
        if nr > 1:
            sms = ctypes.c_int32(0)
            _capi.check(lib.um_sm_count(d, ctypes.byref(sms)), "um_sm_count")
            caps[d] = max(1, (sms.value // 2) // nr)
            _capi.check(lib.um_gemm_set_grid_limit(d, caps[d]), "um_gemm_set_grid_limit")
    return caps


GRAPH_MAX_FLOPS = 1 << 36   # graph_replay: multiplies up to ~42 us of tensor-core time
GRAPH_AFTER = 2             # eager multiplies of one (A, B, C, config) before it is captured


def _graph_replay(A, B, C, cfg: ExecConfig) -> dict[int, RunStats] | None:
    """ExecConfig.graph_replay: the third and later calls of a small direct
    multiply on the same (A, B, C, config) run as one CUDA graph replay.

    The host issue of a multiply (per rank: plan lookup, stream fork/join, a
    ctypes call per launch) costs ~50 us, more than the GPU work of a 1024^3
    multiply.  Eligible: one process, every local rank on the current device,
    <= GRAPH_MAX_FLOPS, not inside another capture, launch tracing off.  The
    graph lives in A's schedule cache next to the plans it replays (dropped
    with them).  Returns None when the caller must run the multiply eagerly."""
    fab = A.fabric
    m, k = A.global_shape.rows, A.global_shape.cols
    n = B.global_shape.cols
    if (2 * m * n * k > GRAPH_MAX_FLOPS or fab.world.size != 1 or engine.TRACE_ENABLED
            or torch.cuda.is_current_stream_capturing()):
        return None
    dev = torch.cuda.current_device()
    if any(fab.device_of(r) != dev for r in fab.local_ranks()):
        return None
    cache = schedule_cache(A, B, C)
    key = ("graph", tuple(cfg.__dict__.values()), dev)     # field values: enums, ints, strings
    hit = cache.get(key, 0)
    if hit is None:                                        # capture failed once: eager for good
        return None
    if isinstance(hit, int):
        if hit < GRAPH_AFTER:
            cache[key] = hit + 1
            return None
        from paper_2510_08874_b200.graphs import CapturedMultiply

        # this call's multiply runs eagerly with the graph's config (barrier-form
        # K4), which also builds every plan the capture then records
        gcfg = dataclasses.replace(cfg, graph_replay=False, overlap_reduce=False)
        stats = execute_multiply(A, B, C, gcfg)
        counts = [c.copy() for c in (fab.counters.bytes, fab.counters.msgs, fab.counters.wire_bytes,
                                     fab.counters.flops)]
        try:
            cache[key] = CapturedMultiply(A, B, C, gcfg, warmup=0)
        except Exception:   # noqa: BLE001 -- a path that cannot be captured stays eager
            cache[key] = None
            # a failed capture may have run the host-side counting of a multiply
            for dst, src in zip((fab.counters.bytes, fab.counters.msgs, fab.counters.wire_bytes,
                                 fab.counters.flops), counts):
                dst[...] = src
    else:
        stats = hit.replay()
    out = {}
    for r, st in stats.items():
        out[r] = copy.copy(st)
        out[r].flops = int(fab.counters.flops[r])     # as the eager path reports it
    return out


@nvtx("um:execute_multiply")
def execute_multiply(A: DistributedMatrix, B: DistributedMatrix, C: DistributedMatrix, cfg: ExecConfig,
                     execution: str = "direct", machine=None, max_compute: int | None = None,
                     max_comm: int | None = None, threaded: bool = False) -> dict[int, RunStats]:
    """Run every (local) rank, barrier, then reduce replicated C into replica 0.

    execution: "direct" | "ir:greedy" | "ir:cost" | "ir:exhaustive".
    All ranks are issued asynchronously on their own streams (co-resident
    ranks overlap); `threaded` is accepted for API parity.
    """
    if execution not in ("direct", "ir:greedy", "ir:cost", "ir:exhaustive"):
        raise ValueError(f"unknown execution mode {execution!r}")
    _check_operands(A, B, C)
    if execution == "direct" and cfg.graph_replay:
        replayed = _graph_replay(A, B, C, cfg)
        if replayed is not None:
            return replayed
    fab = A.fabric
    fab.heap.exchange()
    ranks = fab.local_ranks()
    results: dict[int, RunStats] = {}
    cross = _cross_process(A, B, C, cfg) if execution == "direct" else fab.world.size > 1
    ovl = _overlap_for(A, B, C, cfg) if execution == "direct" else None
    if cross:
        fab.synchronize()            # owners' pending writes visible before any remote pull
    start = _current_events(fab)
    done = []
    if execution == "direct":
        runs = []
        caps = _share_sms(fab, ranks) if cfg.share_sms else {}
        try:
            for r in ranks:
                sched = lower_direct(A, B, C, cfg, r)
                _count_reference_traffic(A, B, C, cfg, sched)
                run = _RankRun(A, B, C, cfg, sched, start)
                if ovl is not None:
                    # computed once per schedule (the plan built from it is cached too)
                    memo = sched.__dict__.setdefault("signals_memo", {})
                    if id(ovl) not in memo:
                        memo[id(ovl)] = ovl.signals_for(sched)
                    run.signals, run.signals_key = memo[id(ovl)], ("ovl", id(ovl))
                runs.append(run.issue())
        finally:
            # the grid cap is process-global per device: never leave it set
            for dev in caps:
                _capi.check(_capi.load().um_gemm_set_grid_limit(dev, 0), "um_gemm_set_grid_limit")
        for run in runs:
            run.stats.flops = int(fab.counters.flops[run.caller])
            results[run.caller] = run.stats
            done.append(run.done)
    else:
        mats = {"A": A, "B": B, "C": C}
        for r in ranks:
            ops = opgen.generate(cfg.stationarity, A, B, C, r)
            g = lowering.build_graph(ops, mats, r)
            if execution == "ir:greedy":
                prog = lowering.lower_greedy(g, max_compute, max_comm)
            elif execution == "ir:cost":
                prog = lowering.lower_cost_greedy(g, machine, max_compute, max_comm)
            else:
                prog = lowering.lower_exhaustive(g, machine, max_compute, max_comm)
            results[r] = run_ir(prog, g, A, B, C, cfg, r)
        done = _current_events(fab)
    kmode = resolve_reduce_mode(C, cfg.reduce_mode) if C.c > 1 else "peer"
    if ovl is not None:
        # K4 per sub-slice, each started by its replicas' completion signals
        # (no run-level barrier between the GEMMs and the reduction)
        _join_current(fab, ovl.reduce(start, kmode) + done)
        if fab.world.size > 1:
            fab.synchronize()
    elif cross:
        fab.synchronize()            # run-level barrier across processes
    if C.c > 1 and ovl is None:
        reduce_replicas(C, 0, distributed=cfg.reduce_distributed, start_events=done, mode=kmode)
    if C.c > 1:
        for t in C.grid.tiles():      # reference-model accounting of the pulls
            dst = C.segment(t, 0)
            for r in range(1, C.c):
                src = C.segment(t, r)
                if src.length:
                    fab.counters.add_traffic(dst.owner, src.owner, ELEM_BYTES * src.length, 1, 4 * src.length)
    else:
        _join_current(fab, done)
    return results
