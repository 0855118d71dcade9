"""Multiply straight from host memory, streaming operands in and C out.

`multiply_from_host` is the end-to-end form of `execute_multiply` for data that
starts and ends in (pinned) host memory.  Instead of upload-all / compute /
download-all, the multiply is cut into row panels of C (rows of A): panel
i's A rows go up on an H2D stream while panel i-1 computes and panel i-2's C
rows come back on a D2H stream, so PCIe transfers in both directions and the
tensor cores run concurrently.  Each panel is an ordinary direct execution of
the ops restricted to the panel's rows (same planner, fetch-once gets, K1,
K4), so results are identical to execute_multiply.
"""

from __future__ import annotations

import torch

from paper_2510_08874_b200.trace import nvtx
from paper_2510_08874_b200 import runtime as rt
from paper_2510_08874_b200.errors import ContractError
from paper_2510_08874_b200.opgen import LocalMatMulOp
from paper_2510_08874_b200.tiling import Bounds2D, Range


def _restrict(op: LocalMatMulOp, r0: int, r1: int) -> LocalMatMulOp | None:
    lo, hi = max(op.m_bound.lo, r0), min(op.m_bound.hi, r1)
    if hi <= lo:
        return None
    da, db = lo - op.m_bound.lo, hi - op.m_bound.lo
    return LocalMatMulOp(
        op.a_tile, op.b_tile, op.c_tile, Range(lo, hi), op.k_bound, op.n_bound,
        Bounds2D(Range(op.a_local.rows.lo + da, op.a_local.rows.lo + db), op.a_local.cols),
        op.b_local,
        Bounds2D(Range(op.c_local.rows.lo + da, op.c_local.rows.lo + db), op.c_local.cols))


def _copy_rows(M, host: torch.Tensor, r0: int, r1: int, stream_of, to_device: bool, events: dict):
    """Copy the global rows [r0, r1) of every locally hosted tile of M (all replicas)."""
    fab = M.fabric
    for (rep, t), seg in M._segments.items():
        if seg.storage is None or seg.length == 0:
            continue
        b = M.tile_bounds(t)
        lo, hi = max(r0, b.rows.lo), min(r1, b.rows.hi)
        if hi <= lo:
            continue
        if not to_device and rep != 0:
            continue
        dev = seg.device
        s = stream_of(dev)
        view = seg.view2d()[lo - b.rows.lo:hi - b.rows.lo]
        hslice = host[lo:hi, b.cols.lo:b.cols.hi]
        with torch.cuda.stream(s):
            if to_device:
                view.copy_(hslice, non_blocking=True)
            else:
                hslice.copy_(view, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s)
        events.setdefault(dev, []).append(ev)
    return fab


@nvtx("um:multiply_from_host")
def multiply_from_host(A, B, C, a_host: torch.Tensor, b_host: torch.Tensor, c_out: torch.Tensor,
                       cfg: rt.ExecConfig | None = None, panels: int = 8, copy_streams: int = 1) -> dict:
    """C += A @ B with A, B uploaded from host and replica 0 of C downloaded to c_out.

    a_host: (m, k) host tensor in A's dtype; b_host: (k, n) in B's dtype;
    c_out: (m, n) float32 host tensor.  Pinned memory makes all three copies
    asynchronous.  Returns {rank: RunStats} summed over panels.
    """
    cfg = cfg or rt.ExecConfig()
    rt._check_operands(A, B, C)
    m, k = A.global_shape.rows, A.global_shape.cols
    n = B.global_shape.cols
    if tuple(a_host.shape) != (m, k) or tuple(b_host.shape) != (k, n) or tuple(c_out.shape) != (m, n):
        raise ContractError("host buffers must match the global shapes of A, B and C")
    fab = A.fabric
    fab.heap.exchange()
    devs = sorted({fab.device_of(r) for r in fab.local_ranks()})
    # copy streams per direction (measured on cfg2: 1 stream 202 TFLOP/s e2e,
    # 2 / 3 / 4 streams 172 / 164 / 161 — concurrent copies contend on PCIe)
    nst = max(1, copy_streams)
    h2d_s = {d: [_side_stream(fab, d, f"h2d{i}") for i in range(nst)] for d in devs}
    d2h_s = {d: [_side_stream(fab, d, f"d2h{i}") for i in range(nst)] for d in devs}
    start = rt._current_events(fab)
    for d in devs:
        for ev in start:
            for st_ in h2d_s[d] + d2h_s[d]:
                st_.wait_event(ev)
    # B is needed by every panel: upload it whole first
    up: dict = {}
    _copy_rows(B, b_host, 0, k, lambda d: h2d_s[d][0], True, up)
    b_events = [e for evs in up.values() for e in evs]
    full_ops = {r: rt.rotated_ops(A, B, C, cfg, r) for r in fab.local_ranks()}
    cross = rt._cross_process(A, B, C, cfg)
    results = {r: rt.RunStats() for r in fab.local_ranks()}
    bounds = [m * i // panels for i in range(panels + 1)]
    done_all = []
    for i in range(panels):
        r0, r1 = bounds[i], bounds[i + 1]
        if r1 <= r0:
            continue
        up = {}
        _copy_rows(A, a_host, r0, r1, lambda d: h2d_s[d][i % nst], True, up)
        ready = b_events + [e for evs in up.values() for e in evs]
        if cross:
            fab.synchronize()            # remote ranks may pull these rows
        runs = []
        for r in fab.local_ranks():
            ops = [o for o in (_restrict(op, r0, r1) for op in full_ops[r]) if o is not None]
            if not ops:
                continue
            # panel schedules (and their issue plans) are cached like full ones
            pkey = ("panel", cfg.stationarity, cfg.staging, cfg.same_device_gets, r, r0, r1)
            cache = rt.schedule_cache(A, B, C)
            sched = cache.get(pkey)
            if sched is None:
                sched = cache[pkey] = rt.lower_direct(A, B, C, cfg, r, ops=ops)
            rt._count_reference_traffic(A, B, C, cfg, sched)
            runs.append(rt._RankRun(A, B, C, cfg, sched, ready).issue())
        done = [run.done for run in runs]
        for run in runs:
            st = results[run.caller]
            st.executed_ops += run.stats.executed_ops
            st.device_order += run.stats.device_order
            st.a_requests += run.stats.a_requests
            st.b_requests += run.stats.b_requests
            st.launches += run.stats.launches
            st.gets += run.stats.gets
            st.staged_bytes += run.stats.staged_bytes
        if cross:
            fab.synchronize()
        if C.c > 1:
            done = rt.reduce_replicas(C, 0, distributed=cfg.reduce_distributed, start_events=done, rows=(r0, r1),
                                      mode=cfg.reduce_mode)
        for d in devs:
            for ev in done:
                d2h_s[d][i % nst].wait_event(ev)
        down: dict = {}
        _copy_rows(C, c_out, r0, r1, lambda d: d2h_s[d][i % nst], False, down)
        done_all += [e for evs in down.values() for e in evs] + done
    rt._join_current(fab, done_all)
    for r, st in results.items():
        st.flops = int(fab.counters.flops[r])
    return results


def _side_stream(fab, dev: int, kind: str) -> torch.cuda.Stream:
    key = (("dev", dev), kind)
    s = fab._streams.get(key)
    if s is None:
        s = torch.cuda.Stream(device=dev)
        fab._streams[key] = s
    return s
