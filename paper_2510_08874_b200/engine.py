"""Device issue of one rank's direct schedule: issue plans and their replay.

A plan (built once per schedule and knob set) holds the persistent staging
pool, the copy-engine pulls, and one prepared K1 launch per group
(um_gemm_prepare) carrying the in-kernel pulls; every multiply replays it.
"""

from __future__ import annotations

import ctypes
import os

import torch

from paper_2510_08874_b200.trace import nvtx
from paper_2510_08874_b200 import _capi
from paper_2510_08874_b200 import schedule as _sch
from paper_2510_08874_b200.config import ExecConfig, RunStats
from paper_2510_08874_b200.fabric import pitch_for, um_dtype
from paper_2510_08874_b200.schedule import DirectSchedule, _tma_ok, plan_bands

# Launch tracing for the benchmark's roofline: (start, end, algorithmic flops)
# CUDA events recorded on the compute stream around every grouped K1 launch.
TRACE: list = []
TRACE_ENABLED = False


def _current_events(fabric) -> list:
    evs = []
    for d in sorted({fabric.device_of(r) for r in fabric.local_ranks()}):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(d))
        evs.append(ev)
    return evs


def _join_current(fabric, events):
    for d in sorted({fabric.device_of(r) for r in fabric.local_ranks()}):
        cur = torch.cuda.current_stream(d)
        for ev in events:
            cur.wait_event(ev)


# profiling knob (UM_DEBUG_NO_PULLS=1): launches drop their in-kernel pulls and
# waits, so a rank's op list runs as if every operand were already staged --
# the compute-only bound of the same launch (results are wrong)
_NO_PULLS = os.environ.get("UM_DEBUG_NO_PULLS") == "1"


class _IssuePlan:
    """One rank's issue plan: persistent staging buffers, copy-engine pulls,
    and an action list of prepared K1 launches / stream waits / unfused
    scratch updates, replayed by every multiply with the same schedule."""

    def __init__(self, nprocs: int):
        from paper_2510_08874_b200.fabric import FabricCounters

        self.staged: list = []
        self.host_fetches: list = []      # (fetch index, src view, dst view)
        self.actions: list = []           # ("launch", handle, flops) | ("wait", j) | ("scratch", op, ga, gb)
        self.final_waits: list = []
        self.handles: list = []
        self.traffic = FabricCounters(nprocs)   # wire bytes of the pulls, added per run
        self.stats = RunStats()
        self.flag = None                  # arrival flag of the flagged copy-engine pulls (device int32)
        self.flagged: set = set()         # fetches whose arrival K1 observes through `flag`

    def __del__(self):
        try:
            lib = _capi.load()
            for h in self.handles:
                lib.um_gemm_destroy(ctypes.c_void_p(h))
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class _RankRun:
    """Device work of one rank's direct schedule (issued asynchronously)."""

    def __init__(self, A, B, C, cfg: ExecConfig, sched: DirectSchedule, start_events):
        self.A, self.B, self.C, self.cfg, self.sched = A, B, C, cfg, sched
        fab = A.fabric
        self.fab = fab
        self.caller = sched.caller
        self.dev = fab.device_of(self.caller)
        self.gs = fab.stream(self.caller, "get")
        self.cs = fab.stream(self.caller, "compute")
        self.stats = RunStats()
        self.buffers = []
        self.done = None
        self.signals = None        # op -> (row cuts, (m0, m1) -> done_flag): overlapped replica reduction
        self.signals_key = None
        self.start_events = list(start_events)
        for ev in self.start_events:   # the get stream waits only if the plan uses it (_replay)
            self.cs.wait_event(ev)

    def _mat(self, name):
        return self.A if name == "A" else self.B

    def issue(self):
        """Replay this rank's issue plan (built once per schedule and knob set)."""
        self._replay(self.plan())
        return self

    def plan(self) -> "_IssuePlan":
        """This rank's issue plan, built once per schedule and knob set (cached on the schedule)."""
        key = (self.cfg.get_engine, self.cfg.gemm_batch, self.cfg.max_inflight_accums, self.cfg.fused_accumulate,
               self.cfg.fine_waits,
               self.cfg.k_split, self.cfg.mn_split, self.cfg.chain_order, _sch._SPLIT_BYTES, _sch._SPLIT_MIN, _sch._RASTER_N, self.signals_key,
               self.cfg.pool_capacity, self.cfg.prefetch_depth if self.cfg.pool_capacity else 0,
               self.cfg.max_inflight_gemms if self.cfg.pool_capacity else 0)
        plans = self.sched.__dict__.setdefault("plans", {})
        plan = plans.get(key)
        if plan is None:
            plan = plans[key] = (self._build_bounded_plan() if self.cfg.pool_capacity is not None
                                 else self._build_plan())
        return plan

    @nvtx("um:plan")
    def _build_plan(self) -> "_IssuePlan":
        """Resolve everything host-side once: persistent staging buffers (the
        paper's pre-allocated pool), which pulls run inside
        the GEMM launch and which on the copy engines, the launch split, and one
        prepared K1 launch (um_gemm_prepare) per group."""
        lib = _capi.load()
        s, fab = self.sched, self.fab
        nf = len(s.fetches)
        plan = _IssuePlan(fab.counters.nprocs)
        st = plan.stats
        with torch.cuda.device(self.dev):
            for f in s.fetches:
                M = self._mat(f.mat)
                with torch.cuda.stream(self.cs):
                    buf = torch.empty((f.r1 - f.r0, pitch_for(f.c1 - f.c0, M.dtype)), dtype=M.dtype,
                                      device=f"cuda:{self.dev}")
                buf.record_stream(self.gs)
                plan.staged.append(buf)
        staged = plan.staged
        views = [(self._operand_view("A", op.a_tile, op.a_local, s.a_src[i], staged),
                  self._operand_view("B", op.b_tile, op.b_local, s.b_src[i], staged)) for i, op in enumerate(s.ops)]
        # which pulls run inside the K1 launch (get warps) and which on the copy
        # engines.  get_engine "kernel": all in-kernel; "copy": all copy engine,
        # the host splitting launches at each pull; "auto": pulls from the
        # caller's own GPU in-kernel, pulls across GPUs (NVLink) on the copy
        # engines, each followed by an arrival flag the K1 producer waits on
        # (one launch, no SM spent on the transfer); "ce": every pull on the
        # copy engines with flags.  Every op reading an in-kernel or flagged
        # slice must see a TMA-readable view of it (16-byte column start);
        # the rest fall back to copy engine + host-side ordering.
        eng = self.cfg.get_engine
        shared = fab.world.size > 1 and fab.devices_shared_across_processes()

        def owner_gpu(j):
            """The owner's device index as seen here (-1: unknown, another process's GPU)."""
            d = fab.device_of(s.fetches[j].owner)
            return self.dev if (d < 0 and shared) else d

        def ce_ok(j):
            # a flagged copy-engine pull is only safe where the driver runs it
            # without SMs while K1 holds them all (um_ce_probe, measured once per
            # device pair); another process's GPU is probed through any peer
            src = owner_gpu(j)
            if src < 0:
                n = ctypes.c_int32(0)
                _capi.check(lib.um_device_count(ctypes.byref(n)), "um_device_count")
                src = (self.dev + 1) % max(1, n.value)
            ok = ctypes.c_int32(0)
            _capi.check(lib.um_ce_probe(self.dev, src, ctypes.byref(ok)), "um_ce_probe")
            return bool(ok.value)

        in_kernel = [eng == "kernel" or (eng == "auto" and (owner_gpu(j) == self.dev or not ce_ok(j)))
                     for j in range(nf)]
        flagged = [eng in ("auto", "ce") and not in_kernel[j] and ce_ok(j) for j in range(nf)]
        for i in range(len(s.ops)):
            for src, v in ((s.a_src[i], views[i][0]), (s.b_src[i], views[i][1])):
                if src >= 0 and not _tma_ok(v):
                    in_kernel[src] = False
                    flagged[src] = False

        def fetch_views(j, band=None):
            f = s.fetches[j]
            br0, br1, bc0, bc1 = band if band is not None else (0, f.r1 - f.r0, 0, f.c1 - f.c0)
            src = self._mat(f.mat).segment(f.tile, f.replica).um_view(f.r0 + br0, f.r0 + br1, f.c0 + bc0, f.c0 + bc1)
            dst = _capi.UmView(staged[j].data_ptr(), br0, br1, bc0, bc1, staged[j].stride(0),
                               um_dtype(staged[j].dtype), self.dev)
            return src, dst

        items, bands, need = plan_bands(s, in_kernel, self.cfg,
                                        None if self.signals is None else {i: cuts for i, (cuts, _) in
                                                                           self.signals.items()})

        flag_value = {}                  # flagged fetch -> arrival-flag value once it has landed
        if any(flagged):
            with torch.cuda.device(self.dev):
                plan.flag = torch.zeros(4, dtype=torch.int32, device=f"cuda:{self.dev}")
        for j, f in enumerate(s.fetches):
            if not in_kernel[j]:
                plan.host_fetches.append((j, *fetch_views(j)))
                if flagged[j]:
                    flag_value[j] = len(flag_value) + 1
                    plan.flagged.add(j)
                nbytes = (f.r1 - f.r0) * (f.c1 - f.c0) * staged[j].element_size()
            else:
                nbytes = sum((r1 - r0) * (c1 - c0) for r0, r1, c0, c1 in bands[j]) * staged[j].element_size()
            plan.traffic.add_traffic(self.caller, f.owner, 0, 0, nbytes)
            st.gets += 1
            st.staged_bytes += nbytes
        st.pool_acquired = st.pool_released = st.pool_peak = nf

        # ---- K1 launch groups.  In-kernel pulls (bands) travel with the first
        # launch that needs them; a copy-engine pull not yet waited on splits
        # the group (the compute stream waits for its event).
        batch: list = []
        batch_gets: list = []            # (fetch, band) units of this launch, in first-use order
        gets_slot: dict = {}             # unit -> 0-based slot in batch_gets
        launched: set = set()
        batch_remote = 0
        waited = [False] * nf
        cap = self.cfg.gemm_batch or _capi.GEMM_MAX_INLINE_OPS

        def flush():
            nonlocal batch, batch_remote, batch_gets, gets_slot
            if not batch and not batch_gets:
                return
            arr = (_capi.UmGemmOp * max(1, len(batch)))(*batch)
            garr = (_capi.UmGetDesc * max(1, len(batch_gets)))()
            for gi, (j, k) in enumerate(batch_gets):
                garr[gi].src, garr[gi].dst = fetch_views(j, bands[j][k])
                launched.add((j, k))
            h = ctypes.c_void_p()
            ng = len(batch_gets)
            if _NO_PULLS:                # profiling only: operands treated as resident (stale staging, wrong C)
                for g in arr:
                    g.a_get = g.b_get = 0
                    g.get_mask = 0
                ng = 0
            _capi.check(lib.um_gemm_prepare(arr, len(batch), garr, ng, self.dev, ctypes.byref(h)),
                        "um_gemm_prepare")
            plan.handles.append(h.value)
            flops = float(sum(2 * (g.a.row_hi - g.a.row_lo) * (g.a.col_hi - g.a.col_lo) * (g.b.col_hi - g.b.col_lo)
                              for g in batch))
            plan.actions.append(("launch", h.value, flops))
            st.launches += 1
            st.peak_ops_per_launch = max(st.peak_ops_per_launch, len(batch))
            st.peak_inflight_accums = max(st.peak_inflight_accums, batch_remote)
            batch, batch_remote, batch_gets, gets_slot = [], 0, [], {}

        def host_wait(j):
            if not waited[j]:
                flush()
                plan.actions.append(("wait", j))
                waited[j] = True

        last_piece = {(i, m0, m1): it for it, (i, _, m0, m1, *_) in enumerate(items)}
        for it, (i, t, m0, m1, n0, n1, k0, k1) in enumerate(items):
            op = s.ops[i]
            srcs = [j for j in (s.a_src[i], s.b_src[i]) if j >= 0]
            unfused = s.c_remote[i] and not self.cfg.fused_accumulate
            for j in srcs:
                if not in_kernel[j] and (not flagged[j] or unfused):
                    host_wait(j)
            remote = s.c_remote[i] and self.fab.device_of(
                self.C.owner_rank(op.c_tile, self.C.replica_of(self.caller))) != self.dev
            units = [(j, k) for j in dict.fromkeys(srcs) if in_kernel[j] for k in need[(it, j)]]
            new_units = [u for u in units if u not in launched and u not in gets_slot]
            if (len(batch) >= cap or (remote and batch_remote >= self.cfg.max_inflight_accums)
                    or len(batch_gets) + len(new_units) > _capi.GEMM_MAX_GETS):
                flush()
                new_units = [u for u in units if u not in launched]
            ga, gb = views[i]
            sub = (m0, m1, n0, n1, k0, k1) != (0, len(op.m_bound), 0, len(op.n_bound), 0, len(op.k_bound))
            if sub:
                ga = _capi.UmView(ga.base, ga.row_lo + m0, ga.row_lo + m1, ga.col_lo + k0, ga.col_lo + k1, ga.pitch,
                                  ga.dtype, ga.device)
                gb = _capi.UmView(gb.base, gb.row_lo + k0, gb.row_lo + k1, gb.col_lo + n0, gb.col_lo + n1, gb.pitch,
                                  gb.dtype, gb.device)
            if remote and not self.cfg.fused_accumulate:
                # unfused remote update (scratch GEMM + K3): its pulls must have landed
                flush()
                batch_gets.extend(new_units)
                flush()
                plan.actions.append(("scratch", op, ga, gb))
                st.launches += 2
                st.peak_ops_per_launch = max(st.peak_ops_per_launch, 1)
                st.peak_inflight_accums = max(st.peak_inflight_accums, 1)
                continue
            for u in new_units:
                gets_slot[u] = len(batch_gets)
                batch_gets.append(u)
            cseg = self.C.segment(op.c_tile, self.C.replica_of(self.caller))
            cl = op.c_local
            gc = cseg.um_view(cl.rows.lo + m0, cl.rows.lo + m1, cl.cols.lo + n0, cl.cols.lo + n1)
            g = _capi.UmGemmOp(ga, gb, gc, 1 if remote else 0)
            fv = [flag_value[j] for j in srcs if j in flag_value and not waited[j]]
            if fv:                       # copy-engine pulls: wait on the arrival flag in the kernel
                g.wait_flag = plan.flag.data_ptr()
                g.wait_value = max(fv)
            # an operand read from ONE band of this launch (inside its columns)
            # waits chunk by chunk: A for its tile rows, B for each k-block's rows
            fine = {}
            for name, j, v in (("a", s.a_src[i], ga), ("b", s.b_src[i], gb)):
                if self.cfg.fine_waits and j >= 0 and in_kernel[j] and len(need[(it, j)]) == 1:
                    u = (j, need[(it, j)][0])
                    br0, br1, bc0, bc1 = bands[j][u[1]]
                    if (u in gets_slot and bc0 <= v.col_lo and v.col_hi <= bc1 and br0 <= v.row_lo
                            and v.row_hi <= br1):
                        fine[name] = u
            g.a_get = gets_slot[fine["a"]] + 1 if "a" in fine else 0
            g.b_get = gets_slot[fine["b"]] + 1 if "b" in fine else 0
            g.get_mask = sum(1 << gets_slot[u] for u in units if u in gets_slot and u not in fine.values())
            if self.signals is not None and i in self.signals:
                g.done_flag = self.signals[i][1](m0, m1)
                # pieces of one (op, sub-slice) along n: the last one issued counts
                g.done_piece = 1 if it != last_piece[(i, m0, m1)] else 0
            batch.append(g)
            batch_remote += int(remote)
        flush()
        # RunStats report the reference's execution order (runtime.py:213-236),
        # whatever order the device runs the (sub-)ops in
        st.executed_ops = list(s.ops)
        st.a_requests = [op.a_tile for op in s.ops]
        st.b_requests = [op.b_tile for op in s.ops]
        st.device_order = [s.ops[i] for i in dict.fromkeys(it[0] for it in items)]
        plan.final_waits = [j for j in range(nf) if not in_kernel[j] and not waited[j]]
        st.peak_inflight_gemms = 1 if s.ops else 0
        return plan

    @nvtx("um:plan_bounded")
    def _build_bounded_plan(self) -> "_IssuePlan":
        """Bounded staging (ExecConfig.pool_capacity set): the reference's
        bounded-asynchrony discipline (runtime.py:43-73,186-231) on the device.

        * a pool of `pool_capacity` staging slots, each as large as the largest
          remote operand slice one (sub-)op reads, allocated once (the
          reference's BufferPool of tile-sized buffers);
        * the (sub-)ops run in device order in launch groups of at most
          min(max_inflight_gemms, prefetch_depth + 1) ops — the GEMMs in
          flight together, whose pulls are issued at most prefetch_depth ops
          ahead of the oldest — whose remote slices fit the free slots; the
          group's pulls run inside its K1 launch (get warps) and each op waits
          only for its own slices (fine waits);
        * a slot is refilled only by a later launch: stream order is the
          back-pressure (every reader of the old contents has finished), and a
          slice evicted before its next use is pulled again, as the reference
          re-fetches per op (runtime.py:219-231);
        * an op that needs more slots than the pool holds raises the
          reference's RuntimeError (runtime.py:62-67)."""
        lib = _capi.load()
        s, fab, cfg = self.sched, self.fab, self.cfg
        plan = _IssuePlan(fab.counters.nprocs)
        st = plan.stats
        cap = cfg.pool_capacity
        items, _, _ = plan_bands(s, [False] * len(s.fetches), cfg,
                                 None if self.signals is None else {i: cuts for i, (cuts, _) in self.signals.items()})
        last_piece = {(i, m0, m1): it for it, (i, _, m0, m1, *_) in enumerate(items)}

        def units_of(item):
            """(key, src view, rows, cols, mat) of each remote operand slice the item reads."""
            i, t, m0, m1, n0, n1, k0, k1 = item
            op = s.ops[i]
            out = {}
            for name, j, loc, (dr0, dr1, dc0, dc1) in (
                    ("a", s.a_src[i], op.a_local, (m0, m1, k0, k1)), ("b", s.b_src[i], op.b_local, (k0, k1, n0, n1))):
                if j < 0:
                    continue
                f = s.fetches[j]
                r0, r1 = loc.rows.lo + dr0, loc.rows.lo + dr1
                c0, c1 = loc.cols.lo + dc0, loc.cols.lo + dc1
                M = self._mat(f.mat)
                key = (f.mat, f.tile, f.replica, r0, r1, c0, c1)
                out[name] = (key, M.segment(f.tile, f.replica).um_view(r0, r1, c0, c1), r1 - r0, c1 - c0, M)
            return out

        per_item = [units_of(it) for it in items]
        # a slot holds any one slice (its own 16-byte pitch, rows packed)
        slot_elems = max([u[2] * pitch_for(u[3], u[4].dtype) for us in per_item for u in us.values()], default=0)
        for us in per_item:
            if len({u[0] for u in us.values()}) > cap:
                raise RuntimeError("buffer pool exhausted with nothing left to drain; increase pool_capacity")
        slots = []
        if slot_elems:
            with torch.cuda.device(self.dev), torch.cuda.stream(self.cs):
                slots = [torch.empty(slot_elems, dtype=torch.bfloat16, device=f"cuda:{self.dev}")
                         for _ in range(cap)]
        plan.staged = slots
        st.staged_bytes = sum(t.numel() * t.element_size() for t in slots)

        resident: dict = {}              # slice key -> slot (contents valid after the launch that pulled it)
        holder = [None] * cap            # slot -> slice key
        group_max = max(1, min(cfg.max_inflight_gemms, cfg.prefetch_depth + 1))
        batch, gets, in_group = [], [], set()
        in_use = 0

        def flush():
            nonlocal batch, gets, in_group
            if not batch:
                return
            arr = (_capi.UmGemmOp * len(batch))(*batch)
            garr = (_capi.UmGetDesc * max(1, len(gets)))(*gets)
            h = ctypes.c_void_p()
            _capi.check(lib.um_gemm_prepare(arr, len(batch), garr, len(gets), self.dev, ctypes.byref(h)),
                        "um_gemm_prepare")
            plan.handles.append(h.value)
            flops = float(sum(2 * (g.a.row_hi - g.a.row_lo) * (g.a.col_hi - g.a.col_lo) * (g.b.col_hi - g.b.col_lo)
                              for g in batch))
            plan.actions.append(("launch", h.value, flops))
            st.launches += 1
            st.peak_ops_per_launch = max(st.peak_ops_per_launch, len(batch))
            batch, gets, in_group = [], [], set()

        for it, (item, us) in enumerate(zip(items, per_item)):
            keys = {u[0] for u in us.values()}
            new = [k for k in keys if k not in resident]
            slot_of = {k: resident[k] for k in keys if k in resident}

            def free_slots():
                # slots not read by the current launch group nor holding this op's own slices;
                # empty ones first
                fs = [x for x in range(cap) if (holder[x] is None or holder[x] not in in_group)
                      and x not in slot_of.values()]
                return sorted(fs, key=lambda x: holder[x] is not None)

            free = free_slots()
            if (len(batch) >= group_max or len(new) > len(free) or len(gets) + len(new) > _capi.GEMM_MAX_GETS):
                flush()
                free = free_slots()
            get_slot = {}
            for k in new:
                x = free.pop(0)
                if holder[x] is not None:
                    resident.pop(holder[x], None)
                holder[x] = k
                resident[k] = x
                slot_of[k] = x
                u = next(v for v in us.values() if v[0] == k)
                dst = _capi.UmView(slots[x].data_ptr(), 0, u[2], 0, u[3], pitch_for(u[3], u[4].dtype), _capi.UM_BF16,
                                   self.dev)
                get_slot[k] = len(gets)
                gets.append(_capi.UmGetDesc(u[1], dst))
                plan.traffic.add_traffic(self.caller, u[4].owner_rank(k[1], k[2]), 0, 0, u[2] * u[3] * 2)
                st.gets += 1
                st.pool_acquired += 1
                st.pool_released += 1
            in_group |= keys
            in_use = len({holder[x] for x in range(cap) if holder[x] in in_group})
            st.pool_peak = max(st.pool_peak, in_use)
            i, t, m0, m1, n0, n1, k0, k1 = item
            op = s.ops[i]
            views = {}
            for name, j, loc, (dr0, dr1, dc0, dc1), M in (
                    ("a", s.a_src[i], op.a_local, (m0, m1, k0, k1), self.A),
                    ("b", s.b_src[i], op.b_local, (k0, k1, n0, n1), self.B)):
                if name in us:
                    key, _, rows, cols, Mu = us[name]
                    x = slot_of[key]
                    views[name] = _capi.UmView(slots[x].data_ptr(), 0, rows, 0, cols, pitch_for(cols, Mu.dtype),
                                               _capi.UM_BF16, self.dev)
                else:
                    seg = M.segment(op.a_tile if name == "a" else op.b_tile, M.replica_of(self.caller))
                    views[name] = seg.um_view(loc.rows.lo + dr0, loc.rows.lo + dr1, loc.cols.lo + dc0,
                                              loc.cols.lo + dc1)
            remote = s.c_remote[i] and self.fab.device_of(
                self.C.owner_rank(op.c_tile, self.C.replica_of(self.caller))) != self.dev
            cseg = self.C.segment(op.c_tile, self.C.replica_of(self.caller))
            cl = op.c_local
            gc = cseg.um_view(cl.rows.lo + m0, cl.rows.lo + m1, cl.cols.lo + n0, cl.cols.lo + n1)
            g = _capi.UmGemmOp(views["a"], views["b"], gc, 1 if remote else 0)
            ga_new = "a" in us and us["a"][0] in get_slot
            gb_new = "b" in us and us["b"][0] in get_slot
            if ga_new:
                g.a_get = get_slot[us["a"][0]] + 1
            if gb_new:
                g.b_get = get_slot[us["b"][0]] + 1
            # a slice pulled earlier in this launch (not by this op's own get) must have landed
            mask = 0
            for name in ("a", "b"):
                if name in us:
                    k = us[name][0]
                    if k not in get_slot:
                        pos = next((q for q, gd in enumerate(gets) if gd.dst.base == slots[slot_of[k]].data_ptr()),
                                   None)
                        if pos is not None:
                            mask |= 1 << pos
            g.get_mask = mask
            if self.signals is not None and i in self.signals:
                g.done_flag = self.signals[i][1](m0, m1)
                g.done_piece = 1 if it != last_piece[(i, m0, m1)] else 0
            batch.append(g)
        flush()
        st.executed_ops = list(s.ops)
        st.a_requests = [op.a_tile for op in s.ops]
        st.b_requests = [op.b_tile for op in s.ops]
        st.device_order = [s.ops[i] for i in dict.fromkeys(it[0] for it in items)]
        st.peak_inflight_gemms = min(group_max, len(s.ops)) if s.ops else 0
        return plan

    @nvtx("um:issue_rank")
    def _replay(self, plan: "_IssuePlan"):
        lib = _capi.load()
        fab = self.fab
        with torch.cuda.device(self.dev):
            events = {}
            gsp = ctypes.c_void_p(self.gs.cuda_stream)
            # the get stream carries copy-engine pulls only; a plan without
            # them (every pull in-kernel, or none) neither forks nor joins it
            uses_gs = bool(plan.host_fetches) or bool(plan.flagged)
            if uses_gs:
                for ev in self.start_events:
                    self.gs.wait_event(ev)
            if plan.flagged:
                # reset the arrival flag before this run's K1 can read it
                fptr = ctypes.c_void_p(plan.flag.data_ptr())
                _capi.check(lib.um_signal(fptr, 0, gsp), "um_signal")
                ev = torch.cuda.Event()
                ev.record(self.gs)
                self.cs.wait_event(ev)
            landed = 0
            for j, src, dst in plan.host_fetches:        # K2 on the copy engines, first-use order
                if j in plan.flagged:
                    _capi.check(lib.um_get_ce(ctypes.byref(src), ctypes.byref(dst), gsp), "um_get_ce")
                    landed += 1
                    _capi.check(lib.um_signal(fptr, landed, gsp), "um_signal")
                else:
                    _capi.check(lib.um_get(ctypes.byref(src), ctypes.byref(dst), gsp), "um_get")
                ev = torch.cuda.Event()
                ev.record(self.gs)
                events[j] = ev
            csp = ctypes.c_void_p(self.cs.cuda_stream)
            for act in plan.actions:
                if act[0] == "launch":
                    if TRACE_ENABLED:
                        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        t0.record(self.cs)
                    _capi.check(lib.um_gemm_launch(ctypes.c_void_p(act[1]), csp), "um_gemm_launch")
                    if TRACE_ENABLED:
                        t1.record(self.cs)
                        TRACE.append((t0, t1, act[2]))
                elif act[0] == "wait":
                    self.cs.wait_event(events[act[1]])
                else:
                    self._scratch_gemm(*act[1:])
            for j in plan.final_waits:
                self.cs.wait_event(events[j])
            if uses_gs:
                # join the get stream back (a multiply stays capturable into a
                # CUDA graph: no unjoined forked stream)
                ev = torch.cuda.Event()
                ev.record(self.gs)
                self.cs.wait_event(ev)
            self.done = torch.cuda.Event()
            self.done.record(self.cs)
        fab.counters.merge(plan.traffic)
        t = plan.stats
        self.stats = RunStats(list(t.executed_ops), list(t.a_requests), list(t.b_requests), t.peak_inflight_gemms,
                              t.peak_inflight_accums, t.pool_acquired, t.pool_released, t.pool_peak, 0, t.gets,
                              t.staged_bytes, t.launches, t.peak_ops_per_launch, list(t.device_order))

    def _operand_view(self, name, t, loc, src_idx, staged):
        M = self._mat(name)
        if src_idx < 0:
            seg = M.segment(t, M.replica_of(self.caller))
            return seg.um_view(loc.rows.lo, loc.rows.hi, loc.cols.lo, loc.cols.hi)
        f = self.sched.fetches[src_idx]
        buf = staged[src_idx]
        return _capi.UmView(buf.data_ptr(), loc.rows.lo - f.r0, loc.rows.hi - f.r0, loc.cols.lo - f.c0,
                            loc.cols.hi - f.c0, buf.stride(0), um_dtype(M.dtype), self.dev)

    def _scratch_gemm(self, op, ga, gb):
        """Unfused remote update: GEMM into zeroed scratch, then K3 accumulate."""
        lib = _capi.load()
        m, n = len(op.m_bound), len(op.n_bound)
        pitch = pitch_for(n, torch.float32)
        with torch.cuda.stream(self.cs):
            scratch = torch.zeros((m, pitch), dtype=torch.float32, device=f"cuda:{self.dev}")
        self.buffers.append(scratch)
        gs = _capi.UmView(scratch.data_ptr(), 0, m, 0, n, pitch, _capi.UM_F32, self.dev)
        _capi.check(lib.um_gemm_acc(ctypes.byref(ga), ctypes.byref(gb), ctypes.byref(gs),
                                    ctypes.c_void_p(self.cs.cuda_stream)), "um_gemm_acc")
        cseg = self.C.segment(op.c_tile, self.C.replica_of(self.caller))
        dst = cseg.um_view(op.c_local.rows.lo, op.c_local.rows.hi, op.c_local.cols.lo, op.c_local.cols.hi)
        with torch.cuda.device(self.dev), torch.cuda.stream(self.cs):
            _capi.check(lib.um_accumulate(ctypes.byref(gs), ctypes.byref(dst), ctypes.c_void_p(self.cs.cuda_stream)),
                        "um_accumulate")
