"""Execution engine: op lists -> one-sided gets + tcgen05 GEMMs on B200.

Drop-in for unimul.runtime (runtime.py:26-387): same ExecConfig, RunStats,
iteration_offset, local_gemm, run_direct, run_ir and execute_multiply
signatures.  What runs underneath is B200-native:

* schedule lowering (direct execution, runtime.py:193-256): the caller's op
  list comes from the C++ planner, rotated by the reference's iteration
  offset (runtime.py:213-214).  Remote operand slices are then DEDUPLICATED:
  every remote (matrix, tile) is pulled once, as the bounding box of the
  slices this rank's ops need (the reference re-fetches the whole tile for
  every op: distmatrix.py:158, runtime.py:219-231).  Pulls are issued in
  first-use order on a per-rank copy stream (K2, copy engines), each
  followed by an event.
* GEMM issue: ops are grouped into persistent grouped launches (K1); a group
  is flushed whenever the next op needs a pull that has not been waited on,
  so pulls overlap the GEMMs of earlier ops.
* remote C (Stationary A/B): the K1 epilogue accumulates straight into the
  owner's tile (TMA reduce-add on the same GPU, red.global.add over NVLink to
  a peer GPU) — the reference's scratch + accumulate_tile round trip
  (runtime.py:362-373) disappears.
* replicated C: after a run-level barrier, K4 reduces the replicas into
  replica 0, distributed over the replica owners' GPUs.

Everything is stream-ordered: work starts after whatever is pending on the
devices' current streams and the current streams wait for completion on
return, so torch code sees the results without host synchronisation.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

from paper_2510_08874_b200 import _capi, kernels, lowering, opgen
from paper_2510_08874_b200.distmatrix import DistributedMatrix
from paper_2510_08874_b200.errors import ContractError
from paper_2510_08874_b200.fabric import ELEM_BYTES, AccumulateMode, pitch_for, um_dtype
from paper_2510_08874_b200.opgen import LocalMatMulOp, Stationarity
from paper_2510_08874_b200.tiling import TileIdx

# Launch tracing for the benchmark's roofline: (start, end, algorithmic flops)
# CUDA events recorded on the compute stream around every grouped K1 launch.
TRACE: list = []
TRACE_ENABLED = False

__all__ = ["ExecConfig", "BufferPool", "RunStats", "iteration_offset", "local_gemm", "run_direct",
           "run_ir", "execute_multiply", "reduce_replicas", "lower_direct", "DirectSchedule"]


@dataclass
class ExecConfig:
    """Reference knobs (runtime.py:26-40) plus B200 knobs.

    B200 knobs:
      staging            "slice": pull the bounding box of the slices a rank
                         needs from each remote tile, once; "tile": pull whole
                         remote tiles once.
      same_device_gets   "copy": ranks co-resident on one GPU still pull
                         (one-sided semantics, exercises K2); "direct": read
                         the owner's tile in place.
      gemm_batch         max ops per grouped K1 launch (0 = unlimited).
      fused_accumulate   remote C updates from the K1 epilogue (K3 fused);
                         False = scratch GEMM + um_accumulate.
      reduce_distributed K4 over all replica owners (True) or pull-to-origin.
      mn_split           max sub-ops along m (pulled A dominates) or n (pulled
                         B dominates) for an op whose first use pulls >= 64
                         MiB: each sub-op starts when its band has landed.
      k_split            > 1: split such ops along k instead (one A and one B
                         slab per sub-op, one extra C read-modify-write each).
      overlap_reduce     replicated C under Stationary C: each C tile is cut
                         into c * reduce_panels row sub-slices; the K1
                         epilogue signals every finished sub-slice to its
                         reducer (done_flag), whose K4 starts on a stream wait
                         (um_wait_geq) while the GEMMs go on — no run-level
                         barrier between the GEMMs and the reduction.
      reduce_panels      sub-slices per replica and tile (>= 1).
      chain_order        issue ops that write the same C region back to back
                         (K1 accumulates such a k-chain in TMEM and reduces
                         into C once per tile).
      get_engine         "kernel": remote slices are pulled by get warps INSIDE
                         the K1 launch (um_gemm_acc_fused) and each op starts
                         when its pulls have landed — one launch per rank (up
                         to UM_GEMM_MAX_INLINE_OPS ops / UM_GEMM_MAX_GETS pulls)
                         with the gets overlapping the GEMMs of earlier ops;
                         "copy": copy-engine pulls on a get stream, the host
                         splits K1 launches at every pull not yet waited on.
    """

    stationarity: Stationarity = Stationarity.STATIONARY_C
    prefetch_depth: int = 2
    max_inflight_gemms: int = 4
    max_inflight_accums: int = 4
    accumulate_mode: AccumulateMode = AccumulateMode.PEER_ATOMIC
    pool_capacity: int | None = None
    staging: str = "slice"
    same_device_gets: str = "copy"
    gemm_batch: int = 0
    fused_accumulate: bool = True
    reduce_distributed: bool = True
    get_engine: str = "kernel"
    mn_split: int = 4
    overlap_reduce: bool = True
    chain_order: bool = True
    reduce_panels: int = 2
    k_split: int = 0

    def __post_init__(self):
        if self.prefetch_depth < 1 or self.max_inflight_gemms < 1 or self.max_inflight_accums < 1:
            raise ValueError("ExecConfig counts must be >= 1")
        if self.pool_capacity is not None and self.pool_capacity < 3:
            raise ValueError("pool_capacity must cover at least one op (3 buffers)")
        if self.staging not in ("slice", "tile"):
            raise ValueError(f"unknown staging mode {self.staging!r}")
        if self.same_device_gets not in ("copy", "direct"):
            raise ValueError(f"unknown same_device_gets {self.same_device_gets!r}")
        if self.get_engine not in ("kernel", "copy"):
            raise ValueError(f"unknown get_engine {self.get_engine!r}")
        if self.k_split < 0 or self.mn_split < 0:
            raise ValueError("k_split / mn_split must be >= 0")
        if self.reduce_panels < 1:
            raise ValueError("reduce_panels must be >= 1")
        if self.gemm_batch < 0:
            raise ValueError("gemm_batch must be >= 0")


class BufferPool:
    """Fixed set of staging slots; no allocation after construction (runtime.py:43-73).

    Kept for API parity (IR replay uses it for scratch accounting).  With
    `buffer_elems` > 0 and a device, the slots are device buffers.
    """

    def __init__(self, capacity: int, buffer_elems: int, device=None, dtype=torch.float32):
        self._arena = torch.zeros((capacity, max(1, buffer_elems)), dtype=dtype,
                                  device=device if device is not None else "cpu")
        self._free = list(range(capacity))
        self.capacity = capacity
        self.acquired = 0
        self.released = 0
        self.peak_in_use = 0

    @property
    def free_count(self) -> int:
        return len(self._free)

    def acquire(self, drain=None):
        while not self._free:
            if drain is None or not drain():
                raise RuntimeError("buffer pool exhausted with nothing left to drain; increase pool_capacity")
        slot = self._free.pop()
        self.acquired += 1
        self.peak_in_use = max(self.peak_in_use, self.capacity - len(self._free))
        return slot, self._arena[slot]

    def release(self, slot: int):
        self._free.append(slot)
        self.released += 1


@dataclass
class RunStats:
    """Per-rank record (runtime.py:76-86) plus what the B200 engine did."""

    executed_ops: list[LocalMatMulOp] = field(default_factory=list)
    a_requests: list[TileIdx] = field(default_factory=list)
    b_requests: list[TileIdx] = field(default_factory=list)
    peak_inflight_gemms: int = 0
    peak_inflight_accums: int = 0
    pool_acquired: int = 0
    pool_released: int = 0
    pool_peak: int = 0
    flops: int = 0
    gets: int = 0
    staged_bytes: int = 0
    launches: int = 0
    peak_ops_per_launch: int = 0


def iteration_offset(stationary_tile: TileIdx, nops: int) -> int:
    """(i + j) mod nops of the first op's stationary tile (runtime.py:89-93)."""
    out = ctypes.c_int64(0)
    _capi.check(_capi.load().um_iteration_offset(stationary_tile.i, stationary_tile.j, nops, ctypes.byref(out)),
                "iteration_offset")
    return int(out.value)


def local_gemm(a, b, c, counters=None, rank: int = 0) -> None:
    """c += a @ b on K1, reporting flops (runtime.py:96-107)."""
    m, k = a.shape
    k2, n = b.shape
    if k != k2 or tuple(c.shape) != (m, n):
        raise ContractError(f"gemm shape mismatch: {tuple(a.shape)} x {tuple(b.shape)} -> {tuple(c.shape)}")
    kernels.gemm_accumulate(a, b, c)
    if counters is not None:
        counters.add_flops(rank, 2 * m * k * n)


# ---------------------------------------------------------------------------
# schedule lowering for direct execution
# ---------------------------------------------------------------------------

@dataclass
class _Fetch:
    mat: str                 # "A" | "B"
    tile: TileIdx
    replica: int
    owner: int
    r0: int                  # tile-local bounding box of the needed slices
    r1: int
    c0: int
    c1: int
    first_use: int


@dataclass
class DirectSchedule:
    """Lowered direct-execution schedule of one rank."""

    caller: int
    ops: list                        # rotated op list
    fetches: list                    # _Fetch in first-use order
    a_src: list                      # per op: fetch index or -1 (read in place)
    b_src: list
    c_remote: list                   # per op: True if the C tile belongs to another rank


def _in_place(fabric, owner: int, caller: int, cfg: ExecConfig) -> bool:
    if owner == caller:
        return True
    if cfg.same_device_gets == "direct" and fabric.world.size == 1 and not fabric.placement_only:
        return fabric.device_of(owner) == fabric.device_of(caller)
    return False


def rotated_ops(A, B, C, cfg: ExecConfig, caller: int) -> list:
    """The caller's op list in execution order (runtime.py:207,213-214)."""
    ops = opgen.generate(cfg.stationarity, A, B, C, caller)
    if ops:
        s = iteration_offset(ops[0].stationary_tile(cfg.stationarity), len(ops))
        ops = ops[s:] + ops[:s]
    return ops


def lower_direct(A, B, C, cfg: ExecConfig, caller: int, ops: list | None = None) -> DirectSchedule:
    """Rotated op list + fetch-once staging plan (host-side, no device work).

    `ops` overrides the planner's list (e.g. ops restricted to a row panel).
    Schedules of the planner's own list are cached per (matrices, knobs, rank):
    placement is immutable, so repeated multiplies skip the host work."""
    if ops is None:
        key = (id(B), id(C), cfg.stationarity, cfg.staging, cfg.same_device_gets, caller)
        cache = A.__dict__.setdefault("_sched_cache", {})
        hit = cache.get(key)
        if hit is not None and hit[0] is B and hit[1] is C:
            return hit[2]
        sched = lower_direct(A, B, C, cfg, caller, rotated_ops(A, B, C, cfg, caller))
        cache[key] = (B, C, sched)
        return sched
    fabric = A.fabric
    fetches: list[_Fetch] = []
    index: dict = {}
    a_src, b_src, c_remote = [], [], []
    for i, op in enumerate(ops):
        for name, M, t, loc, srcs in (("A", A, op.a_tile, op.a_local, a_src), ("B", B, op.b_tile, op.b_local, b_src)):
            rep = M.replica_of(caller)
            owner = M.owner_rank(t, rep)
            if _in_place(fabric, owner, caller, cfg):
                srcs.append(-1)
                continue
            key = (name, t)
            j = index.get(key)
            if cfg.staging == "tile":
                b = M.tile_bounds(t)
                r0, r1, c0, c1 = 0, len(b.rows), 0, len(b.cols)
            else:
                r0, r1, c0, c1 = loc.rows.lo, loc.rows.hi, loc.cols.lo, loc.cols.hi
            if j is None:
                index[key] = len(fetches)
                srcs.append(len(fetches))
                fetches.append(_Fetch(name, t, rep, owner, r0, r1, c0, c1, i))
            else:
                f = fetches[j]
                f.r0, f.r1, f.c0, f.c1 = min(f.r0, r0), max(f.r1, r1), min(f.c0, c0), max(f.c1, c1)
                srcs.append(j)
        c_owner = C.owner_rank(op.c_tile, C.replica_of(caller))
        c_remote.append(c_owner != caller)
    return DirectSchedule(caller, ops, fetches, a_src, b_src, c_remote)


def _count_reference_traffic(A, B, C, cfg: ExecConfig, sched: DirectSchedule):
    """FabricCounters exactly as the reference's run_direct would record them.

    Every remote A/B tile is a whole-tile get per op (runtime.py:427-438,
    distmatrix.py:158); every remote C update one accumulate_tile
    (runtime.py:338-341: one message if full-width, else one per row;
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


def _check_operands(A, B, C):
    if A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise ContractError("A and B must be bfloat16 matrices (tensor-core inputs); "
                            "construct them with dtype=torch.bfloat16")
    if C.dtype != torch.float32:
        raise ContractError("C must be a float32 matrix (fp32 accumulation)")
    A.fabric._require_data()


_SPLIT_BYTES = 64 << 20       # an op whose first use pulls at least this much runs as sub-ops
_SPLIT_MIN = 2048             # minimum extent of a sub-op along the split dimension


def _tma_ok(v) -> bool:
    """K1 reads a view in place iff its column start, pitch and base are 16-byte aligned."""
    es = 2 if v.dtype == _capi.UM_BF16 else 4
    return (v.col_lo * es) % 16 == 0 and (v.pitch * es) % 16 == 0 and (v.base or 0) % 16 == 0


def plan_bands(s: DirectSchedule, in_kernel: list, cfg: ExecConfig, row_cuts: dict | None = None):
    """Host-only planning of a rank's in-kernel pulls (no device work).

    Returns (items, bands, need):
      items  (op, sub, m0, m1, n0, n1, k0, k1): the ops in execution order, an
             op that must first pull >= _SPLIT_BYTES split into sub-ops
             (offsets relative to the op's m / n / k ranges);
      bands  per fetch: (r0, r1, c0, c1) rectangles of the staged slice, cut
             along the dimension in which the (sub-)ops' slices differ, bands
             no op reads dropped (None for copy-engine fetches);
      need   (item, fetch) -> indices of the bands the item reads.
    row_cuts   op -> cut positions along its m range (relative): the op is split
             exactly there and nowhere else (overlapped replica reduction:
             every item then lies in one reduction sub-slice of its C tile).
    """
    nf = len(s.fetches)
    # Sub-ops: an op that must first pull a large amount (cfg4: whole 8192^2
    # A and B tiles) runs as sub-ops that each wait only for their part of
    # the pull.  Default split: along m when the pulled A dominates, along n
    # when B does (rows / columns of C: no extra C traffic, the tensor cores
    # start once B / A and the first A / B band have landed).  k_split > 1
    # instead cuts k into slabs (every sub-op waits for one A and one B
    # slab, at the price of one more fp32 C read-modify-write per slab).
    first_user: dict = {}
    for i in range(len(s.ops)):
        for j in (s.a_src[i], s.b_src[i]):
            if j >= 0:
                first_user.setdefault(j, i)

    def pulled(i, j):
        if j < 0 or not in_kernel[j] or first_user[j] != i:
            return 0
        f = s.fetches[j]
        return (f.r1 - f.r0) * (f.c1 - f.c0) * 2

    items = []                       # (op, sub, dm0, dm1, dn0, dn1, k0, k1), offsets relative to the op
    for i, op in enumerate(s.ops):
        mlen, nlen, klen = len(op.m_bound), len(op.n_bound), len(op.k_bound)
        pa = pulled(i, s.a_src[i])
        pb = pulled(i, s.b_src[i]) if s.b_src[i] != s.a_src[i] else 0
        unfused_remote = s.c_remote[i] and not cfg.fused_accumulate
        nsub, dim = 1, None
        if row_cuts is not None and i in row_cuts:
            cuts_i = sorted({0, mlen} | {c for c in row_cuts[i] if 0 < c < mlen})
            for t in range(len(cuts_i) - 1):
                items.append((i, t, cuts_i[t], cuts_i[t + 1], 0, nlen, 0, klen))
            continue
        if not unfused_remote and pa + pb >= _SPLIT_BYTES:
            if cfg.k_split > 1 and klen >= 2 * _SPLIT_MIN:
                nsub, dim = int(min(cfg.k_split, klen // _SPLIT_MIN, max(2, (pa + pb) // _SPLIT_BYTES))), "k"
            elif cfg.mn_split > 1 and pa >= pb and mlen >= 2 * _SPLIT_MIN:
                nsub, dim = int(min(cfg.mn_split, mlen // _SPLIT_MIN)), "m"
            elif cfg.mn_split > 1 and pb > pa and nlen >= 2 * _SPLIT_MIN:
                nsub, dim = int(min(cfg.mn_split, nlen // _SPLIT_MIN)), "n"
        full = {"m": mlen, "n": nlen, "k": klen}
        cut = sorted({0, full[dim]} | {full[dim] * t // nsub // 64 * 64 for t in range(1, nsub)}) if dim else [0, 0]
        for t in range(len(cut) - 1):
            lo, hi = cut[t], cut[t + 1]
            mm = (lo, hi) if dim == "m" else (0, mlen)
            nn = (lo, hi) if dim == "n" else (0, nlen)
            kk = (lo, hi) if dim == "k" else (0, klen)
            items.append((i, t, *mm, *nn, *kk))

    # device order: items writing the same C region run back to back (K1 chains
    # them into one accumulator: one epilogue per tile), groups in order of first
    # appearance; the pulls then arrive in the order those chains need them.
    # (RunStats keep the reference's execution order: this is device-internal.)
    if cfg.chain_order:
        def ckey(it):
            i, t, m0, m1, n0, n1, k0, k1 = it
            cl = s.ops[i].c_local
            return (s.ops[i].c_tile, cl.rows.lo + m0, cl.rows.lo + m1, cl.cols.lo + n0, cl.cols.lo + n1)

        first = {}
        for pos, it in enumerate(items):
            first.setdefault(ckey(it), pos)
        items = sorted(items, key=lambda it: first[ckey(it)])      # stable: k order kept inside a chain

    # in-kernel pulls are cut into bands along the dimension in which the
    # (sub-)ops' slices differ, so an op waits only for the slab it reads
    # (cfg5: a 64 MiB B tile feeds 4 ops with one 16 MiB k-slab each)
    uses = [[] for _ in range(nf)]
    for it, (i, t, m0, m1, n0, n1, k0, k1) in enumerate(items):
        op = s.ops[i]
        a, b = op.a_local, op.b_local
        for src, (r0, r1, c0, c1) in ((s.a_src[i], (a.rows.lo + m0, a.rows.lo + m1, a.cols.lo + k0, a.cols.lo + k1)),
                                      (s.b_src[i], (b.rows.lo + k0, b.rows.lo + k1, b.cols.lo + n0, b.cols.lo + n1))):
            if src >= 0:
                f = s.fetches[src]
                uses[src].append((it, r0 - f.r0, r1 - f.r0, c0 - f.c0, c1 - f.c0))
    bands = [None] * nf              # per fetch: list of (r0, r1, c0, c1) in staged-buffer coordinates
    need = {}                        # (item, fetch) -> band indices
    for j, f in enumerate(s.fetches):
        if not in_kernel[j]:
            continue
        H, W = f.r1 - f.r0, f.c1 - f.c0
        sl = uses[j]
        # cells of the grid spanned by the slices' row and column boundaries;
        # keep the cells some slice reads
        rcuts = sorted({x for _, r0, r1, _, _ in sl for x in (r0, r1)})
        ccuts = sorted({x for _, _, _, c0, c1 in sl for x in (c0, c1)})
        cand = [(r0, r1, c0, c1) for r0, r1 in zip(rcuts, rcuts[1:]) for c0, c1 in zip(ccuts, ccuts[1:])]

        def key(bd, u):
            return bd[0] < u[2] and u[1] < bd[1] and bd[2] < u[4] and u[3] < bd[3]

        cand = [bd for bd in cand if any(key(bd, u) for u in sl)]    # drop cells no op reads
        if len(cand) > 16:
            cand = [(0, H, 0, W)]
        bands[j] = cand
        for u in sl:
            need[(u[0], j)] = [k for k, bd in enumerate(cand) if key(bd, u)]
    return items, bands, need


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
        for ev in start_events:
            self.gs.wait_event(ev)
            self.cs.wait_event(ev)

    def _mat(self, name):
        return self.A if name == "A" else self.B

    def issue(self):
        """Replay this rank's issue plan (built once per schedule and knob set)."""
        key = (self.cfg.get_engine, self.cfg.gemm_batch, self.cfg.max_inflight_accums, self.cfg.fused_accumulate,
               self.cfg.k_split, self.cfg.mn_split, self.cfg.chain_order, _SPLIT_BYTES, _SPLIT_MIN, self.signals_key)
        plans = self.sched.__dict__.setdefault("plans", {})
        plan = plans.get(key)
        if plan is None:
            plan = plans[key] = self._build_plan()
        self._replay(plan)
        return self

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
        # which pulls run inside the K1 launch: every op reading the staged slice
        # must see a TMA-readable view of it (16-byte column start); the rest go
        # through the copy engines with host-side ordering
        in_kernel = [self.cfg.get_engine == "kernel"] * nf
        for i in range(len(s.ops)):
            for src, v in ((s.a_src[i], views[i][0]), (s.b_src[i], views[i][1])):
                if src >= 0 and not _tma_ok(v):
                    in_kernel[src] = False

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

        for j, f in enumerate(s.fetches):
            if not in_kernel[j]:
                plan.host_fetches.append((j, *fetch_views(j)))
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
            _capi.check(lib.um_gemm_prepare(arr, len(batch), garr, len(batch_gets), self.dev, ctypes.byref(h)),
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

        for it, (i, t, m0, m1, n0, n1, k0, k1) in enumerate(items):
            op = s.ops[i]
            srcs = [j for j in (s.a_src[i], s.b_src[i]) if j >= 0]
            for j in srcs:
                if not in_kernel[j]:
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
            g.a_get = int(s.a_src[i] >= 0 and in_kernel[s.a_src[i]])
            g.b_get = int(s.b_src[i] >= 0 and in_kernel[s.b_src[i]])
            g.get_mask = sum(1 << gets_slot[u] for u in units if u in gets_slot)
            if self.signals is not None and i in self.signals:
                g.done_flag = self.signals[i][1](m0, m1)
            batch.append(g)
            batch_remote += int(remote)
        flush()
        # RunStats report the reference's execution order (runtime.py:213-236),
        # whatever order the device runs the (sub-)ops in
        st.executed_ops = list(s.ops)
        st.a_requests = [op.a_tile for op in s.ops]
        st.b_requests = [op.b_tile for op in s.ops]
        plan.final_waits = [j for j in range(nf) if not in_kernel[j] and not waited[j]]
        st.peak_inflight_gemms = 1 if s.ops else 0
        return plan

    def _replay(self, plan: "_IssuePlan"):
        lib = _capi.load()
        fab = self.fab
        with torch.cuda.device(self.dev):
            events = {}
            gsp = ctypes.c_void_p(self.gs.cuda_stream)
            for j, src, dst in plan.host_fetches:        # K2 on the copy engines, first-use order
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
            # join the get stream back even when it carried nothing (keeps the
            # multiply capturable into a CUDA graph: no unjoined forked stream)
            ev = torch.cuda.Event()
            ev.record(self.gs)
            self.cs.wait_event(ev)
            self.done = torch.cuda.Event()
            self.done.record(self.cs)
        fab.counters.merge(plan.traffic)
        t = plan.stats
        self.stats = RunStats(list(t.executed_ops), list(t.a_requests), list(t.b_requests), t.peak_inflight_gemms,
                              t.peak_inflight_accums, t.pool_acquired, t.pool_released, t.pool_peak, 0, t.gets,
                              t.staged_bytes, t.launches, t.peak_ops_per_launch)

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
# K4: replica reduction
# ---------------------------------------------------------------------------

def reduce_replicas(C: DistributedMatrix, origin: int = 0, distributed: bool = True, start_events=None,
                    rows: tuple[int, int] | None = None):
    """replica[origin] += sum_{r != origin} replica[r] (in r order), K4 on device.

    distributed: tile rows are split into c slices; slice j is reduced by the
    GPU of replica j's tile owner (slice `origin` by the origin owner), which
    pulls that slice from every other replica over NVLink and adds the sum
    into the origin's slice.
    """
    fab = C.fabric
    fab._require_data()
    lib = _capi.load()
    if start_events is None:
        start_events = _current_events(fab)
    done = []
    for t in C.grid.tiles():
        dst = C.segment(t, origin)
        if dst.length == 0:
            continue
        srcs = [C.segment(t, r) for r in range(C.c) if r != origin]
        nslices = C.c if distributed else 1
        lo, hi = 0, dst.rows
        if rows is not None:     # restrict to a global row window
            tb = C.tile_bounds(t)
            lo, hi = max(rows[0], tb.rows.lo) - tb.rows.lo, min(rows[1], tb.rows.hi) - tb.rows.lo
            if hi <= lo:
                continue
        for j in range(nslices):
            r0, r1 = lo + (hi - lo) * j // nslices, lo + (hi - lo) * (j + 1) // nslices
            if r1 <= r0:
                continue
            reducer = C.owner_rank(t, j) if distributed else dst.owner
            if not fab.is_local(reducer):
                continue
            dev = fab.device_of(reducer)
            stream = fab.stream(reducer, "reduce")
            for ev in start_events:
                stream.wait_event(ev)
            dv = dst.um_view(r0, r1, 0, dst.cols)
            sv = (_capi.UmView * len(srcs))(*[s.um_view(r0, r1, 0, s.cols) for s in srcs])
            with torch.cuda.device(dev):
                _capi.check(lib.um_reduce_replicas(ctypes.byref(dv), sv, len(srcs), ctypes.c_void_p(stream.cuda_stream)),
                            "um_reduce_replicas")
            ev = torch.cuda.Event()
            ev.record(stream)
            done.append(ev)
    _join_current(fab, done)
    if fab.world.size > 1:
        fab.synchronize()
    return done


# ---------------------------------------------------------------------------
# IR replay (runtime.py:259-336)
# ---------------------------------------------------------------------------

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
    key = ("cross", id(B), id(C), cfg.stationarity, cfg.staging, cfg.same_device_gets)
    cache = A.__dict__.setdefault("_sched_cache", {})
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


class _ReduceOverlap:
    """Replica reduction overlapped with the GEMMs (replicated C, Stationary C).

    Every C tile is cut into c * panels row sub-slices (multiples of 256 rows,
    the K1 tile height); sub-slice k is reduced by the owner of replica
    k mod c (the distributed K4 of reduce_replicas, at finer grain, so every
    reducer's work arrives spread over the GEMM).  Each rank's ops are split at
    the sub-slice rows and carry a done_flag pointing at a word on the
    sub-slice's reducer (symmetric heap: a peer or IPC-mapped address); the K1
    epilogue adds the number of finished ops there (release, system scope).
    The reducer's stream waits (um_wait_geq, a stream memory operation, no SM
    held) for every contributing op of every replica in this run, then runs
    K4 for the sub-slice.  Flags only grow: run e waits for e * expected.
    """

    def __init__(self, A, B, C, cfg: ExecConfig):
        fab = C.fabric
        p, c = fab.nprocs, C.c
        self.C = C
        self.subs = {}
        n = c * cfg.reduce_panels
        for t in C.grid.tiles():
            rows = len(C.tile_bounds(t).rows)
            cuts = sorted({0, rows} | {rows * s // n // 256 * 256 for s in range(1, n)})
            self.subs[t] = [(cuts[k], cuts[k + 1], k % c) for k in range(len(cuts) - 1)]
        counts = [0] * p
        self.word = {}
        for t, lst in self.subs.items():
            for k, (_, _, rep) in enumerate(lst):
                red = C.owner_rank(t, rep)
                self.word[(t, k)] = (red, counts[red])
                counts[red] += 1
        # flag words live in the symmetric heap (same allocation order on every process)
        self.flag_segs = [fab.alloc_tile(r, 1, max(1, counts[r]), torch.float32) for r in range(p)]
        for seg in self.flag_segs:
            if seg.storage is not None:
                with torch.cuda.device(seg.device):
                    seg.storage.zero_()
        fab.heap.exchange()
        # ops contributing to each sub-slice, over every replica's owner (host-only planning)
        self.expected = {}
        for r in range(p):
            for op in lower_direct(A, B, C, cfg, r).ops:
                lo, hi = op.c_local.rows.lo, op.c_local.rows.hi
                for k, (r0, r1, _) in enumerate(self.subs[op.c_tile]):
                    if lo < r1 and r0 < hi:
                        self.expected[(op.c_tile, k)] = self.expected.get((op.c_tile, k), 0) + 1
        self.epoch = 0
        if fab.world.size > 1:
            fab.synchronize()        # zeroed flags in place before any process can signal

    def sub_slice_of(self, t, row: int) -> int:
        """Index of the sub-slice of C tile t holding tile-local `row`."""
        for k, (r0, r1, _) in enumerate(self.subs[t]):
            if r0 <= row < r1:
                return k
        raise AssertionError("row outside its C tile")

    def flag_ptr(self, t, k) -> int:
        red, idx = self.word[(t, k)]
        return self.flag_segs[red].ptr + 4 * idx

    def signals_for(self, sched: DirectSchedule) -> dict:
        sig = {}
        for i, op in enumerate(sched.ops):
            t, lo, hi = op.c_tile, op.c_local.rows.lo, op.c_local.rows.hi
            cuts = [r0 - lo for r0, _, _ in self.subs[t] if lo < r0 < hi]

            def flag(m0, m1, t=t, lo=lo):
                return self.flag_ptr(t, self.sub_slice_of(t, lo + m0))

            sig[i] = (cuts, flag)
        return sig

    def reduce(self, start_events) -> list:
        """Enqueue wait + K4 per sub-slice on the reducers' streams; return done events."""
        C, fab = self.C, self.C.fabric
        lib = _capi.load()
        self.epoch += 1
        done = []
        for t, lst in self.subs.items():
            dst = C.segment(t, 0)
            if dst.length == 0:
                continue
            srcs = [C.segment(t, r) for r in range(1, C.c)]
            for k, (r0, r1, rep) in enumerate(lst):
                red = C.owner_rank(t, rep)
                if not fab.is_local(red) or r1 <= r0:
                    continue
                dev = fab.device_of(red)
                stream = fab.stream(red, "reduce")
                for ev in start_events:
                    stream.wait_event(ev)
                sp = ctypes.c_void_p(stream.cuda_stream)
                exp = self.expected.get((t, k), 0)
                with torch.cuda.device(dev):
                    if exp:
                        _capi.check(lib.um_wait_geq(ctypes.c_void_p(self.flag_ptr(t, k)),
                                                    (self.epoch * exp) & 0xFFFFFFFF, sp), "um_wait_geq")
                    dv = dst.um_view(r0, r1, 0, dst.cols)
                    sv = (_capi.UmView * len(srcs))(*[s_.um_view(r0, r1, 0, s_.cols) for s_ in srcs])
                    _capi.check(lib.um_reduce_replicas(ctypes.byref(dv), sv, len(srcs), sp), "um_reduce_replicas")
                    ev = torch.cuda.Event()
                    ev.record(stream)
                done.append(ev)
        return done


def _overlap_for(A, B, C, cfg: ExecConfig):
    if not (cfg.overlap_reduce and cfg.reduce_distributed and C.c > 1
            and cfg.stationarity is Stationarity.STATIONARY_C):
        return None
    # processes time-sharing one GPU (no MPS) could park a stream wait that only
    # another process's kernel can satisfy: keep the barrier + K4 path there
    if C.fabric.devices_shared_across_processes() and os.environ.get("UM_OVERLAP_SHARED") != "1":
        return None
    key = ("ovl", id(A), id(B), cfg.reduce_panels, cfg.staging, cfg.same_device_gets)
    cache = C.__dict__.setdefault("_ovl_cache", {})
    hit = cache.get(key)
    if hit is not None and hit[0] is A and hit[1] is B:
        return hit[2]
    ovl = _ReduceOverlap(A, B, C, cfg)
    cache[key] = (A, B, ovl)
    return ovl


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
        for r in ranks:
            sched = lower_direct(A, B, C, cfg, r)
            _count_reference_traffic(A, B, C, cfg, sched)
            run = _RankRun(A, B, C, cfg, sched, start)
            if ovl is not None:
                run.signals, run.signals_key = ovl.signals_for(sched), ("ovl", id(ovl))
            runs.append(run.issue())
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
    if ovl is not None:
        # K4 per sub-slice, each started by its replicas' completion signals
        # (no run-level barrier between the GEMMs and the reduction)
        _join_current(fab, ovl.reduce(start) + done)
        if fab.world.size > 1:
            fab.synchronize()
    elif cross:
        fab.synchronize()            # run-level barrier across processes
    if C.c > 1 and ovl is None:
        reduce_replicas(C, 0, distributed=cfg.reduce_distributed, start_events=done)
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
