"""K4: replica reduction (distmatrix.py:211-232), barrier form and overlapped form."""

from __future__ import annotations

import ctypes
import os

import torch

from paper_2510_08874_b200.trace import nvtx
from paper_2510_08874_b200 import _capi
from paper_2510_08874_b200.config import ExecConfig
from paper_2510_08874_b200.distmatrix import DistributedMatrix
from paper_2510_08874_b200.engine import _current_events, _join_current
from paper_2510_08874_b200.opgen import Stationarity
from paper_2510_08874_b200.schedule import DirectSchedule, lower_direct


REDUCE_MODES = ("auto", "peer", "nccl", "nvls")


class _NvlsTeam:
    """Multicast team over the c replicas of one C tile (um_nvls_team_create)."""

    def __init__(self, C, t):
        segs = [C.segment(t, r) for r in range(C.c)]
        devs = (ctypes.c_int32 * C.c)(*[s_.device for s_ in segs])
        ptrs = (ctypes.c_void_p * C.c)(*[s_.vmm.ptr for s_ in segs])
        mc = (ctypes.c_void_p * C.c)()
        h = ctypes.c_void_p()
        nbytes = max(s_.vmm.nbytes for s_ in segs)
        _capi.check(_capi.load().um_nvls_team_create(C.c, devs, ptrs, nbytes, mc, ctypes.byref(h)),
                    "um_nvls_team_create")
        self.handle = h.value
        self.mc = {s_.device: int(mc[i]) for i, s_ in enumerate(segs)}
        self._keep = segs

    def view(self, seg, device: int, r0: int, r1: int) -> _capi.UmView:
        """Rows [r0, r1) of the tile in the team's multicast space, as mapped on `device`."""
        return _capi.UmView(self.mc[device], r0, r1, 0, seg.cols, seg.pitch, _capi.UM_F32, device)

    def __del__(self):
        try:
            _capi.load().um_nvls_team_destroy(ctypes.c_void_p(self.handle))
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


def nvls_capable(C: DistributedMatrix) -> tuple[bool, str]:
    """Can K4 run in the switch (NVLS) for C?  (capability probe, no side effects)"""
    fab = C.fabric
    if C.c < 2:
        return False, "C is not replicated"
    if fab.world.size > 1:
        return False, "NVLS teams are built in one-process mode (multicast handles are not exchanged)"
    if getattr(fab, "symmetric", "torch") != "vmm":
        return False, "C's segments are not VMM symmetric memory (Fabric(symmetric='vmm'))"
    lib = _capi.load()
    for t in C.grid.tiles():
        devs = [C.segment(t, r).device for r in range(C.c)]
        if len(set(devs)) < C.c:
            return False, f"replicas of tile {t} share a device ({devs}): a multicast team needs distinct GPUs"
    ok = ctypes.c_int32(0)
    for d in sorted({C.segment(t, r).device for t in C.grid.tiles() for r in range(C.c)}):
        _capi.check(lib.um_nvls_supported(d, ctypes.byref(ok)), "um_nvls_supported")
        if not ok.value:
            return False, f"device {d} does not support multicast objects (NVLS)"
    return True, "ok"


def nccl_capable(C: DistributedMatrix) -> tuple[bool, str]:
    fab = C.fabric
    if C.c < 2:
        return False, "C is not replicated"
    if fab.world.size > 1:
        import torch.distributed as dist

        if dist.get_backend(fab.world.group) != "nccl":
            return False, "the process group is not NCCL"
        if fab.devices_shared_across_processes():
            return False, "processes share a GPU (NCCL needs one GPU per rank)"
        for t in C.grid.tiles():
            if len({fab.process_of(C.owner_rank(t, r)) for r in range(C.c)}) < C.c:
                return False, f"two replicas of tile {t} live in one process"
        return True, "ok"
    for t in C.grid.tiles():
        devs = [C.segment(t, r).device for r in range(C.c)]
        if len(set(devs)) < C.c:
            return False, f"replicas of tile {t} share a device ({devs}): NCCL needs distinct GPUs"
    return True, "ok"


def resolve_reduce_mode(C: DistributedMatrix, mode: str) -> str:
    """"auto" -> "nvls" when capable, else "peer" (one-sided, overlappable).  An
    explicitly requested mode that cannot run raises ConfigError."""
    from paper_2510_08874_b200.errors import ConfigError

    if mode not in REDUCE_MODES:
        raise ConfigError(f"unknown reduce mode {mode!r} (one of {REDUCE_MODES})")
    if mode == "auto":
        return "nvls" if nvls_capable(C)[0] else "peer"
    if mode == "nvls":
        ok, why = nvls_capable(C)
        if not ok:
            raise ConfigError(f"reduce_mode='nvls' unavailable: {why}")
    if mode == "nccl":
        ok, why = nccl_capable(C)
        if not ok:
            raise ConfigError(f"reduce_mode='nccl' unavailable: {why}")
    return mode


def _nvls_team(C, t) -> _NvlsTeam:
    teams = C.__dict__.setdefault("_nvls_teams", {})
    if t not in teams:
        teams[t] = _NvlsTeam(C, t)
    return teams[t]


def _reduce_nccl(C, origin, start_events, rows):
    """K4 as NCCL reduce (SURVEY §7 K4 option b): per C tile, the replica owners
    reduce into the origin's tile (ncclReduce over NVLink).  Single process:
    torch.cuda.nccl over the tile's devices; one process per GPU: the process
    group, one subgroup per replica set."""
    import torch.cuda.nccl as tnccl

    fab = C.fabric
    done = []
    if fab.world.size == 1:
        for t in C.grid.tiles():
            segs = [C.segment(t, r) for r in range(C.c)]
            if segs[origin].length == 0:
                continue
            lo, hi = 0, segs[origin].rows
            if rows is not None:
                tb = C.tile_bounds(t)
                lo, hi = max(rows[0], tb.rows.lo) - tb.rows.lo, min(rows[1], tb.rows.hi) - tb.rows.lo
                if hi <= lo:
                    continue
            streams = []
            for s_ in segs:
                st_ = fab.stream(s_.owner, "reduce")
                for ev in start_events:
                    st_.wait_event(ev)
                streams.append(st_)
            tnccl.reduce([s_.storage[lo:hi] for s_ in segs], root=origin, streams=streams)
            for st_ in streams:
                ev = torch.cuda.Event()
                ev.record(st_)
                done.append(ev)
        return done
    import torch.distributed as dist

    groups = C.__dict__.get("_nccl_groups")
    if groups is None:
        groups = {}
        for t in C.grid.tiles():          # same order on every process (new_group is collective)
            procs = tuple(sorted({fab.process_of(C.owner_rank(t, r)) for r in range(C.c)}))
            if procs not in groups:
                groups[procs] = dist.new_group(list(procs))
        C.__dict__["_nccl_groups"] = groups
    for t in C.grid.tiles():
        procs = tuple(sorted({fab.process_of(C.owner_rank(t, r)) for r in range(C.c)}))
        mine = [r for r in range(C.c) if fab.is_local(C.owner_rank(t, r))]
        if not mine:
            continue
        seg = C.segment(t, mine[0])
        lo, hi = 0, seg.rows
        if rows is not None:
            tb = C.tile_bounds(t)
            lo, hi = max(rows[0], tb.rows.lo) - tb.rows.lo, min(rows[1], tb.rows.hi) - tb.rows.lo
            if hi <= lo:
                continue
        st_ = fab.stream(seg.owner, "reduce")
        for ev in start_events:
            st_.wait_event(ev)
        with torch.cuda.device(seg.device), torch.cuda.stream(st_):
            buf = seg.storage[lo:hi]
            dist.reduce(buf, dst=fab.process_of(C.owner_rank(t, origin)), group=groups[procs])
            ev = torch.cuda.Event()
            ev.record(st_)
        done.append(ev)
    return done


@nvtx("um:K4_reduce_replicas")
def reduce_replicas(C: DistributedMatrix, origin: int = 0, distributed: bool = True, start_events=None,
                    rows: tuple[int, int] | None = None, mode: str = "peer"):
    """replica[origin] += sum_{r != origin} replica[r] (in r order), K4 on device.

    distributed: tile rows are split into c slices; slice j is reduced by the
    GPU of replica j's tile owner (slice `origin` by the origin owner), which
    pulls that slice from every other replica over NVLink and adds the sum
    into the origin's slice.
    mode: "peer" (P2P loads, the reference's summation order), "nvls" (one
    multimem.ld_reduce per 16 bytes through the tile's multicast team: the
    switch adds the replicas), "nccl" (ncclReduce per tile), "auto" (nvls
    when capable, else peer).  See resolve_reduce_mode.
    """
    fab = C.fabric
    fab._require_data()
    lib = _capi.load()
    if start_events is None:
        start_events = _current_events(fab)
    mode = resolve_reduce_mode(C, mode) if C.c > 1 else "peer"
    if mode == "nccl":
        done = _reduce_nccl(C, origin, start_events, rows)
        _join_current(fab, done)
        if fab.world.size > 1:
            fab.synchronize()
        return done
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
            if mode == "nvls":
                sv = (_capi.UmView * 1)(_nvls_team(C, t).view(dst, dev, r0, r1))
                nsrc, kmode = 1, _capi.UM_REDUCE_NVLS
            else:
                sv = (_capi.UmView * len(srcs))(*[s.um_view(r0, r1, 0, s.cols) for s in srcs])
                nsrc, kmode = len(srcs), _capi.UM_REDUCE_PEER
            with torch.cuda.device(dev):
                _capi.check(lib.um_reduce_replicas(ctypes.byref(dv), sv, nsrc, kmode,
                                                   ctypes.c_void_p(stream.cuda_stream)), "um_reduce_replicas")
            ev = torch.cuda.Event()
            ev.record(stream)
            done.append(ev)
    _join_current(fab, done)
    if fab.world.size > 1:
        fab.synchronize()
    return done


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

    @nvtx("um:K4_overlapped")
    def reduce(self, start_events, mode: str = "peer") -> list:
        """Enqueue wait + K4 per sub-slice on the reducers' streams; return done events.
        mode: "peer" or "nvls" (resolved by the caller)."""
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
                    if mode == "nvls":
                        sv = (_capi.UmView * 1)(_nvls_team(C, t).view(dst, dev, r0, r1))
                        _capi.check(lib.um_reduce_replicas(ctypes.byref(dv), sv, 1, _capi.UM_REDUCE_NVLS, sp),
                                    "um_reduce_replicas")
                    else:
                        sv = (_capi.UmView * len(srcs))(*[s_.um_view(r0, r1, 0, s_.cols) for s_ in srcs])
                        _capi.check(lib.um_reduce_replicas(ctypes.byref(dv), sv, len(srcs), _capi.UM_REDUCE_PEER,
                                                           sp), "um_reduce_replicas")
                    ev = torch.cuda.Event()
                    ev.record(stream)
                done.append(ev)
        return done


def _overlap_for(A, B, C, cfg: ExecConfig):
    if not (cfg.overlap_reduce and cfg.reduce_distributed and C.c > 1
            and cfg.stationarity is Stationarity.STATIONARY_C):
        return None
    if resolve_reduce_mode(C, cfg.reduce_mode) == "nccl":
        return None                  # a two-sided collective: barrier form
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
