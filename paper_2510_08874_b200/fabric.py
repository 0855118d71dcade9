"""One-sided fabric over B200 HBM and NVLink (drop-in for unimul.fabric).

The reference simulates a one-sided fabric inside one Python process
(fabric.py:135-242): symmetric segments per logical rank, `get`/`get_async`
snapshots, element-wise `accumulate` (PEER_ATOMIC or LOCK_GET_PUT) and
owner-only `local_view`, with byte/message/flop counters.  Here the segments
are real device allocations:

* single process, several GPUs: logical rank r lives on devices[r % ndev]
  (oversubscription allowed, e.g. the 12-rank sweep on 8 or 1
  GPUs); peer access is enabled between all of them (um_init), so a remote
  pointer is directly addressable by copy engines and kernels;
* one process per GPU (torchrun): rank r is hosted by process r % world on
  that process's device; segments come from a symmetric heap whose chunks
  are exchanged once as CUDA IPC handles (see heap.py).

Transfers go through the C-ABI (um_get = K2 copy-engine pull, um_accumulate
= K3 red.global.add).  Counters keep the reference's accounting model
(8 bytes per element, whole-tile gets: fabric.py:19,152-154) so volume
comparisons stay drop-in comparable; `wire_bytes` records what actually
crossed (storage dtype, fetch-once slices).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from paper_2510_08874_b200 import _capi
from paper_2510_08874_b200.errors import ContractError
from paper_2510_08874_b200.tiling import Range

ELEM_BYTES = 8  # reference accounting unit per element (fabric.py:19)

_TORCH_TO_UM = {torch.bfloat16: _capi.UM_BF16, torch.float32: _capi.UM_F32}


def um_dtype(dt: torch.dtype) -> int:
    try:
        return _TORCH_TO_UM[dt]
    except KeyError:
        raise ContractError(f"unsupported storage dtype {dt}; use torch.bfloat16 or torch.float32") from None


def pitch_for(cols: int, dtype: torch.dtype) -> int:
    """Row pitch in elements, rounded up to 16 bytes (TMA stride rule)."""
    per16 = 16 // torch.empty((), dtype=dtype).element_size()
    return max(per16, -(-cols // per16) * per16)


class AccumulateMode(Enum):
    PEER_ATOMIC = "peer_atomic"
    LOCK_GET_PUT = "lock_get_put"


@dataclass(eq=False)
class SymSegment:
    """A symmetric-memory segment owned by one logical rank (fabric.py:27-38).

    Storage is a row-major (rows x pitch) device tensor; the logical contents
    are rows x cols (`length` = rows*cols elements, as in the reference).
    `storage` is None when the owner lives in another process; `ptr` is then
    the IPC-mapped address.
    """

    owner: int
    length: int
    rows: int
    cols: int
    pitch: int
    dtype: torch.dtype
    device: int
    storage: torch.Tensor | None = field(default=None, repr=False)
    ptr: int = 0
    lock: threading.Lock = field(default_factory=threading.Lock, repr=False)

    @property
    def esize(self) -> int:
        return torch.empty((), dtype=self.dtype).element_size()

    def view2d(self) -> torch.Tensor:
        if self.storage is None:
            raise ContractError(f"segment of rank {self.owner} is not addressable from this process")
        return self.storage[:, : self.cols]

    @property
    def data(self) -> torch.Tensor:
        """Logical contents: flat when unpadded (as the reference), else rows x cols."""
        v = self.view2d()
        return v.reshape(-1) if self.pitch == self.cols or self.rows <= 1 else v

    def um_view(self, r0: int, r1: int, c0: int, c1: int) -> _capi.UmView:
        return _capi.UmView(self.ptr, r0, r1, c0, c1, self.pitch, um_dtype(self.dtype), self.device)

    def row_pieces(self, lo: int, hi: int):
        """Split flat logical range [lo,hi) into (row0, row1, col0, col1) rectangles."""
        if hi <= lo:
            return []
        cols = max(self.cols, 1)
        pieces = []
        r, c = divmod(lo, cols)
        er, ec = divmod(hi, cols)
        if r == er:
            return [(r, r + 1, c, ec)]
        if c:
            pieces.append((r, r + 1, c, cols))
            r += 1
        if er > r:
            pieces.append((r, er, 0, cols))
        if ec:
            pieces.append((er, er + 1, 0, ec))
        return pieces


class PendingCopy:
    """Future for an asynchronous get; wait() exactly once (fabric.py:41-58).

    The copy is in flight on the caller device's stream when get_async
    returns; wait() orders the caller's current stream after it.
    """

    def __init__(self, buffer: torch.Tensor, event: torch.cuda.Event, on_wait):
        self._buffer = buffer
        self._event = event
        self._on_wait = on_wait
        self._done = False

    def wait(self) -> torch.Tensor:
        if self._done:
            raise RuntimeError("PendingCopy waited on twice")
        self._done = True
        torch.cuda.current_stream(self._buffer.device).wait_event(self._event)
        self._on_wait(self)
        return self._buffer

    @property
    def complete(self) -> bool:
        return self._done


class FabricCounters:
    """Per-(initiator, peer) traffic and per-rank flops (fabric.py:61-107).

    `bytes`/`msgs` follow the reference model (ELEM_BYTES per element);
    `wire_bytes` counts the bytes the B200 path actually moved.
    """

    def __init__(self, nprocs: int):
        self.nprocs = nprocs
        self.bytes = np.zeros((nprocs, nprocs), dtype=np.int64)
        self.msgs = np.zeros((nprocs, nprocs), dtype=np.int64)
        self.wire_bytes = np.zeros((nprocs, nprocs), dtype=np.int64)
        self.flops = np.zeros(nprocs, dtype=np.int64)
        self._lock = threading.Lock()

    def add_traffic(self, initiator: int, peer: int, nbytes: int, nmsgs: int = 1, wire: int = 0):
        with self._lock:
            self.bytes[initiator, peer] += nbytes
            self.msgs[initiator, peer] += nmsgs
            self.wire_bytes[initiator, peer] += wire

    def merge(self, other: "FabricCounters"):
        """Add another counter set (same rank count) into this one."""
        with self._lock:
            self.bytes += other.bytes
            self.msgs += other.msgs
            self.wire_bytes += other.wire_bytes
            self.flops += other.flops

    def add_flops(self, rank: int, flops: int):
        with self._lock:
            self.flops[rank] += flops

    def comm_bytes(self) -> int:
        """Off-process bytes in the reference model (diagonal excluded)."""
        return int(self.bytes.sum() - np.trace(self.bytes))

    def local_bytes(self) -> int:
        return int(np.trace(self.bytes))

    def comm_wire_bytes(self) -> int:
        return int(self.wire_bytes.sum() - np.trace(self.wire_bytes))

    def total_flops(self) -> int:
        return int(self.flops.sum())

    def link_csv(self) -> str:
        out = ["src,dst,bytes,msgs"]
        for s, d in zip(*np.nonzero((self.bytes != 0) | (self.msgs != 0))):
            out.append(f"{s},{d},{self.bytes[s, d]},{self.msgs[s, d]}")
        return "\n".join(out) + "\n"

    def flops_csv(self) -> str:
        return "\n".join(["rank,flops"] + [f"{r},{f}" for r, f in enumerate(self.flops)]) + "\n"


class LinkTable:
    """Per-link bandwidth in bytes/s (fabric.py:110-132)."""

    def __init__(self, bandwidth: np.ndarray):
        bandwidth = np.asarray(bandwidth, dtype=float)
        if (bandwidth <= 0).any():
            raise ValueError("all link bandwidths must be positive")
        self.bandwidth = bandwidth

    @classmethod
    def uniform(cls, nprocs: int, bw: float) -> "LinkTable":
        return cls(np.full((nprocs, nprocs), float(bw)))

    @classmethod
    def two_level(cls, nprocs: int, group_size: int, intra_bw: float, inter_bw: float) -> "LinkTable":
        g = np.arange(nprocs) // group_size
        return cls(np.where(g[:, None] == g[None, :], float(intra_bw), float(inter_bw)))

    @classmethod
    def nvswitch(cls, nprocs: int, per_direction_bw: float = 7.7e11) -> "LinkTable":
        """B200 NVLink 5 through NVSwitch: uniform to every peer (measured peer copy ≈770 GB/s)."""
        return cls.uniform(nprocs, per_direction_bw)

    def bw(self, src: int, dst: int) -> float:
        return float(self.bandwidth[src, dst])


def _visible_devices() -> list[int]:
    n = ctypes.c_int32(0)
    _capi.check(_capi.load().um_device_count(ctypes.byref(n)), "um_device_count")
    return list(range(n.value))


class Fabric:
    """The shared one-sided substrate of p logical ranks (fabric.py:135-145).

    devices: CUDA devices to spread ranks over (default: all visible).  With
    no CUDA device the fabric is placement-only: planning, lowering and cost
    queries work, any data movement raises.
    """

    def __init__(self, nprocs: int, links: LinkTable | None = None, devices=None, process_group=None,
                 device_api=None, symmetric: str = "torch"):
        """symmetric: "torch" (segments from torch's caching allocator) or "vmm"
        (one-process mode: every segment its own um_sym_alloc block, bindable
        to an NVLS multicast team for reduce_mode="nvls")."""
        if nprocs < 1:
            raise ValueError("need at least one process")
        if symmetric not in ("torch", "vmm"):
            raise ValueError(f"unknown symmetric memory kind {symmetric!r}")
        self.symmetric = symmetric
        self.nprocs = nprocs
        self.links = links or LinkTable.uniform(nprocs, 1e9)
        self.counters = FabricCounters(nprocs)
        self._outstanding = 0
        self._outstanding_lock = threading.Lock()
        from paper_2510_08874_b200 import heap as _heap

        self.world = _heap.World.detect(process_group)
        if devices is None:
            devices = _visible_devices() if self.world.size == 1 else [torch.cuda.current_device()]
        self.devices = list(devices)
        self.placement_only = len(self.devices) == 0
        if not self.placement_only and self.world.size == 1 and len(self.devices) > 1:
            arr = (ctypes.c_int32 * len(self.devices))(*self.devices)
            _capi.check(_capi.load().um_init(len(self.devices), arr), "um_init")
        self.heap = _heap.SymmetricHeap(self, device_api)
        self._streams: dict = {}

    # -- placement ---------------------------------------------------------------

    def process_of(self, rank: int) -> int:
        return rank % self.world.size

    def is_local(self, rank: int) -> bool:
        """True when this process hosts logical rank `rank`."""
        return self.process_of(rank) == self.world.rank

    def device_of(self, rank: int) -> int:
        if self.placement_only:
            raise RuntimeError("placement-only fabric: no CUDA device available")
        if self.world.size > 1:
            return self.devices[0] if self.is_local(rank) else -1
        return self.devices[rank % len(self.devices)]

    def local_ranks(self) -> list[int]:
        return [r for r in range(self.nprocs) if self.is_local(r)]

    def stream(self, rank: int, kind: str) -> torch.cuda.Stream:
        """Per-(rank, role) stream: co-resident ranks overlap like separate processes."""
        key = (rank, kind)
        s = self._streams.get(key)
        if s is None:
            s = torch.cuda.Stream(device=self.device_of(rank))
            self._streams[key] = s
        return s

    def devices_shared_across_processes(self) -> bool:
        """True when two processes of the world drive the same physical GPU
        (e.g. several ranks on a one-GPU box).  Decided once, collectively."""
        if self.world.size == 1 or self.placement_only:
            return False
        if not hasattr(self, "_shared_devs"):
            uuid = str(torch.cuda.get_device_properties(self.devices[0]).uuid)
            ids = self.world.all_gather_object(uuid)
            self._shared_devs = len(set(ids)) < len(ids)
        return self._shared_devs

    def _require_data(self):
        if self.placement_only:
            raise RuntimeError("placement-only fabric (no CUDA device): data movement is unavailable")

    # -- allocation ----------------------------------------------------------------

    def alloc(self, owner: int, length: int, dtype: torch.dtype = torch.float32) -> SymSegment:
        """Flat segment of `length` elements (fabric.py:147-150)."""
        return self.alloc_tile(owner, 1 if length else 0, length, dtype)

    def alloc_tile(self, owner: int, rows: int, cols: int, dtype: torch.dtype) -> SymSegment:
        if not 0 <= owner < self.nprocs:
            raise ValueError(f"owner {owner} out of range")
        return self.heap.allocate(owner, rows, cols, dtype)

    # -- one-sided operations ---------------------------------------------------------

    def _count_get(self, seg: SymSegment, n: int, caller: int):
        if n > 0:
            self.counters.add_traffic(caller, seg.owner, ELEM_BYTES * n, 1, seg.esize * n)

    def _issue_get(self, seg: SymSegment, elem_range: Range, caller: int, out):
        self._require_data()
        lo, hi = elem_range.lo, elem_range.hi
        if hi > seg.length:
            raise IndexError(f"range {elem_range} outside segment of {seg.length}")
        n = hi - lo
        dev = self.device_of(caller)
        if out is None:
            buf = torch.empty(n, dtype=seg.dtype, device=f"cuda:{dev}")
        else:
            if out.dtype != seg.dtype or out.numel() < n:
                raise ContractError("get: out buffer has the wrong dtype or is too small")
            buf = out.reshape(-1)[:n]
        lib = _capi.load()
        stream = torch.cuda.current_stream(dev)
        self.heap.order_before_remote_access(seg, dev)
        with torch.cuda.device(dev):
            done = 0
            for r0, r1, c0, c1 in seg.row_pieces(lo, hi):
                cnt = (r1 - r0) * (c1 - c0)
                if r1 - r0 == 1:
                    dst = _capi.UmView(buf.data_ptr() + done * seg.esize, 0, 1, 0, c1 - c0, c1 - c0,
                                       um_dtype(seg.dtype), dev)
                else:
                    dst = _capi.UmView(buf.data_ptr() + done * seg.esize, 0, r1 - r0, 0, c1 - c0, c1 - c0,
                                       um_dtype(seg.dtype), dev)
                src = seg.um_view(r0, r1, c0, c1)
                _capi.check(lib.um_get(ctypes.byref(src), ctypes.byref(dst),
                                       ctypes.c_void_p(stream.cuda_stream)), "um_get")
                done += cnt
        self._count_get(seg, n, caller)
        return buf, stream

    def get(self, seg: SymSegment, elem_range: Range, caller: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """Snapshot of seg[lo:hi] on the caller's device (fabric.py:156-175)."""
        buf, _ = self._issue_get(seg, elem_range, caller, out)
        return buf

    def get_async(self, seg: SymSegment, elem_range: Range, caller: int,
                  out: torch.Tensor | None = None) -> PendingCopy:
        """As get(), returning a future (fabric.py:177-192); the copy is in flight."""
        buf, stream = self._issue_get(seg, elem_range, caller, out)
        ev = torch.cuda.Event()
        ev.record(stream)
        with self._outstanding_lock:
            self._outstanding += 1
        return PendingCopy(buf, ev, self._retire_copy)

    def _retire_copy(self, _pending: PendingCopy):
        with self._outstanding_lock:
            self._outstanding -= 1

    @property
    def outstanding_copies(self) -> int:
        """Issued-but-unwaited async gets; nonzero at teardown means a leak."""
        return self._outstanding

    def accumulate(self, seg: SymSegment, elem_range: Range, values, caller: int,
                   mode: AccumulateMode = AccumulateMode.PEER_ATOMIC):
        """Element-wise += into seg[lo:hi] (fabric.py:203-234).

        Both modes run the same atomic red.global.add kernel (K3); the mode
        selects the accounting (1x bytes/1 msg vs 2x bytes/2 msgs).
        """
        lo, hi = elem_range.lo, elem_range.hi
        if hi > seg.length:
            raise IndexError(f"range {elem_range} outside segment of {seg.length}")
        n = hi - lo
        vals = torch.as_tensor(values)
        if vals.numel() != n:
            raise ContractError(f"payload of {vals.numel()} for range of {n}")
        if n == 0:
            return
        self._require_data()
        if seg.dtype != torch.float32:
            raise ContractError("accumulate targets must be float32 segments")
        dev = self.device_of(caller)
        vals = vals.reshape(-1).to(device=f"cuda:{dev}", dtype=torch.float32).contiguous()
        lib = _capi.load()
        stream = torch.cuda.current_stream(dev)
        self.heap.order_before_remote_access(seg, dev)
        with torch.cuda.device(dev):
            done = 0
            for r0, r1, c0, c1 in seg.row_pieces(lo, hi):
                w = c1 - c0
                src = _capi.UmView(vals.data_ptr() + done * 4, 0, r1 - r0, 0, w, w, _capi.UM_F32, dev)
                dst = seg.um_view(r0, r1, c0, c1)
                _capi.check(lib.um_accumulate(ctypes.byref(src), ctypes.byref(dst),
                                              ctypes.c_void_p(stream.cuda_stream)), "um_accumulate")
                done += (r1 - r0) * w
        self.heap.mark_remote_write(seg, dev)
        if mode is AccumulateMode.PEER_ATOMIC:
            self.counters.add_traffic(caller, seg.owner, ELEM_BYTES * n, 1, 4 * n)
        else:
            self.counters.add_traffic(caller, seg.owner, 2 * ELEM_BYTES * n, 2, 8 * n)

    def local_view(self, seg: SymSegment, caller: int) -> torch.Tensor:
        """Zero-copy view of a segment; owner only (fabric.py:236-242)."""
        if caller != seg.owner:
            raise ContractError(f"rank {caller} asked for a local view of rank {seg.owner}'s segment")
        return seg.data

    def synchronize(self):
        """Host barrier over every device this process uses."""
        if self.placement_only:
            return
        for d in sorted({self.device_of(r) for r in self.local_ranks()}):
            torch.cuda.synchronize(d)
        self.world.barrier()
