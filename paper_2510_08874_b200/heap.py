"""Symmetric memory for the one-sided fabric (single- and multi-process).

The paper allocates every rank's tiles from a pre-registered symmetric pool
(PAPER.md:208-210); the reference simulates it with one numpy array per
segment (fabric.py:147-150).  Here:

* one process driving all GPUs: each segment is a device tensor on its owner
  rank's GPU (torch caching allocator); peer pointers are valid everywhere
  because um_init enabled peer access;
* one process per GPU (torchrun): every process replays the same SPMD
  allocation sequence, so the (process, chunk, offset) of every segment is
  known everywhere without communication.  Each process backs only its own
  chunks (cudaMalloc via um_device_alloc); chunk bases are published once as
  CUDA IPC handles (`SymmetricHeap.exchange`, a collective) and remote
  segments resolve to IPC-mapped pointers.

Cross-device stream ordering for the API-level fabric calls is kept here too
(order_before_remote_access / mark_remote_write).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from paper_2510_08874_b200 import _capi

ALIGN = 256
FIRST_CHUNK = 64 << 20
MAX_CHUNK = 4 << 30


def _align(n: int, a: int = ALIGN) -> int:
    return -(-n // a) * a


class World:
    """Process group view: size/rank plus the two collectives the heap needs."""

    def __init__(self, size: int = 1, rank: int = 0, group=None):
        self.size, self.rank, self.group = size, rank, group

    @classmethod
    def detect(cls, process_group=None) -> "World":
        import torch.distributed as dist

        if process_group is not None:
            return cls(dist.get_world_size(process_group), dist.get_rank(process_group), process_group)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return cls(dist.get_world_size(), dist.get_rank(), None)
        return cls()

    def barrier(self):
        if self.size > 1:
            import torch.distributed as dist

            dist.barrier(group=self.group)

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        """Element-wise sum over processes (used by the collective gather)."""
        if self.size == 1:
            return t
        import torch.distributed as dist

        backend = dist.get_backend(self.group)
        if backend == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
            x = t.to(dev)
            dist.all_reduce(x, group=self.group)
            return x.to(t.device)
        x = t.cpu()
        dist.all_reduce(x, group=self.group)
        return x.to(t.device)

    def all_gather_object(self, obj):
        if self.size == 1:
            return [obj]
        import torch.distributed as dist

        out = [None] * self.size
        dist.all_gather_object(out, obj, group=self.group)
        return out


class CudaDeviceApi:
    """Device memory + IPC through the C-ABI (the production backend)."""

    def alloc(self, device: int, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _capi.check(_capi.load().um_device_alloc(device, nbytes, ctypes.byref(p)), "um_device_alloc")
        return int(p.value)

    def free(self, device: int, ptr: int):
        _capi.load().um_device_free(device, ctypes.c_void_p(ptr))

    def ipc_handle(self, ptr: int) -> bytes:
        buf = ctypes.create_string_buffer(_capi.UM_IPC_HANDLE_BYTES)
        _capi.check(_capi.load().um_ipc_get_handle(ctypes.c_void_p(ptr), buf), "um_ipc_get_handle")
        return buf.raw

    def ipc_open(self, handle: bytes, device: int) -> int:
        p = ctypes.c_void_p()
        _capi.check(_capi.load().um_ipc_open_handle(handle, device, ctypes.byref(p)), "um_ipc_open_handle")
        return int(p.value)

    def ipc_close(self, ptr: int):
        _capi.load().um_ipc_close_handle(ctypes.c_void_p(ptr))

    def tensor(self, ptr: int, rows: int, pitch: int, dtype: torch.dtype, device: int, keepalive) -> torch.Tensor:
        return _wrap_device_ptr(ptr, rows, pitch, dtype, device, keepalive)


class _CudaArray:
    """__cuda_array_interface__ shim to view heap memory as a torch tensor."""

    def __init__(self, ptr: int, shape, typestr: str, keepalive):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}
        self._keepalive = keepalive


def _wrap_device_ptr(ptr, rows, pitch, dtype, device, keepalive) -> torch.Tensor:
    if dtype == torch.bfloat16:
        t = torch.as_tensor(_CudaArray(ptr, (rows, pitch), "<i2", keepalive), device=f"cuda:{device}")
        return t.view(torch.bfloat16)
    return torch.as_tensor(_CudaArray(ptr, (rows, pitch), "<f4", keepalive), device=f"cuda:{device}")


class _VmmBlock:
    """One um_sym_alloc block (CUDA VMM physical memory mapped on every peer),
    freed when the last tensor viewing it is gone."""

    def __init__(self, device: int, nbytes: int):
        p = ctypes.c_void_p()
        _capi.check(_capi.load().um_sym_alloc(device, nbytes, ctypes.byref(p)), "um_sym_alloc")
        self.ptr, self.device, self.nbytes = int(p.value), device, nbytes

    def __del__(self):
        try:
            _capi.load().um_sym_free(ctypes.c_void_p(self.ptr))
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


@dataclass
class _Chunk:
    process: int
    index: int
    size: int
    base: int = 0        # local or IPC-mapped base address (0 = unresolved)
    owned: bool = False


class _ChunkOwner:
    """Frees the process's own chunks / closes IPC mappings when the heap dies."""

    def __init__(self, api, device):
        self.api, self.device, self.own, self.mapped = api, device, [], []

    def __del__(self):
        try:
            for p in self.mapped:
                self.api.ipc_close(p)
            for p in self.own:
                self.api.free(self.device, p)
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


class SymmetricHeap:
    """Segment allocator for a Fabric (see module docstring)."""

    def __init__(self, fabric, device_api=None, first_chunk: int = FIRST_CHUNK):
        self.fabric = fabric
        self.world = fabric.world
        self.api = device_api or (CudaDeviceApi() if self.world.size > 1 else None)
        self.first_chunk = first_chunk
        # multi-process bookkeeping, replicated identically on every process
        self._chunks: dict[int, list[_Chunk]] = {q: [] for q in range(self.world.size)}
        self._cursor: dict[int, int] = {q: 0 for q in range(self.world.size)}
        self._unresolved: list = []
        self._owner_box = None
        self._dirty = False   # chunks appended since the last exchange (same on every process)

    # -- allocation -------------------------------------------------------------------

    def allocate(self, owner: int, rows: int, cols: int, dtype: torch.dtype):
        from paper_2510_08874_b200.fabric import SymSegment, pitch_for

        pitch = pitch_for(cols, dtype)
        if self.fabric.placement_only:
            return SymSegment(owner, rows * cols, rows, cols, pitch, dtype, -1, None, 0)
        if self.world.size == 1:
            dev = self.fabric.device_of(owner)
            if getattr(self.fabric, "symmetric", "torch") == "vmm":
                esize = torch.empty((), dtype=dtype).element_size()
                box = _VmmBlock(dev, max(rows, 1) * pitch * esize)
                t = _wrap_device_ptr(box.ptr, max(rows, 1), pitch, dtype, dev, box)[:rows]
                t.zero_()
                seg = SymSegment(owner, rows * cols, rows, cols, pitch, dtype, dev, t, box.ptr)
                seg.vmm = box
                return seg
            t = torch.zeros((max(rows, 1), pitch), dtype=dtype, device=f"cuda:{dev}")[:rows]
            return SymSegment(owner, rows * cols, rows, cols, pitch, dtype, dev, t, t.data_ptr())
        return self._allocate_symmetric(owner, rows, cols, pitch, dtype)

    def place(self, process: int, nbytes: int) -> tuple[int, int]:
        """Deterministic (chunk index, offset) for the next segment of `process`."""
        nbytes = _align(max(nbytes, 1))
        chunks = self._chunks[process]
        if not chunks or self._cursor[process] + nbytes > chunks[-1].size:
            size = self.first_chunk if not chunks else min(MAX_CHUNK, 2 * chunks[-1].size)
            size = max(size, _align(nbytes, 2 << 20))
            chunks.append(_Chunk(process, len(chunks), size, owned=process == self.world.rank))
            self._dirty = True
            self._cursor[process] = 0
            if process == self.world.rank:
                self._materialise(chunks[-1])
        off = self._cursor[process]
        self._cursor[process] += nbytes
        return len(chunks) - 1, off

    def _materialise(self, ch: _Chunk):
        if self._owner_box is None:
            self._owner_box = _ChunkOwner(self.api, self.fabric.devices[0])
        ch.base = self.api.alloc(self.fabric.devices[0], ch.size)
        self._owner_box.own.append(ch.base)

    def _allocate_symmetric(self, owner, rows, cols, pitch, dtype):
        from paper_2510_08874_b200.fabric import SymSegment

        esize = torch.empty((), dtype=dtype).element_size()
        q = self.fabric.process_of(owner)
        idx, off = self.place(q, rows * pitch * esize)
        ch = self._chunks[q][idx]
        if q == self.world.rank:
            dev = self.fabric.devices[0]
            ptr = ch.base + off
            t = self.api.tensor(ptr, max(rows, 1), pitch, dtype, dev, self._owner_box)[:rows]
            t.zero_()
            return SymSegment(owner, rows * cols, rows, cols, pitch, dtype, dev, t, ptr)
        seg = SymSegment(owner, rows * cols, rows, cols, pitch, dtype, -1, None, 0)
        self._unresolved.append((seg, q, idx, off))
        return seg

    # -- multi-process publication ---------------------------------------------------------

    def exchange(self):
        """Collective: publish own chunk handles, map every peer chunk, resolve segments.

        A no-op unless chunks were added since the last call; every process
        replays the same allocation sequence, so all take the same branch."""
        if self.world.size == 1 or not self._dirty:
            return
        self._dirty = False
        mine = {ch.index: self.api.ipc_handle(ch.base) for ch in self._chunks[self.world.rank]
                if ch.owned}
        all_handles = self.world.all_gather_object(mine)
        for q, handles in enumerate(all_handles):
            if q == self.world.rank:
                continue
            for idx, h in handles.items():
                ch = self._chunks[q][idx]
                if not ch.base:
                    ch.base = self.api.ipc_open(h, self.fabric.devices[0])
                    self._owner_box.mapped.append(ch.base)
        still = []
        for seg, q, idx, off in self._unresolved:
            base = self._chunks[q][idx].base
            if base:
                seg.ptr = base + off
                seg.device = self.fabric.devices[0]   # addressable from this process's GPU
            else:
                still.append((seg, q, idx, off))
        self._unresolved = still

    def layout(self):
        """(process -> [(chunk size, base)]) for diagnostics and tests."""
        return {q: [(c.size, c.base) for c in chs] for q, chs in self._chunks.items()}

    # -- stream ordering for API-level one-sided calls ----------------------------------------

    def order_before_remote_access(self, seg, dev: int):
        """Make `dev`'s current stream wait for pending work on the owner's device."""
        if self.world.size > 1 or seg.device < 0 or seg.device == dev:
            return
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(seg.device))
        torch.cuda.current_stream(dev).wait_event(ev)

    def mark_remote_write(self, seg, dev: int):
        """Order the owner's current stream after a write issued from `dev`."""
        if self.world.size > 1 or seg.device < 0 or seg.device == dev:
            return
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        torch.cuda.current_stream(seg.device).wait_event(ev)
