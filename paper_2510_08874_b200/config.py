"""Execution knobs and per-rank records of the engine (runtime.py:26-86).

Split out of `runtime` so the schedule, engine and replica modules share them
without import cycles; `runtime` re-exports every name (drop-in API).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from paper_2510_08874_b200.fabric import AccumulateMode
from paper_2510_08874_b200.opgen import LocalMatMulOp, Stationarity
from paper_2510_08874_b200.tiling import TileIdx

__all__ = ["ExecConfig", "BufferPool", "RunStats"]


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
      fine_waits         an operand pulled into one band waits chunk by chunk
                         (A: its tile's rows; B: each k-block's rows) instead of
                         for the whole band, so the first tiles start as soon
                         as their first rows land.
      share_sms          ranks co-resident on one GPU each get an equal share of
                         its SMs for their K1 launches, which then run side by
                         side (off: measured 10-25 % slower than whole-GPU
                         launches one after the other, e.g. cfg3 p=8 1118 vs
                         1415 TFLOP/s).
      chain_order        issue ops that write the same C region back to back
                         (K1 accumulates such a k-chain in TMEM and reduces
                         into C once per tile).
      get_engine         "kernel": remote slices are pulled by get warps INSIDE
                         the K1 launch (um_gemm_acc_fused) and each op starts
                         when its pulls have landed — one launch per rank (up
                         to UM_GEMM_MAX_INLINE_OPS ops / UM_GEMM_MAX_GETS pulls)
                         with the gets overlapping the GEMMs of earlier ops;
                         "copy": copy-engine pulls on a get stream, the host
                         splits K1 launches at every pull not yet waited on;
                         "auto": pulls from the caller's own GPU in-kernel,
                         pulls from other GPUs on the copy engines (um_get_ce,
                         no SMs) followed by an arrival flag (um_signal) that
                         the K1 producer waits on inside the same launch --
                         where um_ce_probe shows the driver runs such a copy
                         without SMs, else in-kernel; the launch leaves two
                         CTA pairs' SMs free so an SM-run copy still
                         progresses.  "ce": every pull that way (a protocol
                         test mode: with several ranks co-resident on ONE
                         GPU, full-size same-device pulls deadlocked the
                         spinning K1s on the test box).  The default stays
                         "kernel" (deadlock-free by construction: every pull
                         is done by warps of the same launch) until the
                         cross-GPU copy-engine path is validated on a
                         multi-GPU box.
      reduce_mode        K4 for replicated C: "peer" (P2P loads, reference
                         summation order), "nvls" (multimem.ld_reduce through a
                         multicast team: needs Fabric(symmetric="vmm") and the
                         replicas on distinct multicast-capable GPUs), "nccl"
                         (ncclReduce per tile; barrier form), "auto" (nvls when
                         capable, else peer).
      graph_replay       a small single-process direct multiply (<= 2^36 flops)
                         repeated on the same (A, B, C, config) is captured into
                         a CUDA graph on its third call and replayed from then
                         on (graphs.CapturedMultiply): one cudaGraphLaunch
                         instead of the per-rank host issue that dominates such
                         multiplies.  Same kernels and plans; a replicated C is
                         reduced in the barrier form inside the graph.
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
    fine_waits: bool = True
    share_sms: bool = False
    reduce_panels: int = 4
    k_split: int = 0
    reduce_mode: str = "auto"
    graph_replay: bool = True

    def __post_init__(self):
        if self.prefetch_depth < 1 or self.max_inflight_gemms < 1 or self.max_inflight_accums < 1:
            raise ValueError("ExecConfig counts must be >= 1")
        if self.pool_capacity is not None and self.pool_capacity < 3:
            raise ValueError("pool_capacity must cover at least one op (3 buffers)")
        if self.staging not in ("slice", "tile"):
            raise ValueError(f"unknown staging mode {self.staging!r}")
        if self.same_device_gets not in ("copy", "direct"):
            raise ValueError(f"unknown same_device_gets {self.same_device_gets!r}")
        if self.get_engine not in ("kernel", "copy", "auto", "ce"):
            raise ValueError(f"unknown get_engine {self.get_engine!r}")
        if self.k_split < 0 or self.mn_split < 0:
            raise ValueError("k_split / mn_split must be >= 0")
        if self.reduce_panels < 1:
            raise ValueError("reduce_panels must be >= 1")
        if self.reduce_mode not in ("auto", "peer", "nccl", "nvls"):
            raise ValueError(f"unknown reduce_mode {self.reduce_mode!r}")
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
    # the order in which the device actually starts the ops (first (sub-)op of
    # each, as the K1 tile scheduler hands them out): k-chains grouped, pulls
    # in this order.  executed_ops / a_requests / b_requests keep the
    # reference's execution order (runtime.py:213-236).
    device_order: list[LocalMatMulOp] = field(default_factory=list)
