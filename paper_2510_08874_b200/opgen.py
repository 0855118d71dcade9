"""Slicing-based op generation (drop-in for unimul.opgen).

`generate` calls the C++ planner (um_plan, csrc/planner.cpp), which restates
opgen.py:106-200 with integer arithmetic and emits the op rows in the
reference's exact order; this module turns them into the same frozen
`LocalMatMulOp` records.  Plans are cached per (matrices, stationarity,
caller): placement is immutable once a DistributedMatrix exists.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np

from paper_2510_08874_b200 import _capi
from paper_2510_08874_b200.errors import ContractError
from paper_2510_08874_b200.tiling import Bounds2D, Range, TileIdx

__all__ = ["Stationarity", "LocalMatMulOp", "restrict_for_replication", "global_to_local", "generate",
           "generate_stationary_a", "generate_stationary_b", "generate_stationary_c", "format_op",
           "plan_rows"]


class Stationarity(Enum):
    STATIONARY_A = "a"
    STATIONARY_B = "b"
    STATIONARY_C = "c"


_UM_STAT = {Stationarity.STATIONARY_A: _capi.UM_STATIONARY_A,
            Stationarity.STATIONARY_B: _capi.UM_STATIONARY_B,
            Stationarity.STATIONARY_C: _capi.UM_STATIONARY_C}


@dataclass(frozen=True)
class LocalMatMulOp:
    """C[m,n] += A[m,k] @ B[k,n] over tile slices (opgen.py:27-54).

    m/k/n bounds are global; *_local are the same bounds in tile coordinates.
    """

    a_tile: TileIdx
    b_tile: TileIdx
    c_tile: TileIdx
    m_bound: Range
    k_bound: Range
    n_bound: Range
    a_local: Bounds2D
    b_local: Bounds2D
    c_local: Bounds2D

    @property
    def flops(self) -> int:
        return 2 * len(self.m_bound) * len(self.k_bound) * len(self.n_bound)

    def stationary_tile(self, stationarity: Stationarity) -> TileIdx:
        return {Stationarity.STATIONARY_A: self.a_tile, Stationarity.STATIONARY_B: self.b_tile}.get(
            stationarity, self.c_tile)


def restrict_for_replication(inner: Range, c: int, replica_idx: int) -> Range:
    """Chunk `replica_idx` of `inner` split c ways; remainder on the last (opgen.py:57-68)."""
    if not 0 <= replica_idx < c:
        raise ValueError(f"replica {replica_idx} out of range for c={c}")
    step = len(inner) // c
    lo = inner.lo + replica_idx * step
    return Range(lo, inner.hi if replica_idx == c - 1 else lo + step)


def global_to_local(global_bounds: Bounds2D, tile_bounds: Bounds2D) -> Bounds2D:
    """Shift global bounds into tile coordinates (opgen.py:71-78)."""
    if not tile_bounds.contains(global_bounds):
        raise ContractError(f"{global_bounds} not contained in tile {tile_bounds}")
    return Bounds2D(global_bounds.rows.shift(-tile_bounds.rows.lo),
                    global_bounds.cols.shift(-tile_bounds.cols.lo))


def plan_rows(a_desc, b_desc, c_desc, nprocs: int, stationarity: Stationarity, caller: int) -> np.ndarray:
    """Raw planner output: an (nops, 24) int64 array in reference order."""
    lib = _capi.load()
    n = ctypes.c_int64(0)
    cap = 256
    while True:
        buf = np.zeros((cap, _capi.UM_OP_FIELDS), dtype=np.int64)
        rc = lib.um_plan(ctypes.byref(a_desc), ctypes.byref(b_desc), ctypes.byref(c_desc), nprocs,
                         _UM_STAT[stationarity], caller,
                         buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap, ctypes.byref(n))
        if rc == _capi.UM_ECAPACITY:
            cap = int(n.value)
            continue
        _capi.check(rc, "um_plan")
        return buf[: n.value]


def _row_to_op(r) -> LocalMatMulOp:
    r = [int(x) for x in r]
    return LocalMatMulOp(
        TileIdx(r[0], r[1]), TileIdx(r[2], r[3]), TileIdx(r[4], r[5]),
        Range(r[6], r[7]), Range(r[8], r[9]), Range(r[10], r[11]),
        Bounds2D(Range(r[12], r[13]), Range(r[14], r[15])),
        Bounds2D(Range(r[16], r[17]), Range(r[18], r[19])),
        Bounds2D(Range(r[20], r[21]), Range(r[22], r[23])),
    )


def generate(stationarity: Stationarity, A, B, C, caller: int) -> list[LocalMatMulOp]:
    """Per-rank op list, identical to the reference's opgen.generate (opgen.py:193-200)."""
    key = (id(A), id(B), id(C), stationarity, caller)
    cache = A.__dict__.setdefault("_plan_cache", {})
    hit = cache.get(key)
    if hit is not None and hit[0] is B and hit[1] is C:
        return list(hit[2])
    if not (A.p == B.p == C.p):
        raise ContractError("A, B and C must span the same number of ranks")
    rows = plan_rows(A.desc(), B.desc(), C.desc(), A.fabric.nprocs, stationarity, caller)
    ops = [_row_to_op(r) for r in rows]
    cache[key] = (B, C, tuple(ops))
    return ops


def generate_stationary_c(A, B, C, caller: int) -> list[LocalMatMulOp]:
    return generate(Stationarity.STATIONARY_C, A, B, C, caller)


def generate_stationary_b(A, B, C, caller: int) -> list[LocalMatMulOp]:
    return generate(Stationarity.STATIONARY_B, A, B, C, caller)


def generate_stationary_a(A, B, C, caller: int) -> list[LocalMatMulOp]:
    return generate(Stationarity.STATIONARY_A, A, B, C, caller)


def format_op(op: LocalMatMulOp) -> str:
    """Debug line, same text as opgen.format_op (opgen.py:203-208)."""
    return (f"a=({op.a_tile.i},{op.a_tile.j}) b=({op.b_tile.i},{op.b_tile.j}) "
            f"c=({op.c_tile.i},{op.c_tile.j}) m={op.m_bound} k={op.k_bound} n={op.n_bound}")
