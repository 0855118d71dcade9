"""ctypes binding of the C-ABI library (include/unimul_b200.h).

This is the only place Python touches native code.  The library is built
in-tree (``paper_2510_08874_b200/_lib/libunimul_b200.so``) by
``__graft_entry__.build()`` / ``make -C paper_2510_08874_b200/csrc``.  There is
no fallback: if the library is missing, importing anything that needs it
raises immediately.
"""

from __future__ import annotations

import ctypes
import os

from paper_2510_08874_b200.errors import ConfigError, ContractError, OwnershipError

_HERE = os.path.dirname(os.path.abspath(__file__))
# UNIMUL_B200_LIB points at an alternative build of the same library (A/B
# experiments with compile-time variants); the default is the in-tree build.
# UM_GEMM_STALLS=1 needs the profiling build (`make -C paper_2510_08874_b200/csrc
# prof`): the default library has no profiling code in its kernels.
LIB_PATH = os.environ.get("UNIMUL_B200_LIB") or os.path.join(
    _HERE, "_lib", "libunimul_b200_prof.so" if os.environ.get("UM_GEMM_STALLS") == "1" else "libunimul_b200.so")

UM_OK = 0
UM_ECONFIG = 1
UM_EOWNERSHIP = 2
UM_ECONTRACT = 3
UM_EINDEX = 4
UM_EVALUE = 5
UM_ECUDA = 6
UM_ECAPACITY = 7

GEMM_MAX_INLINE_OPS = 40   # UM_GEMM_MAX_INLINE_OPS: ops per K1 launch carried in the kernel parameters
GEMM_MAX_GETS = 64         # UM_GEMM_MAX_GETS: in-kernel pulls per fused launch
UM_BF16 = 0
UM_F32 = 1

UM_BLOCK = 0
UM_BLOCK_CYCLIC = 1

UM_STATIONARY_A = 0
UM_STATIONARY_B = 1
UM_STATIONARY_C = 2

UM_REDUCE_PEER = 0
UM_REDUCE_NCCL = 1
UM_REDUCE_NVLS = 2

UM_FILL_ZERO = 0
UM_FILL_INT = 1
UM_FILL_REAL = 2

UM_OP_FIELDS = 24
UM_IPC_HANDLE_BYTES = 64


class UmMatDesc(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("tile_rows", ctypes.c_int64), ("tile_cols", ctypes.c_int64),
        ("grid_pr", ctypes.c_int64), ("grid_pc", ctypes.c_int64),
        ("mapping", ctypes.c_int32), ("c", ctypes.c_int32),
    ]


class UmView(ctypes.Structure):
    _fields_ = [
        ("base", ctypes.c_void_p),
        ("row_lo", ctypes.c_int64), ("row_hi", ctypes.c_int64),
        ("col_lo", ctypes.c_int64), ("col_hi", ctypes.c_int64),
        ("pitch", ctypes.c_int64),
        ("dtype", ctypes.c_int32), ("device", ctypes.c_int32),
    ]


class UmGemmOp(ctypes.Structure):
    _fields_ = [("a", UmView), ("b", UmView), ("c", UmView),
                ("c_remote", ctypes.c_int32), ("wait_value", ctypes.c_uint32),
                ("wait_flag", ctypes.c_void_p), ("a_get", ctypes.c_int32), ("b_get", ctypes.c_int32),
                ("get_mask", ctypes.c_uint64), ("done_flag", ctypes.c_void_p),
                ("done_piece", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class UmGetDesc(ctypes.Structure):
    _fields_ = [("src", UmView), ("dst", UmView)]


class UmExecCfg(ctypes.Structure):
    _fields_ = [("stationarity", ctypes.c_int32), ("prefetch_depth", ctypes.c_int32),
                ("max_inflight_gemms", ctypes.c_int32), ("max_inflight_accums", ctypes.c_int32),
                ("accumulate_mode", ctypes.c_int32), ("pool_capacity", ctypes.c_int32),
                ("reduce_mode", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class UmExecAction(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("arg", ctypes.c_int32), ("handle", ctypes.c_void_p)]


class UmRankPlan(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("device", ctypes.c_int32), ("ncopies", ctypes.c_int32),
                ("nactions", ctypes.c_int32), ("copies", ctypes.POINTER(UmGetDesc)),
                ("actions", ctypes.POINTER(UmExecAction))]


class UmReduceStep(ctypes.Structure):
    _fields_ = [("dst", UmView), ("srcs", ctypes.POINTER(UmView)), ("nsrc", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("device", ctypes.c_int32), ("reserved", ctypes.c_int32)]


UM_ACT_LAUNCH = 0
UM_ACT_WAIT_COPY = 1
UM_ACT_WAIT_FLAG = 2


# Exported symbols and their C signatures (kept in sync with the header; the
# CPU test suite asserts every header declaration is exported and bound).
_P = ctypes.POINTER
_SIGS = {
    "um_plan": (ctypes.c_int, [_P(UmMatDesc), _P(UmMatDesc), _P(UmMatDesc), ctypes.c_int32, ctypes.c_int32,
                               ctypes.c_int32, _P(ctypes.c_int64), ctypes.c_int64, _P(ctypes.c_int64)]),
    "um_iteration_offset": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P(ctypes.c_int64)]),
    "um_owner_rank": (ctypes.c_int, [_P(UmMatDesc), ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int32, _P(ctypes.c_int32)]),
    "um_most_square_grid": (ctypes.c_int, [ctypes.c_int64, _P(ctypes.c_int64), _P(ctypes.c_int64)]),
    "um_gemm_acc": (ctypes.c_int, [_P(UmView), _P(UmView), _P(UmView), ctypes.c_void_p]),
    "um_gemm_acc_batch": (ctypes.c_int, [_P(UmGemmOp), ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]),
    "um_gemm_acc_fused": (ctypes.c_int, [_P(UmGemmOp), ctypes.c_int32, _P(UmGetDesc), ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_void_p]),
    "um_gemm_prepare": (ctypes.c_int, [_P(UmGemmOp), ctypes.c_int32, _P(UmGetDesc), ctypes.c_int32,
                                       ctypes.c_int32, _P(ctypes.c_void_p)]),
    "um_gemm_launch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "um_gemm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "um_gemm_set_grid_limit": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32]),
    "um_gemm_config": (ctypes.c_int, [_P(ctypes.c_int32)] * 5),
    "um_get": (ctypes.c_int, [_P(UmView), _P(UmView), ctypes.c_void_p]),
    "um_signal": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]),
    "um_signal_supported": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_int32)]),
    "um_wait_geq": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p]),
    "um_accumulate": (ctypes.c_int, [_P(UmView), _P(UmView), ctypes.c_void_p]),
    "um_reduce_replicas": (ctypes.c_int, [_P(UmView), _P(UmView), ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]),
    "um_get_ce": (ctypes.c_int, [_P(UmView), _P(UmView), ctypes.c_void_p]),
    "um_ce_probe": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _P(ctypes.c_int32)]),
    "um_execute": (ctypes.c_int, [_P(UmRankPlan), ctypes.c_int32, _P(UmReduceStep), ctypes.c_int32, _P(UmExecCfg)]),
    "um_sync_all": (ctypes.c_int, []),
    "um_execute_wait": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "um_execute_after": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "um_sym_granularity": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_uint64)]),
    "um_sym_alloc": (ctypes.c_int, [ctypes.c_int32, ctypes.c_uint64, _P(ctypes.c_void_p)]),
    "um_sym_free": (ctypes.c_int, [ctypes.c_void_p]),
    "um_nvls_supported": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_int32)]),
    "um_nvls_team_create": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_int32), _P(ctypes.c_void_p), ctypes.c_uint64,
                                           _P(ctypes.c_void_p), _P(ctypes.c_void_p)]),
    "um_nvls_team_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "um_copy": (ctypes.c_int, [_P(UmView), _P(UmView), ctypes.c_void_p]),
    "um_fill": (ctypes.c_int, [_P(UmView), ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32,
                               ctypes.c_void_p]),
    "um_init": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_int32)]),
    "um_device_alloc": (ctypes.c_int, [ctypes.c_int32, ctypes.c_uint64, _P(ctypes.c_void_p)]),
    "um_device_free": (ctypes.c_int, [ctypes.c_int32, ctypes.c_void_p]),
    "um_ipc_get_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "um_ipc_open_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, _P(ctypes.c_void_p)]),
    "um_ipc_close_handle": (ctypes.c_int, [ctypes.c_void_p]),
    "um_device_count": (ctypes.c_int, [_P(ctypes.c_int32)]),
    "um_sm_count": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_int32)]),
    "um_version": (ctypes.c_char_p, []),
    "um_last_error": (ctypes.c_char_p, []),
}

_lib = None


def load():
    """Load (once) and return the C-ABI library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"unimul_b200 native library not built: {LIB_PATH} is missing. "
            "Run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2510_08874_b200/csrc` (`make ... prof` for the UM_GEMM_STALLS build).")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def last_error() -> str:
    return load().um_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a C status code to the reference's exception classes."""
    if rc == UM_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == UM_ECONFIG:
        raise ConfigError(msg)
    if rc == UM_EOWNERSHIP:
        raise OwnershipError(msg)
    if rc == UM_ECONTRACT:
        raise ContractError(msg)
    if rc == UM_EINDEX:
        raise IndexError(msg)
    if rc == UM_EVALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


def view(base: int, row_lo: int, row_hi: int, col_lo: int, col_hi: int, pitch: int,
         dtype: int, device: int) -> UmView:
    return UmView(base, row_lo, row_hi, col_lo, col_hi, pitch, dtype, device)
