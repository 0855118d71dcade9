"""Local multiply-accumulate plugin (drop-in for unimul.kernels).

The reference selects a Cython triple loop or a numpy fallback at import
(kernels.py:13-28, _gemmcore.pyx:10-25).  Here there is exactly one backend:
the sm_100a tcgen05 GEMM (K1, csrc/gemm_sm100.cu) behind um_gemm_acc.  No
fallback: the call raises if the native library or a CUDA device is missing,
or if the operands are not CUDA tensors of the tensor-core types.

Contract: `gemm_accumulate(a, b, c)` performs c += a @ b for 2D strided views
(row stride arbitrary, unit column stride) with a, b bfloat16 and c float32
on one device.  It is stream-ordered on the current CUDA stream (torch
semantics), where the reference call was synchronous.
"""

from __future__ import annotations

import ctypes

import torch

from paper_2510_08874_b200 import _capi
from paper_2510_08874_b200.errors import ContractError

BACKEND = "sm100a-tcgen05"

_UM = {torch.bfloat16: _capi.UM_BF16, torch.float32: _capi.UM_F32}


def tensor_view(t: torch.Tensor, device: int | None = None) -> _capi.UmView:
    """um_view of a 2D strided CUDA tensor, expressed against its storage base.

    The base is the storage start (allocation-aligned) and the slice start
    becomes (row_lo, col_lo), which is what the TMA tensor maps want.
    """
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ContractError("gemm operands must be CUDA tensors (no CPU fallback)")
    if t.dim() != 2:
        raise ContractError(f"gemm operands must be 2D, got shape {tuple(t.shape)}")
    if t.dtype not in _UM:
        raise ContractError(f"unsupported dtype {t.dtype}")
    rows, cols = t.shape
    if rows > 1 and t.stride(1) != 1 and cols > 1:
        raise ContractError("gemm operands need unit column stride")
    pitch = t.stride(0) if rows > 1 else max(cols, t.stride(0))
    off = t.storage_offset()
    base = t.untyped_storage().data_ptr()
    if pitch > 0:
        row_lo, col_lo = divmod(off, pitch)
    else:
        row_lo, col_lo = 0, off
    if col_lo + cols > pitch:  # slice wraps a row: re-anchor at its own start
        base, row_lo, col_lo, pitch = t.data_ptr(), 0, 0, max(pitch, cols)
    dev = t.device.index if device is None else device
    return _capi.UmView(base, row_lo, row_lo + rows, col_lo, col_lo + cols, pitch, _UM[t.dtype], dev)


def gemm_accumulate(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor) -> None:
    """c += a @ b on the tensor cores (bf16 inputs, fp32 accumulate)."""
    if a.dim() != 2 or b.dim() != 2 or c.dim() != 2 or a.shape[1] != b.shape[0] \
            or tuple(c.shape) != (a.shape[0], b.shape[1]):
        raise ValueError("inconsistent slice shapes for gemm_accumulate")
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16 or c.dtype != torch.float32:
        raise ContractError("gemm_accumulate expects bfloat16 a/b and float32 c")
    if not (a.device == b.device == c.device):
        raise ContractError("gemm operands must share one device")
    va, vb, vc = tensor_view(a), tensor_view(b), tensor_view(c)
    stream = torch.cuda.current_stream(c.device)
    _capi.check(_capi.load().um_gemm_acc(ctypes.byref(va), ctypes.byref(vb), ctypes.byref(vc),
                                         ctypes.c_void_p(stream.cuda_stream)), "um_gemm_acc")


gemm_accumulate_compiled = gemm_accumulate
