"""NVTX ranges around the host phases of a multiply (plan, issue, K4).

Every range is named "um:<phase>" so an ncu / Nsight capture can be filtered
to one phase (`ncu --nvtx --nvtx-include "um:execute_multiply/"`).  A range
costs ~1 us of host time and nothing on the device.
"""

from __future__ import annotations

import functools

import torch


def nvtx(name: str):
    """Decorator: run the function inside the NVTX range `name`."""

    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()

        return wrapper

    return deco
