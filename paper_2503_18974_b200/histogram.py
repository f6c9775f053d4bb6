"""Histogram maximal rectangle on the GPU: the reference's
``squarelab.histogram.maximal_rectangle`` baseline (histogram.py:60-70) --
column heights per row, then one monotonic-stack sweep per row -- as two
kernels (``msq_max_rectangle_u8``).  Same (area, height, width) as the
reference, including which of several largest rectangles is reported.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .squares import _host_u8, _stream_handle, _torch


@dataclass(frozen=True, slots=True)
class RectResult:
    """histogram.py:17-23."""
    area: int
    height: int
    width: int


def maximal_rectangle(m) -> RectResult:
    torch = _torch()
    if isinstance(m, torch.Tensor):
        t = m.to(torch.uint8).cuda().contiguous()
    else:
        _, _, a = _host_u8(m)
        t = torch.from_numpy(np.array(a, dtype=np.uint8, copy=True)).cuda()
    if t.dim() != 2:
        raise ValueError("expected a 2-D binary matrix")
    rows, cols = (int(x) for x in t.shape)
    if rows == 0 or cols == 0:
        return RectResult(0, 0, 0)
    lib = N.load()
    scratch = torch.empty(int(lib.msq_max_rectangle_scratch_bytes(rows, cols)), dtype=torch.uint8,
                          device=t.device)
    a, h, w = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    N.check(lib.msq_max_rectangle_u8(ctypes.c_void_p(t.data_ptr()), rows, cols, cols,
                                     ctypes.c_void_p(scratch.data_ptr()), ctypes.byref(a), ctypes.byref(h),
                                     ctypes.byref(w), _stream_handle()))
    return RectResult(a.value, h.value, w.value)
