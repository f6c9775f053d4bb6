"""Maximal all-ones cube on the GPU, the reference's
``squarelab.cubes.max_cube`` (cubes.py:105-125): binary search over sides,
each probe one depth sweep.  A probe is ``msq_cube_probe``: one kernel
thresholds the depth-frequency matrix of every depth at k, one batched
maximal-square solve answers exists_cube_at_depth for all depths at once.
``volume_visited`` counts the voxel reads the reference's probes make.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .squares import _stream_handle, _torch


@dataclass(frozen=True, slots=True)
class CubeResult:
    """cubes.py:50-55."""
    side: int
    volume_visited: int


def _device_volume(v):
    torch = _torch()
    if isinstance(v, torch.Tensor):
        if v.dim() != 3:
            raise ValueError("expected a [depth, rows, cols] volume")
        return v.to(torch.uint8).cuda().contiguous()
    if hasattr(v, "depth") and hasattr(v, "cells"):  # squarelab BinaryVolume (grid.py:88-115)
        a = np.frombuffer(bytes(v.cells), np.uint8).reshape(v.depth, v.rows, v.cols) if v.depth else \
            np.zeros((0, 0, 0), np.uint8)
    else:
        a = np.ascontiguousarray(np.asarray(v, dtype=np.uint8))
        if a.ndim != 3:
            raise ValueError("expected a [depth, rows, cols] volume")
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def max_cube(v) -> CubeResult:
    """Largest k with a k x k x k all-ones cube, and the reference's voxel-read count."""
    torch = _torch()
    vol = _device_volume(v)
    depth, rows, cols = (int(x) for x in vol.shape)
    if depth == 0 or rows == 0 or cols == 0:
        return CubeResult(0, 0)
    scratch = torch.empty_like(vol)
    lib, st = N.load(), _stream_handle()
    layer = rows * cols
    lo, hi, best, visited = 1, min(depth, rows, cols), 0, 0
    while lo <= hi:
        mid = (lo + hi) // 2
        first = ctypes.c_int64(-1)
        N.check(lib.msq_cube_probe(ctypes.c_void_p(vol.data_ptr()), depth, rows, cols, mid,
                                   ctypes.c_void_p(scratch.data_ptr()), ctypes.byref(first), st))
        if first.value >= 0:
            visited += (first.value + 1) * layer
            best, lo = mid, mid + 1
        else:
            visited += depth * layer
            hi = mid - 1
    return CubeResult(best, visited)
