"""CPU oracle for the cube extension -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates /root/reference/pkg/src/squarelab/cubes.py: max_cube (:105-125) as a
binary search over sides with one depth sweep per probe (_probe, :92-102);
depth_freq_update (:58-72) as a per-cell run count along depth; and
exists_cube_at_depth (:75-89) as "some k consecutive columns of one row have
vertical runs >= k in the matrix thresholded at k" -- the same predicate as the
reference's dp_full(binarized).side >= k.  Pinned by tests/golden/cubes.json
(made from the reference by tests/golden/make_cube_golden.py).
"""
from __future__ import annotations

import random

import numpy as np


def _exists(b: np.ndarray, k: int) -> bool:
    rows, cols = b.shape
    if rows < k or cols < k:
        return False
    h = np.zeros(cols, np.int64)
    for i in range(rows):
        h = np.where(b[i], h + 1, 0)
        e = (h >= k).astype(np.int64)
        cs = np.concatenate(([0], np.cumsum(e)))
        if np.any(cs[k:] - cs[:-k] == k):
            return True
    return False


def _probe(vol: np.ndarray, k: int):
    depth, rows, cols = vol.shape
    f = np.zeros((rows, cols), np.int64)
    reads = 0
    for d in range(depth):
        f = np.where(vol[d] != 0, f + 1, 0)
        reads += rows * cols
        if d >= k - 1 and _exists(f >= k, k):
            return True, reads
    return False, reads


def max_cube(vol: np.ndarray):
    """(side, volume_visited) of cubes.py:max_cube for a [depth, rows, cols] 0/1 array."""
    vol = np.asarray(vol, np.uint8)
    if vol.size == 0:
        return 0, 0
    hi = min(vol.shape)
    lo, best, visited = 1, 0, 0
    while lo <= hi:
        mid = (lo + hi) // 2
        found, reads = _probe(vol, mid)
        visited += reads
        if found:
            best, lo = mid, mid + 1
        else:
            hi = mid - 1
    return best, visited


def generate_volume(rows: int, cols: int, density: float, seed: int, depth: int) -> np.ndarray:
    """grid.py:289-298: random.Random(seed).random() per cell, depth-major."""
    rng = random.Random(seed)
    n = depth * rows * cols
    return np.array([1 if rng.random() < density else 0 for _ in range(n)], np.uint8).reshape(depth, rows, cols)
