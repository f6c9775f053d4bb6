"""CPU oracle for the histogram maximal rectangle -- TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/squarelab/histogram.py: per-row column
heights (build_histograms, :26-35) and the monotonic-stack sweep with a zero
sentinel (largest_rect_in_histogram, :38-57), the first strictly larger
rectangle kept within a row and across rows (maximal_rectangle, :60-70).
Pinned by tests/golden/histogram.json (tests/golden/make_hist_golden.py).
"""
from __future__ import annotations

import numpy as np


def largest_rect(heights):
    best = (0, 0, 0)
    stack = []
    n = len(heights)
    for idx in range(n + 1):
        bar = heights[idx] if idx < n else 0
        while stack and heights[stack[-1]] >= bar:
            h = heights[stack.pop()]
            left = stack[-1] + 1 if stack else 0
            width = idx - left
            if h * width > best[0]:
                best = (h * width, h, width)
        stack.append(idx)
    return best


def maximal_rectangle(a: np.ndarray):
    a = np.asarray(a, np.uint8)
    best = (0, 0, 0)
    if a.size == 0:
        return best
    h = np.zeros(a.shape[1], np.int64)
    for i in range(a.shape[0]):
        h = np.where(a[i] != 0, h + 1, 0)
        cand = largest_rect(h.tolist())
        if cand[0] > best[0]:
            best = cand
    return best
