"""CPU stand-in for GpuBackend built on the oracle (TEST INFRASTRUCTURE ONLY).

Lets tests drive RowBandSolver's exchange logic (row split, all-gather of the
per-rank bottom runs, carry composition, key all-reduce) under gloo without a
GPU.  Each method restates the per-rank step the CUDA library performs:
msq_rank_pass1 / msq_rank_summary / msq_compose_carry / msq_rank_fixup.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle


class CpuBandBackend:
    def __init__(self, local: np.ndarray, fmt: int, cols: int, row_base: int, nbands: int):
        self.local = np.ascontiguousarray(local)
        self.fmt, self.cols, self.row_base = fmt, cols, row_base
        self.rows = local.shape[0]
        self.nbands = max(1, min(nbands, self.rows))
        self.launches = 0

    def _band(self, k):
        r0 = self.rows * k // self.nbands
        return r0, self.rows * (k + 1) // self.nbands

    def pass1(self, src):
        words = (self.cols + 31) // 32
        self.e = np.zeros((self.nbands, self.cols), np.uint16)
        self.b = np.zeros((self.nbands, self.cols), np.uint16)
        self.ao = np.zeros((self.nbands, words), np.uint32)
        self.h = np.zeros(self.nbands, np.int64)
        self.key1 = 0
        for k in range(self.nbands):
            r0, r1 = self._band(k)
            e, b, ao, key = oracle.band_pass(self.local, self.fmt, r0, r1, self.cols, 1)
            self.e[k], self.b[k], self.ao[k], self.h[k] = e, b, ao, r1 - r0
            if key:  # band_pass keys use local rows; shift to global rows
                s, bottom, right = oracle.unpack_key(key)
                self.key1 = max(self.key1, oracle.pack_key(s, bottom + self.row_base, right))
        self.launches += 1

    def rank_summary(self):
        out = np.zeros(self.cols, np.int64)
        for j in range(self.cols):
            acc = 0
            for k in range(self.nbands - 1, -1, -1):
                full = (self.ao[k, j >> 5] >> (j & 31)) & 1
                if not full:
                    acc += int(self.b[k, j])
                    break
                acc += int(self.h[k])
            out[j] = acc
        return torch.from_numpy(out.astype(np.int32))

    def new_gather_buffer(self, world: int):
        return torch.zeros((world, self.cols), dtype=torch.int32)

    def compose(self, gathered, rank_rows, rank):
        g = gathered.numpy().astype(np.int64)
        c = np.zeros(self.cols, np.int64)
        for q in range(rank):
            full = g[q] == rank_rows[q]
            c = np.where(full, c + g[q], g[q])
        return torch.from_numpy(c.astype(np.uint32).view(np.int32))

    def fixup(self, base):
        base_np = None if base is None else base.numpy().view(np.uint32)
        t0 = max(1, self.key1 >> 42)
        self.keyfix = 0
        first = 0 if base is not None else 1
        for k in range(first, self.nbands):
            c = oracle.band_carry(k, self.h, self.b, self.ao, self.cols, base_np)
            r0, r1 = self._band(k)
            key = oracle.fixup(c, self.e[k], self.cols, r1 - r0, self.row_base + r0, t0)
            self.keyfix = max(self.keyfix, key)
        self.launches += 1

    def key_status(self):
        return torch.tensor([max(self.key1, self.keyfix), 0], dtype=torch.int64)
