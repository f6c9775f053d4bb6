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


class CpuSieveBackend(CpuBandBackend):
    """The sieve protocol's per-rank step (msq_rank_sieve) restated on the
    oracle: Algorithm 1 over (halo rows, local rows); decided when the answer is
    in [lo, hi] with hi <= halo_rows (the real engine: 56..222 with a 256-row
    halo), otherwise status 2 and the solver falls back to the band protocol."""
    is_sieve = True

    def __init__(self, local, fmt, cols, row_base, nbands, halo_rows=16, lo=4, hi=16):
        super().__init__(local, fmt, cols, row_base, nbands)
        self.halo_rows, self.lo, self.hi = halo_rows, lo, hi
        self.sieve_low_max = lo - 1
        self._sieve_ks = None
        self.sieve_calls = 0

    def new_halo_buffer(self, rows, like):
        return torch.zeros((rows,) + tuple(like.shape[1:]), dtype=like.dtype)

    def _cells(self, a):
        a = np.ascontiguousarray(a)
        if self.fmt == 0:
            return a.astype(np.uint8)
        w = a.view(np.uint32)
        bits = ((w[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(np.uint8)
        return bits.reshape(w.shape[0], -1)[:, :self.cols]

    def sieve(self, src, halo=None):
        self.sieve_calls += 1
        parts = ([self._cells(halo.numpy())] if halo is not None else []) + [self._cells(self.local)]
        a = np.concatenate(parts, axis=0)
        r = oracle.freq(a)
        base = self.row_base - (a.shape[0] - self.rows)
        if self.lo <= r.side <= self.hi:
            key = oracle.pack_key(r.side, base + r.top + r.side - 1, r.left + r.side - 1)
            self._sieve_ks = torch.tensor([key, 0], dtype=torch.int64)
        else:  # too large: undecided; too small: nothing above lo - 1 in these rows
            self._sieve_ks = torch.tensor([0, 2 if r.side > self.hi else 1], dtype=torch.int64)

    def pass1(self, src):
        self._sieve_ks = None
        super().pass1(src)

    def key_status(self):
        return self._sieve_ks.clone() if self._sieve_ks is not None else super().key_status()
