"""Row-band sharding of one matrix across GPUs (one process per GPU).

Rank r owns rows [rows*r/N, rows*(r+1)/N).  Per solve:

1. lower-bound seed over the local rows, all-reduce(max) of the seeds' best
   side (8 bytes), band passes from it (msq_rank_seed / msq_rank_band_pass;
   one rank: msq_rank_pass1) -> per-band column summaries + a local key;
2. per column, the bottom run of the local slice (msq_rank_summary, uint32,
   == local rows when the column is all ones);
3. ONE all-gather of those summaries (NCCL over NVLink; cols*4 bytes/rank);
4. carry-in heights for the slice top from the ranks above
   (msq_compose_carry: P5 fold);
5. data-free band-boundary fix-ups, including the slice's top boundary
   (msq_rank_fixup);
6. all-reduce(max) of the 64-bit (side, -bottom, -right) key.

The orchestration is independent of where the per-rank steps run: ``GpuBackend``
calls the C ABI; tests substitute a CPU backend built on the oracle to check
the exchange logic under gloo without a GPU.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .squares import SquareResult

KEY_DIM_BITS = 21
KEY_DIM_MASK = (1 << KEY_DIM_BITS) - 1
SIEVE_LOW_MAX = 62  # status 1 (no block square of side 7 on some rank) is harmless above this side
SIEVE_HALO = 256  # rows a rank borrows from the rank above (msq_sieve.cuh SV_HALO_ROWS)


def slice_rows(rows: int, world: int, rank: int) -> tuple[int, int]:
    r0 = rows * rank // world
    return r0, rows * (rank + 1) // world - r0


def decode_key(key: int, status: int, rows: int, cols: int) -> SquareResult:
    if status & 1:  # 1 (device status) / 3 (reduced [key, status]): an invalid cell
        raise ValueError("cells must contain only 0 or 1")
    if key == 0:
        return SquareResult(0, 0, rows * cols)
    side = key >> (2 * KEY_DIM_BITS)
    bottom = KEY_DIM_MASK - ((key >> KEY_DIM_BITS) & KEY_DIM_MASK)
    right = KEY_DIM_MASK - (key & KEY_DIM_MASK)
    return SquareResult(side, side * side, rows * cols, bottom - side + 1, right - side + 1)


class GpuBackend:
    """Per-rank steps on the local GPU through libmsq."""

    def __init__(self, fmt: int, local_rows: int, cols: int, row_base: int, ld: int | None = None,
                 nbands: int = 0, device=None, engine: int = -1):
        import torch
        self.torch = torch
        words = (cols + 31) // 32
        ld = ld if ld is not None else (cols if fmt == N.FMT_U8 else words)
        self.plan = N.plan(fmt, 1, local_rows, cols, ld, nbands, engine=engine)
        self.sieve_min_rows = 4096 if engine == -1 else 0  # msq_plan_make's automatic choice
        self.plan.row_base = row_base
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ws = torch.empty(max(int(self.plan.ws_bytes), 256), dtype=torch.uint8, device=dev)
        self.res = torch.zeros(32, dtype=torch.uint8, device=dev)
        self.summary = torch.empty(cols, dtype=torch.int32, device=dev)
        self.base = torch.empty(cols, dtype=torch.int32, device=dev)
        self.ks = torch.zeros(2, dtype=torch.int64, device=dev)
        self.cols = cols
        self.lib = N.load()
        self.launches = 0

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def pass1(self, src):
        N.check(self.lib.msq_rank_pass1(ctypes.byref(self.plan), ctypes.c_void_p(src.data_ptr()),
                                        ctypes.c_void_p(self.ws.data_ptr()),
                                        ctypes.c_void_p(self.res.data_ptr()), self._stream()))
        self.launches += int(self.lib.msq_last_launch_count())  # lower-bound seed + band pass

    def seed(self, src):
        """Lower-bound seed over the local rows (resets the result block)."""
        N.check(self.lib.msq_rank_seed(ctypes.byref(self.plan), ctypes.c_void_p(src.data_ptr()),
                                       ctypes.c_void_p(self.res.data_ptr()), self._stream()))
        self.launches += int(self.lib.msq_last_launch_count())

    def best_side(self):
        """The device's shared best side (int32 view into the result block, in place)."""
        return self.res.view(self.torch.int32)[5:6]

    def band_pass(self, src):
        N.check(self.lib.msq_rank_band_pass(ctypes.byref(self.plan), ctypes.c_void_p(src.data_ptr()),
                                            ctypes.c_void_p(self.ws.data_ptr()),
                                            ctypes.c_void_p(self.res.data_ptr()), self._stream()))
        self.launches += int(self.lib.msq_last_launch_count())

    def rank_summary(self):
        N.check(self.lib.msq_rank_summary(ctypes.byref(self.plan),
                                          ctypes.c_void_p(self.ws.data_ptr()),
                                          ctypes.c_void_p(self.summary.data_ptr()), self._stream()))
        self.launches += 1
        return self.summary

    def new_gather_buffer(self, world: int):
        return self.torch.empty((world, self.cols), dtype=self.torch.int32, device=self.summary.device)

    def compose(self, gathered, rank_rows: list[int], rank: int):
        rr = (ctypes.c_int64 * len(rank_rows))(*rank_rows)
        N.check(self.lib.msq_compose_carry(ctypes.c_void_p(gathered.data_ptr()), rr,
                                           len(rank_rows), rank, self.cols,
                                           ctypes.c_void_p(self.base.data_ptr()), self._stream()))
        self.launches += 1
        return self.base

    def fixup(self, base):
        ptr = ctypes.c_void_p(base.data_ptr()) if base is not None else None
        N.check(self.lib.msq_rank_fixup(ctypes.byref(self.plan), ctypes.c_void_p(self.ws.data_ptr()),
                                        ptr, ctypes.c_void_p(self.res.data_ptr()), self._stream()))
        nb = int(self.plan.nbands) - (0 if base is not None else 1)
        self.launches += 2 if nb > 0 else 0  # carry scan + fix-up

    # ---- sieve engine (plan.engine == 2): no band summaries, a halo of rows instead
    @property
    def is_sieve(self) -> bool:
        return int(self.plan.engine) == N.ENGINE_SIEVE

    def new_halo_buffer(self, rows: int, like):
        return self.torch.empty((rows,) + tuple(like.shape[1:]), dtype=like.dtype, device=like.device)

    def _sieve_call(self, fn, src, halo):
        hp = ctypes.c_void_p(halo.data_ptr()) if halo is not None else None
        hr = int(halo.shape[0]) if halo is not None else 0
        hl = int(halo.stride(0)) if halo is not None else 0
        N.check(fn(ctypes.byref(self.plan), ctypes.c_void_p(src.data_ptr()), hp, hr, hl,
                   ctypes.c_void_p(self.ws.data_ptr()), ctypes.c_void_p(self.res.data_ptr()),
                   self._stream()))
        self.launches += int(self.lib.msq_last_launch_count())

    def sieve(self, src, halo=None):
        """Streaming pass + band-top rows + exact candidate windows over (halo, src)."""
        self._sieve_call(self.lib.msq_rank_sieve, src, halo)

    def sieve_pass(self, src, halo=None):
        self._sieve_call(self.lib.msq_rank_sieve_pass, src, halo)

    def sieve_finish(self, src, halo=None):
        self._sieve_call(self.lib.msq_rank_sieve_finish, src, halo)

    def key_status(self):
        """int64 tensor [key, status] for the all-reduce (keys < 2^63), written
        by one library kernel (msq_rank_key_status) into a persistent buffer."""
        N.check(self.lib.msq_rank_key_status(ctypes.c_void_p(self.res.data_ptr()),
                                             ctypes.c_void_p(self.ks.data_ptr()), self._stream()))
        self.launches += 1
        return self.ks


def _all_gather(out, t, group=None):
    """all-gather of one tensor per rank into out[world, ...] (NCCL fast path;
    list form for backends without the base collective)."""
    import torch.distributed as dist
    try:
        dist.all_gather_into_tensor(out, t, group=group)
    except (RuntimeError, NotImplementedError):
        parts = list(out.unbind(0))
        dist.all_gather(parts, t, group=group)


class RowBandSolver:
    """Solve one (rows x cols) matrix sharded by rows over a process group.

    Backends whose plan is a sieve plan (``is_sieve``) try the sieve first: each
    rank borrows the last SIEVE_HALO (256) rows of the rank above (one send/recv, no
    dependence on any kernel) and solves (halo, local rows) alone; the ranks
    all-reduce(max) their [key, status].  When any rank's sieve could not
    decide, all ranks run the band protocol below, now and for later solves."""

    def __init__(self, rows: int, cols: int, rank: int, world: int, backend, group=None):
        self.rows, self.cols, self.rank, self.world = rows, cols, rank, world
        self.row0, self.local_rows = slice_rows(rows, world, rank)
        self.rank_rows = [slice_rows(rows, world, q)[1] for q in range(world)]
        self.backend = backend
        self.group = group
        self.gathered = backend.new_gather_buffer(world) if world > 1 else None
        self._ks = None
        self._src = None
        self._halo = None
        self.halo_rows = int(getattr(backend, "halo_rows", SIEVE_HALO))
        # a rank that finds no 7x7 block square has nothing above 8 * 6 + 14 cells
        self.sieve_low_max = int(getattr(backend, "sieve_low_max", SIEVE_LOW_MAX))
        # every rank must take the same protocol: the automatic plan picks the sieve from
        # 4096 local rows on, so slices on both sides of that line all take the bands
        self.sieve = (bool(getattr(backend, "is_sieve", False)) and min(self.rank_rows) >= self.halo_rows and
                      min(self.rank_rows) >= int(getattr(backend, "sieve_min_rows", 0)))
        self.sieve_retries = 0

    def _exchange_halo(self, src):
        """Rank r receives the last halo_rows rows of rank r-1."""
        import torch.distributed as dist
        be = self.backend
        if self.rank > 0 and self._halo is None:
            self._halo = be.new_halo_buffer(self.halo_rows, src)
        ops = []
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, src[-self.halo_rows:], self.rank + 1, group=self.group))
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, self._halo, self.rank - 1, group=self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return self._halo if self.rank > 0 else None

    def launch(self, src) -> None:
        import torch.distributed as dist
        be = self.backend
        self._src = src
        if self.sieve:
            halo = self._exchange_halo(src) if self.world > 1 else None
            be.sieve(src, halo)
            if self.world > 1:
                ks = be.key_status()
                dist.all_reduce(ks, op=dist.ReduceOp.MAX, group=self.group)
                self._ks = ks
            else:
                self._ks = None
            return
        if self.world > 1 and hasattr(be, "seed"):
            # pool the ranks' lower bounds (8 bytes) before the band passes
            be.seed(src)
            dist.all_reduce(be.best_side(), op=dist.ReduceOp.MAX, group=self.group)
            be.band_pass(src)
        else:
            be.pass1(src)
        base = None
        if self.world > 1:
            summary = be.rank_summary()
            _all_gather(self.gathered, summary, self.group)
            if self.rank > 0:
                base = be.compose(self.gathered, self.rank_rows, self.rank)
        be.fixup(base)
        if self.world > 1:
            ks = be.key_status()
            dist.all_reduce(ks, op=dist.ReduceOp.MAX, group=self.group)
            self._ks = ks
        else:
            self._ks = None  # one rank: decode the device result block directly

    def result(self) -> SquareResult:
        ks = (self._ks if self._ks is not None else self.backend.key_status()).cpu().numpy().astype(np.int64)
        undecided = int(ks[1]) == 2 or (int(ks[1]) == 1 and (int(ks[0]) >> (2 * KEY_DIM_BITS)) <= self.sieve_low_max)
        if self.sieve and undecided:
            # some rank's sieve could not decide (every rank sees the same reduced
            # status): the band protocol, for this solve and the following ones
            self.sieve = False
            self.sieve_retries += 1
            self.launch(self._src)
            return self.result()
        return decode_key(int(ks[0]), int(ks[1]) if int(ks[1]) == 3 else 0, self.rows, self.cols)

    def solve(self, src) -> SquareResult:
        self.launch(src)
        return self.result()
