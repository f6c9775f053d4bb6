"""Drop-in maximal-square solver API on the B200 library (mirror of squarelab.squares).

Reference interface (/root/reference/pkg/src/squarelab/squares.py):

* ``SquareResult(side, area, cells_visited)`` (:24-30) -- kept field for field;
  ``top``/``left`` are appended with defaults so reference-style construction
  ``SquareResult(side=..., area=..., cells_visited=...)`` still works.  They
  carry the location the reference implies (the final threshold raise,
  :93-97), -1 when side == 0.
* ``AllocationAudit`` (:48-65) and the auxiliary-space contract of
  ``freq_square`` (peak == cols, tests/test_squares.py:185-189).
* ``freq_square(m, audit=None)`` (:117-126) -- same signature; ``m`` may be a
  BinaryMatrix (ours or the reference's: anything with rows/cols/cells), a
  2-D numpy uint8 array, or a 2-D torch uint8 tensor (host or CUDA).
* ``ValueError`` for cells outside {0, 1} (grid.py:61-62); other library
  errors raise ``MsqError`` (a RuntimeError).
* The other routes of the reference, same signatures and audit contracts, on
  the GPU too: ``dp_full`` / ``dp_rows`` (:142-200, the row-parallel DP kernel
  of csrc/msq_rowdp.cuh), ``brute_force_square`` (:203-249, one thread per
  anchor, the reference's cap and cell-read count), and
  ``freq_square_traced`` / ``FreqState`` (:33-45, :129-139: the result of
  ``freq_square`` plus per-row height snapshots dumped by the DP kernel).

Every call runs the sm_100a kernels in libmsq.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _native as N


ORACLE_CELL_CAP = 10_000  # squares.py:17


class OracleCapExceededError(ValueError):
    """Input too large for the brute-force oracle (squares.py:20-21)."""


@dataclass(frozen=True, slots=True)
class FreqState:
    """Frequency-solver state after a row (squares.py:33-45): the column
    heights, the best side so far, both thresholds (= best + 1) and the
    counter (0 at every row end, squares.py:102-103)."""

    freq: tuple[int, ...]
    found_max_width: int
    check_max_width: int
    check_max_height: int
    counter: int


@dataclass(frozen=True, slots=True)
class SquareResult:
    """Maximal-square answer plus the solver's cell-visit count (squares.py:24-30)."""

    side: int
    area: int
    cells_visited: int
    top: int = -1
    left: int = -1


class AllocationAudit:
    """Auxiliary working-storage tally (squares.py:48-65)."""

    def __init__(self) -> None:
        self.peak_elements = 0
        self._live = 0

    def add(self, count: int) -> None:
        self._live += count
        if self._live > self.peak_elements:
            self.peak_elements = self._live

    def release(self, count: int) -> None:
        self._live -= count


def _torch():
    import torch
    return torch


def _stream_handle():
    torch = _torch()
    if not torch.cuda.is_available():
        raise N.MsqError("no CUDA device: the maximal-square solver has no CPU fallback")
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _to_result(r: N.MsqResult) -> SquareResult:
    return SquareResult(int(r.side), int(r.area), int(r.cells_visited), int(r.top), int(r.left))


def _decode(dev: np.ndarray, rows: int, cols: int) -> SquareResult:
    """Decode one 32-byte msq_devresult block (host copy)."""
    block = N.MsqDevResult.from_buffer_copy(dev.tobytes())
    out = N.MsqResult()
    N.check(N.load().msq_decode(ctypes.byref(block), rows, cols, ctypes.byref(out)))
    return _to_result(out)


class Solver:
    """A planned solve for one shape: workspace and result blocks live on the device.

    ``launch(src)`` only enqueues kernels on the current stream (used by the
    benchmark and by the distributed driver); ``result()`` synchronises and
    decodes.  ``src`` is a CUDA tensor: uint8 [rows, ld] (fmt u8),
    int32/uint32 [rows, ld_words] (fmt bits) or uint8 [batch, rows, cols].
    """

    def __init__(self, fmt: int, rows: int, cols: int, ld: int | None = None, batch: int = 1,
                 nbands: int = 0, deterministic: bool = False, device=None, engine: int = -1,
                 flags: int = 0, test_floor: int = 0, col_chunks: int = 1):
        """``engine``: -1 automatic, 0 band engine, 1 register team engine, 2 sieve engine.
        ``flags`` (N.PLAN_*) and ``test_floor`` are experiment / test switches
        (``test_floor`` presets the shared best side: the caller vouches that
        the answer is at least that)."""
        torch = _torch()
        self.fmt, self.rows, self.cols, self.batch = fmt, rows, cols, batch
        words = (cols + 31) // 32
        self.ld = ld if ld is not None else (cols if fmt == N.FMT_U8 else words)
        self.plan = N.plan(fmt, batch, rows, cols, self.ld, nbands, deterministic, engine)
        self.plan.flags = flags
        self.plan.test_floor = test_floor
        self.plan.col_chunks = col_chunks
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.ws = torch.empty(max(int(self.plan.ws_bytes), 256), dtype=torch.uint8,
                              device=self.device)
        self.res = torch.zeros(batch * 32, dtype=torch.uint8, device=self.device)

    @property
    def nbands(self) -> int:
        return int(self.plan.nbands)

    def launch(self, src) -> None:
        if not src.is_cuda:
            raise ValueError("Solver.launch expects a CUDA tensor")
        self._src = src
        N.check(N.load().msq_launch(ctypes.byref(self.plan), ctypes.c_void_p(src.data_ptr()),
                                    ctypes.c_void_p(self.ws.data_ptr()),
                                    ctypes.c_void_p(self.res.data_ptr()), _stream_handle()))

    def result(self) -> list[SquareResult]:
        host = self.res.cpu().numpy()
        if int(self.plan.engine) == N.ENGINE_SIEVE and (int(host[16]) & 6):
            # the sieve engine could not decide this input (answer outside 56..222 or
            # too many candidates): the same plan runs the band engine, from now on
            self.sieve_retries = getattr(self, "sieve_retries", 0) + 1
            self.plan.engine = N.ENGINE_BAND
            self.launch(self._src)
            host = self.res.cpu().numpy()
        return [_decode(host[32 * k:32 * k + 32], self.rows, self.cols) for k in range(self.batch)]

    def solve(self, src) -> list[SquareResult]:
        self.launch(src)
        return self.result()

    def views(self):
        """Intermediate device buffers (e, b, allones, band keys) as torch tensors."""
        torch = _torch()
        base = self.ws.data_ptr()
        e, b, ao, bk = (ctypes.c_void_p() for _ in range(4))
        N.check(N.load().msq_ws_views(ctypes.byref(self.plan), ctypes.c_void_p(base),
                                      ctypes.byref(e), ctypes.byref(b), ctypes.byref(ao),
                                      ctypes.byref(bk)))
        nb, cp, w = self.nbands, int(self.plan.words) * 32, int(self.plan.words)

        def view(ptr, n, dt, itemsize):
            off = ptr.value - base
            return self.ws[off:off + n * itemsize].view(dt)

        return (view(e, nb * cp, torch.int16, 2).view(nb, cp),
                view(b, nb * cp, torch.int16, 2).view(nb, cp),
                view(ao, nb * w, torch.int32, 4).view(nb, w),
                view(bk, self.batch * nb, torch.int64, 8))


def _host_u8(m):
    """(rows, cols, numpy uint8 array) from a BinaryMatrix-like or array."""
    if hasattr(m, "rows") and hasattr(m, "cols") and hasattr(m, "cells"):
        rows, cols = int(m.rows), int(m.cols)
        a = np.frombuffer(bytes(m.cells), dtype=np.uint8)
        return rows, cols, (a.reshape(rows, cols) if rows else a.reshape(0, 0))
    a = np.ascontiguousarray(np.asarray(m, dtype=np.uint8))
    if a.ndim != 2:
        raise ValueError("expected a 2-D binary matrix")
    return a.shape[0], a.shape[1], a


def freq_square(m, audit: AllocationAudit | None = None) -> SquareResult:
    """Maximal all-ones square via the B200 band kernels (squares.py:117-126).

    Same answer as the reference Algorithm 1 (side, area, cells_visited) plus
    the implied location (top, left).  Host inputs are copied to the device
    inside the library call (msq_solve_u8_host); CUDA tensors are solved in
    place.
    """
    torch = _torch()
    if isinstance(m, torch.Tensor):
        if m.dim() != 2:
            raise ValueError("expected a 2-D binary matrix")
        rows, cols = int(m.shape[0]), int(m.shape[1])
        if audit is not None and rows and cols:
            audit.add(cols)
        if rows == 0 or cols == 0:
            return SquareResult(0, 0, 0)
        t = m if m.dtype == torch.uint8 else m.to(torch.uint8)
        if not t.is_cuda:
            t = t.cuda()
        t = t.contiguous()
        out = N.MsqResult()
        N.check(N.load().msq_solve_u8(ctypes.c_void_p(t.data_ptr()), rows, cols, cols,
                                      ctypes.byref(out), _stream_handle()))
        return _to_result(out)
    rows, cols, a = _host_u8(m)
    if rows < 0 or cols < 0 or (rows == 0 and cols != 0):
        raise ValueError("empty matrix must be 0x0")
    if audit is not None and rows and cols:
        audit.add(cols)  # O(cols) auxiliary contract (squares.py:76-78)
    if rows == 0 or cols == 0:
        return SquareResult(0, 0, 0)
    out = N.MsqResult()
    N.check(N.load().msq_solve_u8_host(a.ctypes.data_as(ctypes.c_void_p), rows, cols, cols,
                                       ctypes.byref(out), _stream_handle()))
    return _to_result(out)


def _device_u8(m):
    """(rows, cols, CUDA uint8 tensor [rows, cols]) for a BinaryMatrix-like,
    numpy array or torch tensor."""
    torch = _torch()
    if isinstance(m, torch.Tensor):
        if m.dim() != 2:
            raise ValueError("expected a 2-D binary matrix")
        rows, cols = int(m.shape[0]), int(m.shape[1])
        t = m if m.dtype == torch.uint8 else m.to(torch.uint8)
        return rows, cols, (t if t.is_cuda else t.cuda()).contiguous()
    rows, cols, a = _host_u8(m)
    if rows < 0 or cols < 0 or (rows == 0 and cols != 0):
        raise ValueError("empty matrix must be 0x0")
    if rows == 0 or cols == 0:
        return rows, cols, None
    _stream_handle()  # raises without a device
    a = np.ascontiguousarray(a)
    return rows, cols, torch.from_numpy(a if a.flags.writeable else a.copy()).cuda()


def _dp_solve(t, rows: int, cols: int, heights=None, rowmax=None) -> SquareResult:
    out = N.MsqResult()
    hp = ctypes.c_void_p(heights.data_ptr()) if heights is not None else None
    rp = ctypes.c_void_p(rowmax.data_ptr()) if rowmax is not None else None
    N.check(N.load().msq_dp_solve(N.FMT_U8, ctypes.c_void_p(t.data_ptr()), rows, cols, cols, hp, rp,
                                  ctypes.byref(out), _stream_handle()))
    return _to_result(out)


def dp_full(m, audit: AllocationAudit | None = None) -> SquareResult:
    """Full-table DP (squares.py:142-171) on the GPU: dp = min(up, left, diag) + 1
    evaluated row-parallel as min(height, row run, diag + 1) (msq_rowdp.cuh).
    Same result as the reference plus the location of the first strict
    improvement; the audit records the reference's rows*cols table."""
    rows, cols, t = _device_u8(m)
    if rows == 0 or cols == 0:
        return SquareResult(0, 0, 0)
    if audit is not None:
        audit.add(rows * cols)  # squares.py:152-153
    return _dp_solve(t, rows, cols)


def dp_rows(m, audit: AllocationAudit | None = None) -> SquareResult:
    """Row-rolling DP (squares.py:174-200): same recurrence and kernel as
    dp_full; the audit records the reference's two rolling rows (2*cols)."""
    rows, cols, t = _device_u8(m)
    if rows == 0 or cols == 0:
        return SquareResult(0, 0, 0)
    if audit is not None:
        audit.add(2 * cols)  # squares.py:181-182
    return _dp_solve(t, rows, cols)


def brute_force_square(m, audit: AllocationAudit | None = None,
                       cap: int = ORACLE_CELL_CAP) -> SquareResult:
    """Direct oracle (squares.py:203-249): every anchor grows its square on the
    GPU, one thread per anchor; cells_visited is the reference's raw read count
    (which exceeds rows*cols).  Raises OracleCapExceededError past `cap`."""
    if hasattr(m, "rows") and hasattr(m, "cols") and not hasattr(m, "dim"):
        rows, cols = int(m.rows), int(m.cols)
    else:
        shp = getattr(m, "shape", None) or np.asarray(m).shape
        rows, cols = (int(shp[0]), int(shp[1])) if len(shp) == 2 else (0, 0)
    if rows * cols > cap:
        raise OracleCapExceededError(
            f"{rows}x{cols} = {rows * cols} cells exceeds oracle cap {cap}")
    if audit is not None:
        audit.add(0)  # no auxiliary storage (squares.py:219-220)
    rows, cols, t = _device_u8(m)
    if rows == 0 or cols == 0:
        return SquareResult(0, 0, 0)
    out = N.MsqResult()
    N.check(N.load().msq_brute_u8(ctypes.c_void_p(t.data_ptr()), rows, cols, cols,
                                  ctypes.byref(out), _stream_handle()))
    return _to_result(out)


def freq_square_traced(m, audit: AllocationAudit | None = None
                       ) -> tuple[SquareResult, list[FreqState]]:
    """freq_square plus a FreqState after each row (squares.py:129-139).

    The result is freq_square's (the band kernels).  The snapshots come from
    the row-DP kernel's per-row height dump: freq = the column heights after
    row i, found_max_width = the largest square ending in rows 0..i (what
    Algorithm 1 has found after row i), thresholds = found + 1,
    counter = 0.  Memory is O(rows * cols), as in the reference.
    """
    torch = _torch()
    rows, cols, t = _device_u8(m)
    if rows == 0 or cols == 0:
        return SquareResult(0, 0, 0), []
    result = freq_square(t, audit)
    heights = torch.empty((rows, cols), dtype=torch.int32, device=t.device)
    rowmax = torch.empty(rows, dtype=torch.int32, device=t.device)
    dp = _dp_solve(t, rows, cols, heights, rowmax)
    found = torch.cummax(rowmax, 0).values.cpu().numpy()
    h = heights.cpu().numpy()
    if dp.side != result.side or int(found[-1]) != result.side:
        raise N.MsqError("traced snapshots disagree with freq_square")
    snaps = [FreqState(tuple(h[i].tolist()), int(found[i]), int(found[i]) + 1,
                       int(found[i]) + 1, 0) for i in range(rows)]
    return result, snaps


def freq_square_bits(words, cols: int) -> SquareResult:
    """Solve a bit-packed matrix (uint32 words, LSB = lowest column).

    ``words``: CUDA int32/uint32 tensor [rows, ld_words] or host numpy uint32.
    """
    torch = _torch()
    out = N.MsqResult()
    if isinstance(words, torch.Tensor) and words.is_cuda:
        rows, ld = int(words.shape[0]), int(words.shape[1])
        if rows == 0 or cols == 0:
            return SquareResult(0, 0, 0)
        w = words.contiguous()
        N.check(N.load().msq_solve_bits(ctypes.c_void_p(w.data_ptr()), rows, cols, ld,
                                        ctypes.byref(out), _stream_handle()))
        return _to_result(out)
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    rows, ld = w.shape
    if rows == 0 or cols == 0:
        return SquareResult(0, 0, 0)
    N.check(N.load().msq_solve_bits_host(w.ctypes.data_as(ctypes.c_void_p), rows, cols, ld,
                                         ctypes.byref(out), _stream_handle()))
    return _to_result(out)


def solve_batch(cells) -> list[SquareResult]:
    """One launch over a stack of equal-shape matrices (uint8 [batch, rows, cols]);
    host arrays go through msq_solve_batch_u8_host (staged H2D inside the call)."""
    torch = _torch()
    if not isinstance(cells, torch.Tensor):
        a = np.ascontiguousarray(np.asarray(cells, dtype=np.uint8))
        if a.ndim != 3:
            raise ValueError("expected [batch, rows, cols]")
        B, R, C = (int(x) for x in a.shape)
        if R == 0 or C == 0:
            return [SquareResult(0, 0, 0) for _ in range(B)]
        out = (N.MsqResult * B)()
        N.check(N.load().msq_solve_batch_u8_host(a.ctypes.data_as(ctypes.c_void_p), B, R, C,
                                                 ctypes.cast(out, ctypes.POINTER(N.MsqResult)),
                                                 _stream_handle()))
        return [_to_result(out[k]) for k in range(B)]
    t = cells
    if t.dim() != 3:
        raise ValueError("expected [batch, rows, cols]")
    B, R, C = (int(x) for x in t.shape)
    if R == 0 or C == 0:
        return [SquareResult(0, 0, 0) for _ in range(B)]
    t = t.to(torch.uint8).cuda().contiguous()
    out = (N.MsqResult * B)()
    N.check(N.load().msq_solve_batch_u8(ctypes.c_void_p(t.data_ptr()), B, R, C,
                                        ctypes.cast(out, ctypes.POINTER(N.MsqResult)),
                                        _stream_handle()))
    return [_to_result(out[k]) for k in range(B)]


def dp_batch(cells) -> list[SquareResult]:
    """The three-way-min DP (dp_full, squares.py:142-171) over a stack of small
    matrices on the GPU (uint8 [batch, rows, cols], cols <= 256): the
    independent second solver of the GPU campaigns in ``verify``."""
    torch = _torch()
    t = cells if isinstance(cells, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(cells, dtype=np.uint8)))
    if t.dim() != 3:
        raise ValueError("expected [batch, rows, cols]")
    B, R, C = (int(x) for x in t.shape)
    if R == 0 or C == 0:
        return [SquareResult(0, 0, 0) for _ in range(B)]
    t = t.to(torch.uint8).cuda().contiguous()
    out = (N.MsqResult * B)()
    N.check(N.load().msq_dp_batch_u8(ctypes.c_void_p(t.data_ptr()), B, R, C,
                                     ctypes.cast(out, ctypes.POINTER(N.MsqResult)),
                                     _stream_handle()))
    return [_to_result(out[k]) for k in range(B)]


Solver_fn = Callable[[object], SquareResult]

# plug-in registry in the shape of squarelab.verify.DEFAULT_SOLVERS (verify.py:32-37):
# pass `solvers=DEFAULT_SOLVERS + GPU_SOLVERS` to the reference's campaigns.
GPU_SOLVERS: tuple[tuple[str, Solver_fn], ...] = (("gpu", freq_square),)
