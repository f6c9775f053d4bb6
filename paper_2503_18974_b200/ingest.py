"""Text ingest on the GPU: the reference's matrix text format
(grid.py:172-206 ``parse_matrix``: one '0'/'1' line per row, trailing newline
optional, frozen by SPEC.md) parsed by ``msq_parse_text`` straight into solver
input -- bit-packed words (or u8 cells) in device memory -- so the CLI route
``solve`` (cli.py:144-148) of a large file never builds a Python
``BinaryMatrix``.  Errors are the reference's: the kernel reports the first
malformed line and the same exception type and message are raised for it.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .grid import EMPTY_MATRIX, RaggedRowsError, _line_to_bits, parse_matrix
from .squares import AllocationAudit, SquareResult, _stream_handle, _torch, freq_square_bits


def _raise_for_line(text: bytes, lineno: int):
    """The exception the reference's sequential parse raises at line `lineno`."""
    lines = text.decode("utf-8", errors="surrogateescape").split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    cols = len(lines[0])
    line = lines[lineno - 1] if lineno - 1 < len(lines) else ""
    if len(line) != cols:
        raise RaggedRowsError(f"line {lineno} has {len(line)} cells, expected {cols}", lineno)
    _line_to_bits(line, lineno)  # raises InvalidCharError
    raise AssertionError(f"line {lineno} flagged by the ingest kernel but valid")


def parse_matrix_device(text, fmt: str = "bits", device=None):
    """Parse matrix text on the GPU.  Returns (tensor, rows, cols): int32
    [rows, ceil(cols/32)] LSB-first words for fmt="bits", uint8 [rows, cols]
    for fmt="u8"; (None, 0, 0) for the empty text."""
    torch = _torch()
    raw = text.encode("utf-8", errors="surrogateescape") if isinstance(text, str) else bytes(text)
    if not raw:
        return None, 0, 0
    nl = raw.find(b"\n")
    cols = nl if nl >= 0 else len(raw)
    if cols == 0:  # lines of no cells: nothing for the GPU, the reference's rules decide
        m = parse_matrix(raw.decode("utf-8", errors="surrogateescape"))
        return None, m.rows, m.cols
    rows = (len(raw) + cols) // (cols + 1)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    pad = (-len(raw)) % 16
    host = torch.frombuffer(bytearray(raw + b"\n" * pad), dtype=torch.uint8)
    d_text = host.to(dev)
    if fmt == "bits":
        words = (cols + 31) // 32
        out = torch.empty((rows, words), dtype=torch.int32, device=dev)
        f, ld = N.FMT_BITS, words
    elif fmt == "u8":
        out = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
        f, ld = N.FMT_U8, cols
    else:
        raise ValueError("fmt must be 'bits' or 'u8'")
    bad = ctypes.c_int64(0)
    rc = N.load().msq_parse_text(ctypes.c_void_p(d_text.data_ptr()), len(raw), rows, cols, f,
                                 ctypes.c_void_p(out.data_ptr()), ld, ctypes.byref(bad),
                                 _stream_handle())
    if rc == N.MSQ_EVALUE:
        _raise_for_line(raw, int(bad.value))
    N.check(rc)
    return out, rows, cols


def freq_square_text(text, audit: AllocationAudit | None = None) -> SquareResult:
    """``freq_square(parse_matrix(text))`` with both steps on the GPU."""
    words, rows, cols = parse_matrix_device(text, "bits")
    if words is None:
        return SquareResult(0, 0, rows * cols)
    if audit is not None:
        audit.add(cols)
    return freq_square_bits(words, cols)
