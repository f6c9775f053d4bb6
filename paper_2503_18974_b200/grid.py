"""Binary-matrix domain types and seeded generators (mirror of squarelab.grid).

Mirrors the parts of /root/reference/pkg/src/squarelab/grid.py that sit on the
hot path:

* ``BinaryMatrix`` -- immutable dense row-major 0/1 grid, same fields and
  validation as grid.py:40-81 (rows == 0 forces cols == 0; cells in {0, 1}).
* ``GenSpec`` / ``generate_matrix`` -- grid.py:148-169 / :274-286.  Cell (i, j)
  is 1 iff the (i*cols + j)-th ``random.Random(seed).random()`` variate is
  < density.  The variates are drawn with numpy's MT19937 loaded with the
  exact state of ``random.Random(seed)`` (both use genrand_res53), so the
  output is bit-identical to the reference and ~100x faster.
* ``generate_edge_case`` -- grid.py:301-313.
* ``parse_matrix`` / ``serialize_matrix`` -- grid.py:172-215 (text format).

Any object with ``rows``, ``cols`` and ``cells`` attributes (including the
reference's own BinaryMatrix) is accepted by the solvers.
"""
from __future__ import annotations

import random
from dataclasses import dataclass
from enum import Enum

import numpy as np


class MatrixParseError(ValueError):
    """Malformed matrix text.  `line` is 1-based, 0 = unknown (grid.py:16-21)."""

    def __init__(self, message: str, line: int = 0):
        super().__init__(message)
        self.line = line


class RaggedRowsError(MatrixParseError):
    """Rows of unequal length (grid.py:24-25)."""


class InvalidCharError(MatrixParseError):
    """A character other than '0', '1', or newline (grid.py:28-29)."""


_TO_BITS = bytes.maketrans(b"01", b"\x00\x01")
_TO_TEXT = bytes.maketrans(b"\x00\x01", b"01")


@dataclass(frozen=True, slots=True)
class BinaryMatrix:
    """Dense row-major grid of 0/1 cells (grid.py:40-81)."""

    rows: int
    cols: int
    cells: bytes

    def __post_init__(self):
        if self.rows < 0 or self.cols < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        if self.rows == 0 and self.cols != 0:
            raise ValueError("empty matrix must be 0x0")
        if len(self.cells) != self.rows * self.cols:
            raise ValueError(f"cell count {len(self.cells)} != {self.rows}x{self.cols}")
        if len(self.cells) and int(np.frombuffer(self.cells, np.uint8).max()) > 1:
            raise ValueError("cells must contain only 0 or 1")

    @classmethod
    def from_rows(cls, rows: list[list[int]]) -> "BinaryMatrix":
        n_rows = len(rows)
        n_cols = len(rows[0]) if rows else 0
        return cls(n_rows, n_cols, bytes(cell for row in rows for cell in row))

    @classmethod
    def from_array(cls, a) -> "BinaryMatrix":
        a = np.ascontiguousarray(np.asarray(a, dtype=np.uint8))
        if a.ndim != 2:
            raise ValueError("expected a 2-D array")
        if a.shape[0] == 0 or a.shape[1] == 0:
            return EMPTY_MATRIX
        return cls(a.shape[0], a.shape[1], a.tobytes())

    def get(self, i: int, j: int) -> int:
        return self.cells[i * self.cols + j]

    def row(self, i: int) -> bytes:
        return self.cells[i * self.cols:(i + 1) * self.cols]

    def to_rows(self) -> list[list[int]]:
        return [list(self.row(i)) for i in range(self.rows)]

    def to_array(self) -> np.ndarray:
        return np.frombuffer(self.cells, np.uint8).reshape(self.rows, self.cols)

    def ones(self) -> int:
        return self.cells.count(1)


EMPTY_MATRIX = BinaryMatrix(0, 0, b"")


class EdgeKind(str, Enum):
    ALL_ZEROS = "all_zeros"
    ALL_ONES = "all_ones"
    SINGLE_ROW = "single_row"
    SINGLE_COL = "single_col"


@dataclass(frozen=True, slots=True)
class GenSpec:
    """Deterministic recipe for a random grid (grid.py:148-169, matrices only)."""

    rows: int
    cols: int
    density: float
    seed: int

    def __post_init__(self):
        if self.rows < 1 or self.cols < 1:
            raise ValueError("rows and cols must be positive")
        if not 0.0 <= self.density <= 1.0:
            raise ValueError(f"density {self.density} outside [0, 1]")
        if not 0 <= self.seed < 2**64:
            raise ValueError("seed must fit in 64 unsigned bits")


def _python_mt(seed: int) -> np.random.RandomState:
    """numpy MT19937 carrying the exact state of random.Random(seed)."""
    st = random.Random(seed).getstate()
    rs = np.random.RandomState()
    rs.set_state(("MT19937", np.array(st[1][:624], dtype=np.uint32), st[1][624]))
    return rs


def generate_array(spec: GenSpec) -> np.ndarray:
    """generate_matrix as a (rows, cols) uint8 array (grid.py:274-286)."""
    u = _python_mt(spec.seed).random_sample(spec.rows * spec.cols)
    return (u < spec.density).astype(np.uint8).reshape(spec.rows, spec.cols)


def generate_matrix(spec: GenSpec) -> BinaryMatrix:
    """Seeded random matrix; identical to squarelab.grid.generate_matrix."""
    return BinaryMatrix(spec.rows, spec.cols, generate_array(spec).tobytes())


def generate_edge_case(kind: EdgeKind, n: int) -> BinaryMatrix:
    """n x n all-zeros/ones, 1 x n row, n x 1 col (grid.py:301-313)."""
    if n < 1:
        raise ValueError("n must be positive")
    if kind is EdgeKind.ALL_ZEROS:
        return BinaryMatrix(n, n, bytes(n * n))
    if kind is EdgeKind.ALL_ONES:
        return BinaryMatrix(n, n, b"\x01" * (n * n))
    if kind is EdgeKind.SINGLE_ROW:
        return BinaryMatrix(1, n, b"\x01" * n)
    if kind is EdgeKind.SINGLE_COL:
        return BinaryMatrix(n, 1, b"\x01" * n)
    raise ValueError(f"unknown edge case kind: {kind!r}")


def _line_to_bits(line: str, lineno: int) -> bytes:
    try:
        raw = line.encode("ascii")
    except UnicodeEncodeError:
        bad = next(ch for ch in line if ord(ch) > 127)
        raise InvalidCharError(f"invalid character {bad!r} at line {lineno}", lineno) from None
    if not set(raw) <= {0x30, 0x31}:
        bad = next(ch for ch in line if ch not in "01")
        raise InvalidCharError(f"invalid character {bad!r} at line {lineno}", lineno)
    return raw.translate(_TO_BITS)


def parse_matrix(text: str) -> BinaryMatrix:
    """'0'/'1' text, one line per row; empty input is 0x0 (grid.py:186-206)."""
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        return EMPTY_MATRIX
    cols = len(lines[0])
    chunks = []
    for i, line in enumerate(lines):
        if len(line) != cols:
            raise RaggedRowsError(f"line {i + 1} has {len(line)} cells, expected {cols}", i + 1)
        chunks.append(_line_to_bits(line, i + 1))
    return BinaryMatrix(len(lines), cols, b"".join(chunks))


def serialize_matrix(m: BinaryMatrix) -> str:
    """Inverse of parse_matrix (grid.py:209-215)."""
    return "".join(m.row(i).translate(_TO_TEXT).decode("ascii") + "\n" for i in range(m.rows))


def pack_bits(a: np.ndarray) -> np.ndarray:
    """(rows, cols) 0/1 uint8 -> (rows, ceil(cols/32)) uint32, LSB = lowest column."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    rows, cols = a.shape
    words = (cols + 31) // 32
    pad = np.zeros((rows, words * 32), np.uint8)
    pad[:, :cols] = a
    packed = np.packbits(pad, axis=1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u4").reshape(rows, words)


def unpack_bits(w: np.ndarray, cols: int) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype="<u4")
    rows = w.shape[0]
    bits = np.unpackbits(w.view(np.uint8).reshape(rows, -1), axis=1, bitorder="little")
    return np.ascontiguousarray(bits[:, :cols])
