"""GPU-batched verification campaigns.

The reference's parity engine (``squarelab/verify.py``) runs four CPU solvers
on every case, one matrix at a time: ``exhaustive_sweep`` (verify.py:153-181,
every matrix up to max_rows x max_cols, patterns MSB-first) and
``random_campaign`` (verify.py:184-215, a seeded stream of shapes, densities
and matrix seeds).  Here the same case streams go to two independent GPU
solvers in one launch each: the frequency algorithm (``solve_batch``, register
team engine) and the three-way-min DP (``dp_batch``).  Exhaustive shapes are
one launch per shape; the random campaign is one launch for the whole stream
(every case zero-padded to max_dim x max_dim, which changes neither the side
nor the first maximal square; ``cells_visited`` is taken from the true shape).
Optional ``cpu_solvers`` (e.g. the reference's own ``dp_full``) run per case
beside them.  A case is a mismatch when any two solvers disagree on the side
(the reference's rule, verify.py:83-86) or the two GPU solvers disagree on the
location (top, left), which the reference does not report.
"""
from __future__ import annotations

import random
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .grid import BinaryMatrix, GenSpec, generate_matrix
from .squares import SquareResult, dp_batch, solve_batch

ENUMERATION_CAP = 2**20  # verify.py:27

CpuSolver = Callable[[BinaryMatrix], SquareResult]


class EnumerationCapExceededError(ValueError):
    """Exhaustive sweep would enumerate too many matrices (verify.py:43-44)."""


@dataclass(frozen=True, slots=True)
class Mismatch:
    case_id: str
    matrix: BinaryMatrix
    sides: tuple[tuple[str, int], ...]
    locations: tuple[tuple[str, int, int], ...] = ()


@dataclass(frozen=True, slots=True)
class InvariantFailure:
    case_id: str
    row: int
    description: str


@dataclass
class VerifyReport:
    cases_run: int = 0
    mismatches: list[Mismatch] = field(default_factory=list)
    invariant_failures: list[InvariantFailure] = field(default_factory=list)
    elapsed: float = 0.0
    launches: int = 0

    @property
    def clean(self) -> bool:
        return not self.mismatches and not self.invariant_failures


def _check(report: VerifyReport, case_id: str, cells: np.ndarray, freq: SquareResult,
           dp: SquareResult, cpu_solvers: tuple[tuple[str, CpuSolver], ...]) -> None:
    rows, cols = cells.shape
    matrix = None
    results = [("gpu_freq", freq), ("gpu_dp", dp)]
    if cpu_solvers:
        matrix = BinaryMatrix(rows, cols, cells.tobytes())
        results += [(name, fn(matrix)) for name, fn in cpu_solvers]
    sides = tuple((name, r.side) for name, r in results)
    locs = (("gpu_freq", freq.top, freq.left), ("gpu_dp", dp.top, dp.left))
    if len({s for _, s in sides}) > 1 or locs[0][1:] != locs[1][1:]:
        if matrix is None:
            matrix = BinaryMatrix(rows, cols, cells.tobytes())
        report.mismatches.append(Mismatch(case_id, matrix, sides, locs))
    for name, r in results[:2]:  # single-pass solvers (verify.py:40, 88-97)
        if r.cells_visited != rows * cols:
            report.invariant_failures.append(InvariantFailure(
                case_id, -1, f"{name} visited {r.cells_visited} cells, expected {rows * cols}"))
        if r.area != r.side * r.side:
            report.invariant_failures.append(InvariantFailure(
                case_id, -1, f"{name} area {r.area} != side^2 {r.side * r.side}"))
    report.cases_run += 1


def _patterns(rows: int, cols: int) -> np.ndarray:
    """All 2^(rows*cols) matrices of one shape, pattern order and MSB-first
    cells as verify.py:141-150 (_pattern_cells)."""
    bits = rows * cols
    pats = np.arange(2**bits, dtype=np.int64)
    cells = ((pats[:, None] >> np.arange(bits - 1, -1, -1)) & 1).astype(np.uint8)
    return cells.reshape(-1, rows, cols)


def exhaustive_sweep(max_rows: int, max_cols: int,
                     cpu_solvers: tuple[tuple[str, CpuSolver], ...] = ()) -> VerifyReport:
    """Every binary matrix of every shape up to max_rows x max_cols (verify.py:153-181)."""
    total = 0
    for r in range(1, max_rows + 1):
        for c in range(1, max_cols + 1):
            total += 2 ** (r * c)
            if total > ENUMERATION_CAP:
                raise EnumerationCapExceededError(
                    f"sweep up to {max_rows}x{max_cols} exceeds {ENUMERATION_CAP} enumerations")
    report = VerifyReport()
    start = time.perf_counter()
    for r in range(1, max_rows + 1):
        for c in range(1, max_cols + 1):
            stack = _patterns(r, c)
            freq = solve_batch(stack)
            dp = dp_batch(stack)
            report.launches += 2
            for k in range(stack.shape[0]):
                _check(report, f"{r}x{c}#{k}", stack[k], freq[k], dp[k], cpu_solvers)
    report.elapsed = time.perf_counter() - start
    return report


def campaign_specs(count: int, max_dim: int, densities: set[float], seed: int) -> list[GenSpec]:
    """The case stream of verify.py:196-207: density cycle, randint shapes, 64-bit matrix seeds."""
    if count < 1:
        raise ValueError("count must be positive")
    density_cycle = sorted(densities)
    rng = random.Random(seed)
    specs = []
    for index in range(count):
        density = density_cycle[index % len(density_cycle)]
        rows = rng.randint(1, max_dim)
        cols = rng.randint(1, max_dim)
        specs.append(GenSpec(rows, cols, density, rng.getrandbits(64)))
    return specs


def random_campaign(count: int, max_dim: int, densities: set[float], seed: int,
                    cpu_solvers: tuple[tuple[str, CpuSolver], ...] = ()) -> VerifyReport:
    """The seeded case stream of verify.py:184-215 (same shapes, densities and
    matrix seeds for the same arguments), solved in one launch per GPU solver."""
    specs = campaign_specs(count, max_dim, densities, seed)
    shapes, stack = [], np.zeros((count, max_dim, max_dim), np.uint8)
    for index, spec in enumerate(specs):
        m = generate_matrix(spec)
        stack[index, :spec.rows, :spec.cols] = np.frombuffer(m.cells, np.uint8).reshape(spec.rows, spec.cols)
        shapes.append((spec.rows, spec.cols))
    report = VerifyReport()
    start = time.perf_counter()
    freq = solve_batch(stack)
    dp = dp_batch(stack)
    report.launches = 2
    for index, (rows, cols) in enumerate(shapes):
        f, d = freq[index], dp[index]
        # padding is all zeros: side and location stand, visits are the true shape's
        f = SquareResult(f.side, f.area, rows * cols, f.top, f.left)
        d = SquareResult(d.side, d.area, rows * cols, d.top, d.left)
        _check(report, f"random#{index}", stack[index, :rows, :cols], f, d, cpu_solvers)
    report.elapsed = time.perf_counter() - start
    return report


def edge_case_suite() -> VerifyReport:
    """The edge cases of verify.py:218-251 -- constant matrices and the empty
    matrix -- on the GPU: the frequency solver (freq_square) against the DP
    kernel (dp_full), both against the analytically known area, and the
    implied location ((0, 0) for a square, none for side 0)."""
    from .grid import EMPTY_MATRIX, EdgeKind, generate_edge_case
    from .squares import dp_full, freq_square
    cases = [
        ("all_zeros_100", generate_edge_case(EdgeKind.ALL_ZEROS, 100), 0),
        ("all_ones_100", generate_edge_case(EdgeKind.ALL_ONES, 100), 10_000),
        ("single_row_1000", generate_edge_case(EdgeKind.SINGLE_ROW, 1000), 1),
        ("single_col_1000", generate_edge_case(EdgeKind.SINGLE_COL, 1000), 1),
        ("empty", EMPTY_MATRIX, 0),
    ]
    report = VerifyReport()
    start = time.perf_counter()
    for case_id, matrix, expected_area in cases:
        a, b = freq_square(matrix), dp_full(matrix)
        report.launches += 2
        locs = (("gpu_freq", a.top, a.left), ("gpu_dp", b.top, b.left))
        if a.side != b.side or locs[0][1:] != locs[1][1:]:
            report.mismatches.append(
                Mismatch(case_id, matrix, (("gpu_freq", a.side), ("gpu_dp", b.side)), locs))
        for name, result in (("gpu_freq", a), ("gpu_dp", b)):
            if result.area != expected_area:
                report.invariant_failures.append(InvariantFailure(
                    case_id, -1, f"{name} area {result.area}, expected {expected_area}"))
            want_loc = (0, 0) if expected_area else (-1, -1)
            if (result.top, result.left) != want_loc:
                report.invariant_failures.append(InvariantFailure(
                    case_id, -1, f"{name} location {(result.top, result.left)}, expected {want_loc}"))
        report.cases_run += 1
    report.elapsed = time.perf_counter() - start
    return report
