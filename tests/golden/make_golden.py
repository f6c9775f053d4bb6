"""Generate golden parity fixtures by importing the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `squarelab` from /root/reference/pkg/src (or $SQUARELAB_REF) and
records, for every case, the reference's own answer (`freq_square`,
squares.py:117) and the location the reference implies: the row of the final
threshold raise, read from `freq_square_traced` snapshots (squares.py:129-139)
as the first row whose found_max_width equals the final side, and the first
column of that row's `freq` snapshot closing a K-run of heights >= K
(SURVEY.md section 8 row A2 / P4).  The location is cross-checked against a
brute-force lexicographic search for small inputs.

Outputs (committed): golden.json, exhaustive4x4.npz, random_campaign.npz.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("SQUARELAB_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from squarelab.grid import (  # noqa: E402
    EMPTY_MATRIX, BinaryMatrix, EdgeKind, GenSpec, generate_edge_case, generate_matrix,
    parse_matrix,
)
from squarelab.squares import dp_full, freq_square, freq_square_traced  # noqa: E402
from squarelab.verify import _pattern_cells  # noqa: E402


def ref_answer(m: BinaryMatrix, trace: bool = True):
    """(side, top, left) from the reference's public API."""
    r = freq_square(m)
    side = r.side
    assert dp_full(m).side == side
    if side == 0:
        return 0, -1, -1
    if not trace:
        return side, None, None
    _, snaps = freq_square_traced(m)
    i_star = next(i for i, s in enumerate(snaps) if s.found_max_width == side)
    freq = snaps[i_star].freq
    run = 0
    j_star = None
    for j, f in enumerate(freq):
        run = run + 1 if f >= side else 0
        if run >= side:
            j_star = j
            break
    assert j_star is not None
    return side, i_star - side + 1, j_star - side + 1


def brute_loc(m: BinaryMatrix, side: int):
    """Lexicographically smallest (top, left) of an all-ones side x side square."""
    if side == 0:
        return -1, -1
    for top in range(m.rows - side + 1):
        for left in range(m.cols - side + 1):
            if all(m.cells[(top + a) * m.cols + left + b]
                   for a in range(side) for b in range(side)):
                return top, left
    raise AssertionError("no square of the reported side")


def rows_matrix(rows):
    return BinaryMatrix.from_rows(rows)


KATS = {
    # tests/test_squares.py fixtures (file:line in the reference)
    "all_ones_3x3 (test_squares.py:26)": [[1, 1, 1], [1, 1, 1], [1, 1, 1]],
    "all_zeros_2x2 (test_squares.py:33)": [[0, 0], [0, 0]],
    "single_one (test_squares.py:45)": [[1]],
    "single_zero (test_squares.py:46)": [[0]],
    "single_row (test_squares.py:51)": [[1, 1, 1, 1]],
    "single_col (test_squares.py:52)": [[1], [1], [1]],
    "embedded (test_squares.py:57-62)": [
        [1, 0, 1, 1, 1], [1, 1, 1, 1, 1], [0, 1, 1, 1, 0], [1, 1, 1, 1, 0]],
    "two_candidates (test_squares.py:71-77)": [
        [1, 1, 0, 0, 0], [1, 1, 0, 1, 1], [0, 0, 1, 1, 1], [0, 1, 1, 1, 1], [0, 1, 1, 1, 1]],
    "blocked_corner (test_squares.py:82)": [[0, 1, 1], [1, 1, 1], [1, 1, 1]],
    "lower_triangle (test_squares.py:88)": [[1, 0], [1, 1]],
    "upper_triangle (test_squares.py:90)": [[1, 1], [1, 0]],
    "diagonal (test_squares.py:94)": [[1, 0, 0], [0, 1, 0], [0, 0, 1]],
    "traced_runs (test_squares.py:114-118)": [[1, 1, 0, 1], [1, 1, 1, 1], [0, 1, 1, 1]],
    "misaligned (test_squares.py:135-138)": [[1, 1, 0], [0, 1, 1]],
    "mid_row_then_larger (test_squares.py:144-148)": [
        [1, 1, 0, 1, 1, 1], [1, 1, 0, 1, 1, 1], [0, 0, 0, 1, 1, 1]],
}


def main():
    out = {"reference": REF, "kats": [], "edge": [], "genspec": [], "pins": {}}
    for name, rows in KATS.items():
        m = rows_matrix(rows)
        side, top, left = ref_answer(m)
        assert (top, left) == brute_loc(m, side)
        out["kats"].append({"name": name, "rows": rows, "side": side, "top": top, "left": left})
    # tests/test_cli.py:25
    m = parse_matrix("1101\n1111\n1111\n0110\n")
    side, top, left = ref_answer(m)
    out["kats"].append({"name": "cli_solve (test_cli.py:25)", "rows": m.to_rows(),
                        "side": side, "top": top, "left": left})

    # GenSpec-based fixtures: test_squares.py:100,106,126,164; test_grid.py:152-162
    for spec in [(20, 20, 0.5, 42), (4, 4, 0.5, 7), (13, 7, 0.5, 5), (9, 9, 0.6, 21),
                 (20, 20, 0.7, 3), (100, 100, 0.5, 42), (512, 512, 0.7, 0)]:
        g = GenSpec(*spec)
        m = generate_matrix(g)
        side, top, left = ref_answer(m)
        if m.rows * m.cols <= 10_000:
            assert (top, left) == brute_loc(m, side)
        out["genspec"].append({
            "spec": list(spec), "side": side, "top": top, "left": left, "ones": m.ones(),
            "sha256": hashlib.sha256(m.cells).hexdigest(),
        })
    out["pins"]["genspec_4_4_0.5_7_text"] = "1101\n0110\n1111\n1011\n"  # test_grid.py:154

    # edge cases: verify.py:224-230 and test_acceptance.py:176-189
    edges = [("all_zeros_100", EdgeKind.ALL_ZEROS, 100), ("all_ones_100", EdgeKind.ALL_ONES, 100),
             ("single_row_1000", EdgeKind.SINGLE_ROW, 1000),
             ("single_col_1000", EdgeKind.SINGLE_COL, 1000)]
    for name, kind, n in edges:
        m = generate_edge_case(kind, n)
        side, top, left = ref_answer(m)
        out["edge"].append({"name": name, "kind": kind.value, "n": n, "rows": m.rows,
                            "cols": m.cols, "side": side, "top": top, "left": left})
    r = freq_square(EMPTY_MATRIX)
    out["edge"].append({"name": "empty", "kind": "empty", "n": 0, "rows": 0, "cols": 0,
                        "side": r.side, "top": -1, "left": -1, "cells_visited": r.cells_visited})

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)

    # exhaustive <= 4x4 (verify.py:153-181, 74,954 matrices, MSB-first patterns :141-150)
    ex = {}
    total = 0
    for r_ in range(1, 5):
        for c_ in range(1, 5):
            bits = r_ * c_
            n = 2 ** bits
            sides = np.zeros(n, np.int8)
            tops = np.zeros(n, np.int8)
            lefts = np.zeros(n, np.int8)
            for p in range(n):
                m = BinaryMatrix(r_, c_, _pattern_cells(p, bits))
                s, t, l_ = ref_answer(m)
                sides[p], tops[p], lefts[p] = s, t, l_
            ex[f"side_{r_}x{c_}"] = sides
            ex[f"top_{r_}x{c_}"] = tops
            ex[f"left_{r_}x{c_}"] = lefts
            total += n
    assert total == 74_954
    np.savez_compressed(os.path.join(HERE, "exhaustive4x4.npz"), **ex)

    # random campaign stream (verify.py:184-215): count 10000, max_dim 64,
    # densities {0.3,0.5,0.7,0.9,0.99}, seed 0 -- the acceptance run's parameters
    # (test_acceptance.py:70-77).  Matrices are regenerated from (rows, cols,
    # density, seed) by the repo's own generate_matrix mirror.
    count, max_dim, seed = 10_000, 64, 0
    density_cycle = sorted({0.3, 0.5, 0.7, 0.9, 0.99})
    rng = random.Random(seed)
    rec = {k: np.zeros(count, np.int64) for k in ("rows", "cols", "side", "top", "left")}
    rec["density"] = np.zeros(count, np.float64)
    rec["seed"] = np.zeros(count, np.uint64)
    for index in range(count):
        density = density_cycle[index % len(density_cycle)]
        rows_ = rng.randint(1, max_dim)
        cols_ = rng.randint(1, max_dim)
        mseed = rng.getrandbits(64)
        m = generate_matrix(GenSpec(rows_, cols_, density, mseed))
        s, t, l_ = ref_answer(m, trace=(index % 10 == 0))
        if t is None:  # location via traced API on every 10th; dp-location for the rest
            t, l_ = dp_location(m)
        rec["rows"][index], rec["cols"][index] = rows_, cols_
        rec["density"][index], rec["seed"][index] = density, mseed
        rec["side"][index], rec["top"][index], rec["left"][index] = s, t, l_
    np.savez_compressed(os.path.join(HERE, "random_campaign.npz"), **rec)
    print("golden fixtures written to", HERE)


def dp_location(m: BinaryMatrix):
    """First strict improvement of the dp_full recurrence (squares.py:157-169)."""
    rows, cols, cells = m.rows, m.cols, m.cells
    prev = [0] * cols
    best, loc = 0, (-1, -1)
    for i in range(rows):
        cur = [0] * cols
        for j in range(cols):
            if cells[i * cols + j]:
                v = 1 if i == 0 or j == 0 else min(prev[j], cur[j - 1], prev[j - 1]) + 1
                cur[j] = v
                if v > best:
                    best, loc = v, (i - v + 1, j - v + 1)
        prev = cur
    return loc


if __name__ == "__main__":
    main()
