"""Pin the full-size cfg3 / cfg4 answers to the REFERENCE implementation itself.

Run once in the build container (needs /root/reference, read-only; ~10 min):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_large_golden.py [cfg3 cfg4 ...]

The inputs are the repo's seeded counter-hash matrices (configs.py, restated
in numpy here and in CUDA by msq_gen_hash); their sha256 is recorded so the
GPU test (tests/test_gpu_parity.py::test_large_reference_pins) proves it
solved the same bytes.  Each matrix is wrapped in the reference's own
`BinaryMatrix` (grid.py:40-81) and solved by the reference's own `_freq_core`
(squares.py:68-114) -- the function behind `freq_square` -- with a
`snapshots` sink that keeps only the row of the final threshold raise and that
row's `freq` vector (the same data `freq_square_traced`, squares.py:129-139,
would record, without its O(rows*cols) memory).  The location is derived as
in make_golden.py: first row whose found_max_width equals the side, first
column of that row's freq closing a K-run of heights >= K.

Output (committed): tests/golden/large.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("SQUARELAB_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

from squarelab.grid import BinaryMatrix, EdgeKind, generate_edge_case  # noqa: E402
from squarelab.squares import _freq_core  # noqa: E402

from paper_2503_18974_b200 import configs  # noqa: E402


class RaiseSink:
    """`snapshots` stand-in for _freq_core: remembers the last raise row."""

    def __init__(self) -> None:
        self.row = -1
        self.found = 0
        self.freq = None
        self.n = 0

    def append(self, st) -> None:
        if st.found_max_width > self.found:
            self.found = st.found_max_width
            self.row = self.n
            self.freq = st.freq
        self.n += 1


def ref_pin(cells: bytes, rows: int, cols: int) -> dict:
    m = BinaryMatrix(rows, cols, cells)
    sink = RaiseSink()
    t0 = time.time()
    r = _freq_core(m, sink, None)
    dt = time.time() - t0
    side = r.side
    top = left = -1
    if side:
        assert sink.found == side
        run = 0
        for j, f in enumerate(sink.freq):
            run = run + 1 if f >= side else 0
            if run >= side:
                top, left = sink.row - side + 1, j - side + 1
                break
        assert top >= 0
    return {"side": side, "area": r.area, "cells_visited": r.cells_visited, "top": top,
            "left": left, "ref_seconds": round(dt, 1)}


def cfg3_u8() -> np.ndarray:
    c = configs.CONFIGS["cfg3"]
    n, k = c["rows"], c["square"]
    m = np.empty((n, n), np.uint8)
    step = 1024
    for r0 in range(0, n, step):
        m[r0:r0 + step] = configs.hash_u8(c["seed"], configs.thr53(c["p"]), r0, step, n)
    top, left = configs.cfg3_square_pos(c["seed"], n, k)
    m[top:top + k, left:left + k] = 1
    return m


def cfg4_u8_and_sha() -> tuple[np.ndarray, str]:
    c = configs.CONFIGS["cfg4"]
    n = c["rows"]
    m = np.empty((n, n), np.uint8)
    h = hashlib.sha256()
    step = 512
    for r0 in range(0, n, step):
        blk = configs.hash_u8(c["seed"], configs.thr53(c["p"]), r0, step, n)
        m[r0:r0 + step] = blk
        h.update(np.packbits(blk, axis=1, bitorder="little").tobytes())
    return m, h.hexdigest()


def main(which):
    path = os.path.join(HERE, "large.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out["reference"] = REF
    out["note"] = ("side/area/cells_visited from squarelab._freq_core on the same bytes; "
                   "location = implied final-raise cell (make_large_golden.py)")
    if "cfg3" in which:
        m = cfg3_u8()
        n = m.shape[0]
        rec = ref_pin(m.tobytes(), n, n)
        rec["sha256_u8"] = hashlib.sha256(m.tobytes()).hexdigest()
        out["cfg3"] = rec
        print("cfg3", rec, flush=True)
        del m
        for name, kind in (("cfg3_all_zeros", EdgeKind.ALL_ZEROS),
                           ("cfg3_all_ones", EdgeKind.ALL_ONES)):
            e = generate_edge_case(kind, 16384)
            rec = ref_pin(e.cells, e.rows, e.cols)
            out[name] = rec
            print(name, rec, flush=True)
    if "cfg4" in which:
        m, sha = cfg4_u8_and_sha()
        n = m.shape[0]
        cells = m.tobytes()
        del m
        rec = ref_pin(cells, n, n)
        rec["sha256_bits"] = sha
        out["cfg4"] = rec
        print("cfg4", rec, flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3", "cfg4"])
