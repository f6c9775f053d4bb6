"""The reference's other routes on the GPU (squares.py:129-249) and the
AllocationAudit contract (tests/test_squares.py:185-196): dp_full, dp_rows,
brute_force_square, freq_square_traced against vectors made by the reference
itself (tests/golden/baselines.json, make_baseline_golden.py), and the DP
kernel against the oracle at sizes / shapes the band engine does not take."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2503_18974_b200 import (
    AllocationAudit, BinaryMatrix, GenSpec, OracleCapExceededError, brute_force_square, dp_full,
    dp_rows, freq_square, freq_square_traced, generate_matrix,
)

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def torch():
    import torch as t
    from paper_2503_18974_b200 import build
    build.build()
    return t


def _cases():
    with open(os.path.join(GOLDEN, "baselines.json")) as f:
        for rec in json.load(f):
            if "cells" in rec:
                m = BinaryMatrix(rec["rows"], rec["cols"], bytes.fromhex(rec["cells"]))
            else:
                m = generate_matrix(GenSpec(*rec["spec"]))
            yield rec, m


def test_dp_brute_traced_vs_reference(torch):
    n = 0
    for rec, m in _cases():
        want = oracle.freq(np.frombuffer(m.cells, np.uint8).reshape(m.rows, m.cols))
        for fn in (dp_full, dp_rows):
            r = fn(m)
            assert r.side == rec[fn.__name__], (rec["name"], fn.__name__)
            assert (r.side, r.area, r.cells_visited, r.top, r.left) == (
                want.side, want.area, want.cells_visited, want.top, want.left), rec["name"]
        if "brute_side" in rec:
            b = brute_force_square(m)
            assert (b.side, b.cells_visited) == (rec["brute_side"], rec["brute_visited"]), rec["name"]
            assert (b.top, b.left) == (want.top, want.left), rec["name"]
        for fn_name, peak in rec["audit_peak"].items():
            a = AllocationAudit()
            {"freq_square": freq_square, "dp_full": dp_full, "dp_rows": dp_rows,
             "brute_force_square": brute_force_square}[fn_name](m, a)
            assert a.peak_elements == peak, (rec["name"], fn_name)
        if "trace_freq" in rec:
            res, snaps = freq_square_traced(m)
            assert res.side == rec["side"]
            assert [list(s.freq) for s in snaps] == rec["trace_freq"], rec["name"]
            assert [s.found_max_width for s in snaps] == rec["trace_found"], rec["name"]
            assert all(s.counter == 0 and s.check_max_width == s.found_max_width + 1 ==
                       s.check_max_height for s in snaps)
        n += 1
    assert n == 324


def test_audit_contract(torch):
    """tests/test_squares.py:185-196: freq peak == cols, dp_rows == 2*cols."""
    m = generate_matrix(GenSpec(30, 40, 0.8, 3))
    for fn, want in ((freq_square, 40), (dp_rows, 80), (dp_full, 1200), (brute_force_square, 0)):
        a = AllocationAudit()
        fn(m, a)
        assert a.peak_elements == want, fn.__name__


def test_brute_cap(torch):
    with pytest.raises(OracleCapExceededError):
        brute_force_square(generate_matrix(GenSpec(101, 100, 0.5, 1)))
    assert brute_force_square(generate_matrix(GenSpec(101, 100, 0.5, 1)), cap=20_000).side >= 1


@pytest.mark.parametrize("shape", [(300, 70000), (5, 131072), (2000, 333), (1, 17), (4097, 1),
                                   (700, 4112)])
def test_dp_kernel_shapes(torch, shape):
    """Wide (> 65536 columns), thin, ragged and unaligned shapes: dp vs the oracle."""
    rows, cols = shape
    rng = np.random.default_rng(rows * 7 + cols)
    a = (rng.random((rows, cols)) < 0.93).astype(np.uint8)
    if rows > 60 and cols > 60:
        a[rows // 3:rows // 3 + 50, cols // 2:cols // 2 + 50] = 1
    want = oracle.freq(a)
    r = dp_full(torch.from_numpy(a).cuda())
    assert (r.side, r.area, r.cells_visited, r.top, r.left) == (
        want.side, want.area, want.cells_visited, want.top, want.left)


def test_dp_invalid_cells(torch):
    a = np.ones((40, 40), np.uint8)
    a[17, 3] = 2
    with pytest.raises(ValueError):
        dp_full(torch.from_numpy(a).cuda())


def test_dp_cfg3_equals_freq(torch):
    """The DP kernel is an independent algorithm: at cfg3 size it must agree
    with the band engine on side and location."""
    from paper_2503_18974_b200 import configs
    m = configs.cfg3_device()
    a, b = dp_full(m), freq_square(m)
    assert (a.side, a.top, a.left) == (b.side, b.top, b.left) == (2048, 3898, 9709)


@pytest.mark.parametrize("shape", [(300, 70000), (2 ** 21 + 5, 3)])
def test_freq_square_beyond_band_engine(torch, shape):
    """cols > 65536 / rows >= 2^21: the drop-in freq_square still answers (the
    library routes such shapes to the DP kernel); host and device inputs."""
    from paper_2503_18974_b200 import freq_square_bits
    from paper_2503_18974_b200.grid import pack_bits
    rows, cols = shape
    rng = np.random.default_rng(rows + cols)
    a = (rng.random((rows, cols)) < 0.97).astype(np.uint8)
    want = oracle.freq(a)
    for got in (freq_square(a), freq_square(torch.from_numpy(a).cuda()),
                freq_square_bits(pack_bits(a), cols)):
        assert (got.side, got.area, got.cells_visited, got.top, got.left) == (
            want.side, want.area, want.cells_visited, want.top, want.left)
