"""Pin the CPU oracle against the reference's golden vectors (no GPU needed).

The fixtures in tests/golden/ were produced by importing the reference itself
(tests/golden/make_golden.py); this file checks the C restatement and the
repo's generator mirror against them, then checks the band algebra (P5/P6)
that the CUDA kernels implement against the oracle's whole-matrix answer.
"""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import oracle
from paper_2503_18974_b200 import grid

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def _check(res, side, top, left):
    assert (res.side, res.top, res.left) == (side, top, left)
    assert res.area == side * side


def test_kats_freq_and_dp(golden):
    for case in golden["kats"]:
        a = np.array(case["rows"], np.uint8)
        _check(oracle.freq(a), case["side"], case["top"], case["left"])
        _check(oracle.dp(a), case["side"], case["top"], case["left"])
        assert oracle.freq(a).cells_visited == a.size


def test_genspec_pins_and_mirror(golden):
    for case in golden["genspec"]:
        spec = grid.GenSpec(*case["spec"])
        m = grid.generate_matrix(spec)
        assert hashlib.sha256(m.cells).hexdigest() == case["sha256"]
        assert m.ones() == case["ones"]
        _check(oracle.freq(m.to_array()), case["side"], case["top"], case["left"])
    m = grid.generate_matrix(grid.GenSpec(4, 4, 0.5, 7))
    assert grid.serialize_matrix(m) == golden["pins"]["genspec_4_4_0.5_7_text"]


def test_generator_mirror_matches_python_random():
    for seed in (0, 1, 99, 2**63 + 5):
        spec = grid.GenSpec(7, 9, 0.37, seed)
        rng = random.Random(seed)
        want = bytes(1 if rng.random() < 0.37 else 0 for _ in range(63))
        assert grid.generate_matrix(spec).cells == want


def test_edge_cases(golden):
    for case in golden["edge"]:
        if case["kind"] == "empty":
            r = oracle.freq(np.zeros((0, 0), np.uint8))
            assert (r.side, r.area, r.cells_visited, r.top, r.left) == (0, 0, 0, -1, -1)
            continue
        m = grid.generate_edge_case(grid.EdgeKind(case["kind"]), case["n"])
        _check(oracle.freq(m.to_array()), case["side"], case["top"], case["left"])


def test_exhaustive_4x4():
    ex = np.load(os.path.join(GOLDEN, "exhaustive4x4.npz"))
    total = 0
    for r in range(1, 5):
        for c in range(1, 5):
            bits = r * c
            pats = np.arange(2 ** bits, dtype=np.int64)
            # MSB-first pattern bits -> row-major cells (verify.py:141-150)
            cells = ((pats[:, None] >> np.arange(bits - 1, -1, -1)) & 1).astype(np.uint8)
            batch = cells.reshape(-1, r, c)
            res = oracle.freq_batch(batch)
            side = np.array([x.side for x in res])
            top = np.array([x.top for x in res])
            left = np.array([x.left for x in res])
            assert np.array_equal(side, ex[f"side_{r}x{c}"])
            assert np.array_equal(top, ex[f"top_{r}x{c}"])
            assert np.array_equal(left, ex[f"left_{r}x{c}"])
            total += len(pats)
    assert total == 74_954


def test_random_campaign_10k():
    rc = np.load(os.path.join(GOLDEN, "random_campaign.npz"))
    n = len(rc["rows"])
    assert n == 10_000
    for k in range(n):
        spec = grid.GenSpec(int(rc["rows"][k]), int(rc["cols"][k]), float(rc["density"][k]),
                            int(rc["seed"][k]))
        res = oracle.freq(grid.generate_array(spec))
        assert (res.side, res.top, res.left) == (rc["side"][k], rc["top"][k], rc["left"][k]), k


def test_freq_bits_matches_u8():
    rng = np.random.default_rng(5)
    for _ in range(200):
        rows, cols = rng.integers(1, 80, size=2)
        a = (rng.random((rows, cols)) < rng.choice([0.5, 0.8, 0.95])).astype(np.uint8)
        w = grid.pack_bits(a)
        assert np.array_equal(grid.unpack_bits(w, cols), a)
        assert oracle.freq_bits(w, cols) == oracle.freq(a)


def _planted(rng, rows, cols, p, k):
    a = (rng.random((rows, cols)) < p).astype(np.uint8)
    if k and k <= min(rows, cols):
        t = rng.integers(0, rows - k + 1)
        l_ = rng.integers(0, cols - k + 1)
        a[t:t + k, l_:l_ + k] = 1
    return a


def test_band_algebra_matches_whole_matrix():
    """P6: band passes + carries + data-free fix-ups == Algorithm 1 (side+location)."""
    rng = np.random.default_rng(11)
    for it in range(1500):
        rows = int(rng.integers(1, 90))
        cols = int(rng.integers(1, 70))
        p = float(rng.choice([0.5, 0.8, 0.9, 0.97, 1.0]))
        a = _planted(rng, rows, cols, p, int(rng.integers(0, 20)))
        want = oracle.freq(a)
        for nb in (1, 2, 3, int(rng.integers(1, rows + 1))):
            got = oracle.solve_banded(a, 0, cols, nb)
            assert got == want, (it, nb)
        if it % 10 == 0:
            got = oracle.solve_banded(grid.pack_bits(a), 1, cols, 4)
            assert got == want


def test_band_pass_summaries():
    rng = np.random.default_rng(3)
    a = (rng.random((37, 45)) < 0.9).astype(np.uint8)
    e, b, ao, key = oracle.band_pass(a, 0, 5, 20, 45)
    band = a[5:20]
    for j in range(45):
        col = band[:, j]
        zeros = np.nonzero(col == 0)[0]
        assert e[j] == (zeros[0] if len(zeros) else 15)
        assert b[j] == (15 - 1 - zeros[-1] if len(zeros) else 15)
        assert ((ao[j // 32] >> (j % 32)) & 1) == (len(zeros) == 0)
    s, bottom, right = oracle.unpack_key(key)
    whole = oracle.freq(band)
    assert (s, bottom - 5 - s + 1, right - s + 1) == (whole.side, whole.top, whole.left)


def test_hash_generator_numpy_restatement():
    """The counter-hash generator has a vectorised numpy restatement (configs.py)."""
    from paper_2503_18974_b200 import configs
    seed, thr = 1234, configs.thr53(0.9)
    a = oracle.gen_hash_u8(seed, thr, 3, 5, 77)
    assert np.array_equal(a, configs.hash_u8(seed, thr, 3, 5, 77))
    w = oracle.gen_hash_bits(seed, thr, 3, 5, 77)
    assert np.array_equal(w, grid.pack_bits(a))
