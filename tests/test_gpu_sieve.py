"""Sieve engine (csrc/msq_sieve.cuh, plan.engine == 2) against the oracle.

The engine streams the bit-packed matrix once into a bitmap of all-ones 8x8
blocks, runs Algorithm 1 (reference squares.py:84-103) on that bitmap and then
exactly on the cell windows of its few candidates.  It must either return the
reference's answer (side and the implied location) or say it cannot decide
(status bits 1/2 -> MSQ_EAGAIN), in which case the same plan runs the band
engine.  Covered: random sparse-zero matrices with planted squares around the
decidable range 56..222, every alignment of a square against the 8-cell grid,
squares on the matrix borders, ties (first in row-major order of the bottom-right
cell), ragged widths and strides, undecided inputs, and row slices with the
256-row halo (the multi-GPU protocol on virtual ranks).
"""
import ctypes

import numpy as np
import pytest

import oracle
from paper_2503_18974_b200 import _native as N
from paper_2503_18974_b200 import grid

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    from paper_2503_18974_b200 import build
    build.build()
    oracle.build()
    return t


def _same(got, want):
    assert (got.side, got.area, got.top, got.left) == (want.side, want.area, want.top, want.left), (got, want)


def _solve(torch, a, engine=2, ld=None):
    from paper_2503_18974_b200.squares import Solver
    rows, cols = a.shape
    w = grid.pack_bits(a)
    if ld is None and w.shape[1] % 4:
        ld = (w.shape[1] + 3) // 4 * 4  # the sieve streams rows in 16-byte units
    if ld is not None:
        pad = np.zeros((rows, ld), np.uint32)
        pad[:, :w.shape[1]] = w
        pad[:, w.shape[1]:] = 0xDEADBEEF  # never read as cells
        w = pad
    s = Solver(N.FMT_BITS, rows, cols, ld=w.shape[1], engine=engine)
    got = s.solve(torch.from_numpy(w.view(np.int32)).cuda())[0]
    return got, getattr(s, "sieve_retries", 0)


def test_random_sparse_matrices(torch):
    rng = np.random.default_rng(7)
    decided = 0
    for it in range(48):
        rows = int(rng.integers(64, 2600))
        cols = max(64, 128 * int(rng.integers(1, 28)) - int(rng.choice([0, 0, 5, 31, 64, 95])))
        p = [0.999, 0.9995, 0.998, 0.9999, 0.995][it % 5]
        a = (rng.random((rows, cols)) < p).astype(np.uint8)
        k = int(rng.integers(40, 250))
        if it % 4 != 3 and min(rows, cols) > k:
            top, left = int(rng.integers(0, rows - k + 1)), int(rng.integers(0, cols - k + 1))
            a[top:top + k, left:left + k] = 1
        got, retried = _solve(torch, a)
        _same(got, oracle.freq(a))
        decided += 0 if retried else 1
    assert decided >= 24  # most of these are the sieve's own answers, not the fall-back's


@pytest.mark.parametrize("side", [55, 56, 57, 63, 64, 65, 133, 221, 222, 223, 229])
def test_every_alignment_of_a_planted_square(torch, side):
    """A square of the given side at every offset mod 8 in both directions over a
    background whose own squares stay far below it."""
    rng = np.random.default_rng(side)
    rows, cols = 700, 768
    base = (rng.random((rows, cols)) < 0.97).astype(np.uint8)
    for dr in range(8):
        for dc in (dr, (3 * dr + 5) % 8):
            a = base.copy()
            top, left = 200 + dr, 264 + dc
            a[top:top + side, left:left + side] = 1
            if top + side < rows:
                a[top + side, left:left + side:7] = 0  # the square is exactly this tall
            if left + side < cols:
                a[top:top + side:5, left + side] = 0
            a[top - 1, left:left + side:6] = 0
            a[top:top + side:6, left - 1] = 0
            got, _ = _solve(torch, a)
            _same(got, oracle.freq(a))
            assert got.side == side


def test_squares_on_the_borders_and_ties(torch):
    rows, cols = 1000, 1152
    rng = np.random.default_rng(11)
    base = (rng.random((rows, cols)) < 0.98).astype(np.uint8)
    k = 100
    spots = [(0, 0), (0, cols - k), (rows - k, 0), (rows - k, cols - k), (3, cols - k - 2), (rows - k - 1, 5)]
    for top, left in spots:
        a = base.copy()
        a[top:top + k, left:left + k] = 1
        got, _ = _solve(torch, a)
        _same(got, oracle.freq(a))
    # several maximal squares: the first bottom-right cell in row-major order wins
    a = base.copy()
    for top, left in [(500, 700), (500, 100), (493, 400), (120, 900), (121, 30)]:
        a[top:top + k, left:left + k] = 1
    got, _ = _solve(torch, a)
    want = oracle.freq(a)
    _same(got, want)
    assert got.side >= k


def test_strided_rows_and_heights_not_multiples_of_eight(torch):
    rng = np.random.default_rng(12)
    for rows, cols, ld in [(777, 1000, 36), (1501, 2017, 64), (95, 128, 8), (64, 3000, 96), (900, 1100, 36)]:
        a = (rng.random((rows, cols)) < 0.999).astype(np.uint8)
        k = min(rows, 150)
        top = rows - k  # ends in the last (partial) block row
        a[top:top + k, cols - k:cols] = 1
        got, _ = _solve(torch, a, ld=ld)
        _same(got, oracle.freq(a))


def test_undecided_inputs_fall_back_to_the_band_engine(torch):
    from paper_2503_18974_b200.squares import Solver
    rng = np.random.default_rng(13)
    rows, cols = 1200, 1280
    cases = {
        "dense zeros": (rng.random((rows, cols)) < 0.9).astype(np.uint8),
        "all ones": np.ones((rows, cols), np.uint8),
        "all zeros": np.zeros((rows, cols), np.uint8),
    }
    big = (rng.random((rows, cols)) < 0.999).astype(np.uint8)
    big[100:500, 300:700] = 1
    cases["planted 400"] = big
    stripes = np.ones((8192, 8192), np.uint8)
    stripes[:, ::64] = 0  # 16384 maximal squares of side 63: the candidate list overflows
    stripes[::64, :] = 0
    cases["grid of 63-squares"] = stripes
    lib = N.load()
    for name, a in cases.items():
        rows, cols = a.shape
        want = oracle.freq(a)
        got, retried = _solve(torch, a)
        _same(got, want)
        assert retried == 1, name
        # the C ABI says so itself: msq_decode of the undecided launch is MSQ_EAGAIN
        s = Solver(N.FMT_BITS, rows, cols, engine=2)
        w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
        s.launch(w)
        host = s.res.cpu().numpy()
        block = N.MsqDevResult.from_buffer_copy(host[:32].tobytes())
        out = N.MsqResult()
        assert lib.msq_decode(ctypes.byref(block), rows, cols, ctypes.byref(out)) == N.MSQ_EAGAIN, name
        assert block.status & 6
        # and the synchronous call retries on its own
        from paper_2503_18974_b200.squares import freq_square_bits
        _same(freq_square_bits(w, cols), want)


@pytest.mark.parametrize("world", [2, 3])
def test_row_slices_with_halo(torch, world):
    """The multi-GPU sieve protocol on virtual ranks: every rank solves (the last
    256 rows of the rank above, its own rows) alone; the max of the keys is the
    whole matrix's answer, also for squares that cross a rank boundary."""
    from paper_2503_18974_b200.distributed import SIEVE_HALO, GpuBackend, decode_key, slice_rows
    rng = np.random.default_rng(200 + world)
    for it in range(4):
        rows, cols = world * 1024 + 8 * int(rng.integers(0, 40)), 4096
        a = (rng.random((rows, cols)) < 0.9992).astype(np.uint8)
        k = int(rng.integers(90, 215))
        bound = slice_rows(rows, world, 1)[0]
        top = [bound - k // 2, bound - k + 1, bound - 1, bound - k - 3][it]
        left = int(rng.integers(0, cols - k))
        a[top:top + k, left:left + k] = 1
        full = grid.pack_bits(a).view(np.int32)
        keys = []
        for q in range(world):
            r0, n = slice_rows(rows, world, q)
            src = torch.from_numpy(np.ascontiguousarray(full[r0:r0 + n])).cuda()
            halo = torch.from_numpy(np.ascontiguousarray(full[r0 - SIEVE_HALO:r0])).cuda() if q > 0 else None
            be = GpuBackend(N.FMT_BITS, n, cols, r0, engine=2)
            assert be.is_sieve
            be.sieve(src, halo)
            keys.append(be.key_status().clone())
        ks = torch.stack(keys).max(dim=0).values.cpu().numpy()
        assert int(ks[1]) in (0, 1), (ks, [k.cpu().numpy() for k in keys])
        _same(decode_key(int(ks[0]), 0, rows, cols), oracle.freq(a))


def test_row_band_solver_single_rank_uses_the_sieve(torch):
    from paper_2503_18974_b200.distributed import GpuBackend, RowBandSolver
    rng = np.random.default_rng(14)
    rows, cols = 4096, 4096
    a = (rng.random((rows, cols)) < 0.999).astype(np.uint8)
    a[1000:1150, 2000:2150] = 1
    w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
    be = GpuBackend(N.FMT_BITS, rows, cols, 0)
    assert be.is_sieve  # automatic from 4096 x 4096
    solver = RowBandSolver(rows, cols, 0, 1, be)
    _same(solver.solve(w), oracle.freq(a))
    assert solver.sieve and solver.sieve_retries == 0
    a2 = (rng.random((rows, cols)) < 0.97).astype(np.uint8)  # squares far below 56: the band protocol
    w2 = torch.from_numpy(grid.pack_bits(a2).view(np.int32)).cuda()
    _same(solver.solve(w2), oracle.freq(a2))
    assert not solver.sieve and solver.sieve_retries == 1


def test_workspace_is_not_overrun(torch):
    """compute-sanitizer is closed on this GPU pool: a guard band behind the
    plan's workspace (and around the result block) must survive a solve with the
    largest halo, on a shape whose block bitmap ends exactly at the plan's size."""
    from paper_2503_18974_b200.distributed import SIEVE_HALO, GpuBackend
    rng = np.random.default_rng(15)
    for rows, cols in [(1024, 4096), (1000, 2304), (4096, 8192)]:
        a = (rng.random((rows + SIEVE_HALO, cols)) < 0.9993).astype(np.uint8)
        a[200:340, 100:240] = 1
        full = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
        be = GpuBackend(N.FMT_BITS, rows, cols, SIEVE_HALO, engine=2)
        need, guard = int(be.plan.ws_bytes), 1 << 16
        buf = torch.full((guard + need + guard,), 0x5A, dtype=torch.uint8, device="cuda")
        be.ws = buf[guard:guard + need]
        resbuf = torch.full((256 + 32 + 256,), 0x5A, dtype=torch.uint8, device="cuda")
        be.res = resbuf[256:288]
        # the halo comes with its own row stride (msq_rank_sieve's halo_ld)
        halo = torch.full((SIEVE_HALO, full.shape[1] + 8), -1, dtype=full.dtype, device="cuda")
        halo[:, :full.shape[1]] = full[:SIEVE_HALO]
        be.sieve(full[SIEVE_HALO:], halo[:, :full.shape[1]])
        torch.cuda.synchronize()
        assert bool((buf[:guard] == 0x5A).all()) and bool((buf[guard + need:] == 0x5A).all())
        assert bool((resbuf[:256] == 0x5A).all()) and bool((resbuf[288:] == 0x5A).all())
        from paper_2503_18974_b200.distributed import decode_key
        ks = be.key_status().cpu().numpy()
        want = oracle.freq(a)
        got = decode_key(int(ks[0]), 0, rows + SIEVE_HALO, cols)
        assert int(ks[1]) == 0 and (got.side, got.top, got.left) == (want.side, want.top, want.left)


@pytest.mark.parametrize("phases", [2, 3, 4])
def test_streaming_in_sweeps_with_the_coarse_pass_beside_it(torch, phases):
    """From the second sweep on the coarse pass and the verifier run while the
    streaming pass still writes the bitmap (phase counters, done counter).  Forced
    sweeps on small shapes (also fewer block rows than sweeps x bands), squares
    across the sweeps' borders, CTA shapes of 1..8 streaming warps, repeated solves
    on one plan."""
    lib = N.load()
    rng = np.random.default_rng(40 + phases)
    try:
        lib.msq_debug_set_sieve_phases(phases)
        for it in range(10):
            rows = int(rng.choice([200, 1000, 3000, 6000]))
            cols = int(rng.choice([256, 2048, 8192]))
            lib.msq_debug_set_sieve_wpc(int(rng.choice([1, 3, 8])))
            a = (rng.random((rows, cols)) < 0.9994).astype(np.uint8)
            for q in range(1, phases):  # squares over the borders between sweeps
                k = int(rng.integers(60, min(rows, cols, 210)))
                top = max(0, min(rows - k, rows * q // phases - k // 2))
                left = int(rng.integers(0, cols - k + 1))
                a[top:top + k, left:left + k] = 1
            want = oracle.freq(a)
            for _ in range(3):
                got, _ = _solve(torch, a)
                _same(got, want)
    finally:
        lib.msq_debug_set_sieve_phases(0)
        lib.msq_debug_set_sieve_wpc(8)


@pytest.mark.slow
def test_tall_matrix_takes_four_sweeps_on_its_own(torch):
    rng = np.random.default_rng(50)
    rows, cols = 40960, 2048  # 5120 block rows: four sweeps by the plan's own rule
    a = (rng.random((rows, cols)) < 0.9993).astype(np.uint8)
    for top in (10200, 20400, 30700):
        a[top:top + 150, 700:850] = 1
    got, retried = _solve(torch, a, engine=-1)
    _same(got, oracle.freq(a))
    assert retried == 0


def test_repeated_solves_give_one_answer(torch):
    """The coarse pass and the verifier race the streaming pass by design
    (candidates appear in any order, levels rise at different moments): the
    answer must not depend on it.  200 solves of one input, four sweeps."""
    from paper_2503_18974_b200.squares import Solver
    lib = N.load()
    rng = np.random.default_rng(60)
    rows, cols = 6000, 8192
    a = (rng.random((rows, cols)) < 0.9992).astype(np.uint8)
    for top, left in [(1400, 300), (1499, 4000), (2950, 7000), (4490, 5000), (4500, 100)]:
        a[top:top + 120, left:left + 120] = 1  # ties across the sweeps' borders
    want = oracle.freq(a)
    w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
    try:
        lib.msq_debug_set_sieve_phases(4)
        s = Solver(N.FMT_BITS, rows, cols, engine=2)
        for _ in range(200):
            _same(s.solve(w)[0], want)
        assert getattr(s, "sieve_retries", 0) == 0
    finally:
        lib.msq_debug_set_sieve_phases(0)
