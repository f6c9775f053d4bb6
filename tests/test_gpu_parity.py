"""GPU parity: the sm_100a library (through the C ABI) against the CPU oracle
and the reference's golden vectors.  Bit-exact on side, area, cells_visited,
top and left; intermediates (band summaries, band keys) bit-exact against the
oracle's restatement of the band algebra."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2503_18974_b200 import _native as N
from paper_2503_18974_b200 import configs, grid
from paper_2503_18974_b200.squares import Solver, freq_square, freq_square_bits, solve_batch

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def torch():
    import torch as t
    from paper_2503_18974_b200 import build
    build.build()
    return t


def _same(res, want):
    assert (res.side, res.area, res.cells_visited, res.top, res.left) == (
        want.side, want.area, want.cells_visited, want.top, want.left)


def test_golden_kats(torch):
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        g = json.load(f)
    for case in g["kats"]:
        m = grid.BinaryMatrix.from_rows(case["rows"])
        r = freq_square(m)
        assert (r.side, r.top, r.left) == (case["side"], case["top"], case["left"]), case["name"]
        assert r.area == r.side ** 2 and r.cells_visited == m.rows * m.cols
    for case in g["genspec"]:
        m = grid.generate_matrix(grid.GenSpec(*case["spec"]))
        r = freq_square(m)
        assert (r.side, r.top, r.left) == (case["side"], case["top"], case["left"]), case["spec"]
    for case in g["edge"]:
        if case["kind"] == "empty":
            r = freq_square(grid.EMPTY_MATRIX)
            assert (r.side, r.area, r.cells_visited, r.top, r.left) == (0, 0, 0, -1, -1)
            continue
        m = grid.generate_edge_case(grid.EdgeKind(case["kind"]), case["n"])
        r = freq_square(m)
        assert (r.side, r.top, r.left) == (case["side"], case["top"], case["left"]), case["name"]


def test_exhaustive_4x4_batched(torch):
    ex = np.load(os.path.join(GOLDEN, "exhaustive4x4.npz"))
    total = 0
    for r in range(1, 5):
        for c in range(1, 5):
            bits = r * c
            pats = np.arange(2 ** bits, dtype=np.int64)
            cells = ((pats[:, None] >> np.arange(bits - 1, -1, -1)) & 1).astype(np.uint8)
            res = solve_batch(cells.reshape(-1, r, c))
            assert np.array_equal([x.side for x in res], ex[f"side_{r}x{c}"])
            assert np.array_equal([x.top for x in res], ex[f"top_{r}x{c}"])
            assert np.array_equal([x.left for x in res], ex[f"left_{r}x{c}"])
            total += len(pats)
    assert total == 74_954


def test_random_campaign_10k(torch):
    rc = np.load(os.path.join(GOLDEN, "random_campaign.npz"))
    for k in range(len(rc["rows"])):
        spec = grid.GenSpec(int(rc["rows"][k]), int(rc["cols"][k]), float(rc["density"][k]),
                            int(rc["seed"][k]))
        r = freq_square(grid.generate_matrix(spec))
        assert (r.side, r.top, r.left) == (rc["side"][k], rc["top"][k], rc["left"][k]), k


def _planted(rng, rows, cols, p, k):
    a = (rng.random((rows, cols)) < p).astype(np.uint8)
    if k and k <= min(rows, cols):
        t = int(rng.integers(0, rows - k + 1))
        l_ = int(rng.integers(0, cols - k + 1))
        a[t:t + k, l_:l_ + k] = 1
    return a


@pytest.mark.parametrize("fmt", ["u8", "bits"])
def test_band_intermediates_match_oracle(torch, fmt):
    """Deterministic mode: e/b/all-ones summaries and pass-1 band keys == oracle P6 pass."""
    rng = np.random.default_rng(21 if fmt == "u8" else 22)
    for it in range(60):
        rows = int(rng.integers(8, 400))
        cols = int(rng.choice([32, 64, 96, 200, 256, 512, 1000, 2048]))
        p = float(rng.choice([0.6, 0.9, 0.97, 0.995, 1.0]))
        a = _planted(rng, rows, cols, p, int(rng.integers(0, 60)))
        nb = int(rng.integers(1, min(rows, 40) + 1))
        if fmt == "u8":
            src = torch.from_numpy(a).cuda()
            s = Solver(N.FMT_U8, rows, cols, nbands=nb, deterministic=True)
            host = a
            f = 0
        else:
            w = grid.pack_bits(a)
            src = torch.from_numpy(w.view(np.int32)).cuda()
            s = Solver(N.FMT_BITS, rows, cols, nbands=nb, deterministic=True)
            host = w
            f = 1
        res = s.solve(src)[0]
        _same(res, oracle.freq(a))
        if s.nbands > 1:
            e, b, ao, bk = (x.cpu().numpy() for x in s.views())
            for band in range(s.nbands):
                r0 = rows * band // s.nbands
                r1 = rows * (band + 1) // s.nbands
                oe, ob, oao, okey = oracle.band_pass(host, f, r0, r1, cols, 1)
                assert np.array_equal(e[band, :cols].view(np.uint16), oe), (it, band)
                assert np.array_equal(b[band, :cols].view(np.uint16), ob), (it, band)
                assert np.array_equal(ao[band].view(np.uint32), oao), (it, band)
                assert int(bk[band]) == okey, (it, band)


def test_random_banded_solves(torch):
    """Non-deterministic (shared-threshold) mode, many band counts and shapes."""
    rng = np.random.default_rng(7)
    for it in range(300):
        rows = int(rng.integers(1, 700))
        cols = int(rng.integers(1, 700))
        p = float(rng.choice([0.3, 0.8, 0.95, 0.99, 1.0]))
        a = _planted(rng, rows, cols, p, int(rng.integers(0, 120)))
        want = oracle.freq(a)
        src = torch.from_numpy(a).cuda()
        nb = int(rng.integers(1, min(rows, 64) + 1))
        _same(Solver(N.FMT_U8, rows, cols, nbands=nb).solve(src)[0], want)
        if it % 3 == 0:
            w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
            _same(Solver(N.FMT_BITS, rows, cols, nbands=nb).solve(w)[0], want)


@pytest.mark.parametrize("cols", [65536, 40000, 33000])
def test_wide_rows_every_word_width(torch, cols):
    """Widths that select 8 (bits) / 4 (u8) words per thread, both formats."""
    rng = np.random.default_rng(cols)
    a = (rng.random((300, cols)) < 0.995).astype(np.uint8)
    a[100:190, cols - 120:cols - 30] = 1  # planted 90x90 near the right edge
    want = oracle.freq(a)
    w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
    for nb in (1, 7):
        _same(Solver(N.FMT_BITS, 300, cols, nbands=nb).solve(w)[0], want)
        _same(Solver(N.FMT_U8, 300, cols, nbands=nb).solve(torch.from_numpy(a).cuda())[0], want)


def test_strided_and_odd_widths(torch):
    rng = np.random.default_rng(9)
    for cols in (1, 3, 17, 31, 33, 63, 65, 100, 130):
        a = (rng.random((50, cols)) < 0.9).astype(np.uint8)
        wide = np.zeros((50, cols + 19), np.uint8)
        wide[:, :cols] = a
        t = torch.from_numpy(wide).cuda()
        s = Solver(N.FMT_U8, 50, cols, ld=cols + 19, nbands=3)
        _same(s.solve(t)[0], oracle.freq(a))
        _same(freq_square(a), oracle.freq(a))
        _same(freq_square_bits(grid.pack_bits(a), cols), oracle.freq(a))


def test_invalid_cells_raise_value_error(torch):
    a = np.ones((40, 64), np.uint8)
    a[17, 5] = 2
    with pytest.raises(ValueError):
        freq_square(a)
    t = torch.from_numpy(a).cuda()
    with pytest.raises(ValueError):
        freq_square(t)


def test_device_generator_matches_oracle(torch):
    thr = configs.thr53(0.97)
    d = configs.device_hash("u8", 77, 0.97, 64, 300).cpu().numpy()
    assert np.array_equal(d, oracle.gen_hash_u8(77, thr, 0, 64, 300))
    w = configs.device_hash("bits", 77, 0.97, 64, 300).cpu().numpy().view(np.uint32)
    assert np.array_equal(w, oracle.gen_hash_bits(77, thr, 0, 64, 300))


def test_cfg1(torch):
    r = freq_square(grid.generate_matrix(grid.GenSpec(512, 512, 0.7, 0)))
    assert (r.side, r.area, r.cells_visited, r.top, r.left) == (5, 25, 512 * 512, 0, 67)


def test_cfg2_batch_vs_oracle(torch):
    cells = configs.cfg2_array()  # all 4096 matrices of the config
    got = solve_batch(cells)
    want = oracle.freq_batch(cells)
    for g_, w_ in zip(got, want):
        _same(g_, w_)


def test_cfg3_planted_and_edges(torch):
    m = configs.cfg3_device()
    want = oracle.freq(m.cpu().numpy())
    _same(freq_square(m), want)
    top, left = configs.cfg3_square_pos()
    assert want.side >= 2048
    z = torch.zeros((16384, 16384), dtype=torch.uint8, device="cuda")
    r = freq_square(z)
    assert (r.side, r.top, r.left) == (0, -1, -1)
    z.fill_(1)
    r = freq_square(z)
    assert (r.side, r.area, r.top, r.left) == (16384, 16384 ** 2, 0, 0)


@pytest.mark.slow
def test_cfg4_full_size(torch):
    w = configs.cfg4_device()
    got = freq_square_bits(w, 65536)
    host = w.cpu().numpy().view(np.uint32)
    _same(got, oracle.freq_bits(host, 65536))


@pytest.mark.slow
def test_cfg5_full_size(torch):
    m = configs.cfg5_device()
    got = freq_square(m)
    _same(got, oracle.freq(m.cpu().numpy()))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_row_band_ranks_on_one_gpu(torch, world):
    """The rank API (msq_rank_pass1/summary/compose_carry/rank_fixup) with
    `world` virtual ranks run one after another on one GPU (no kernel waits on
    another), gathered on the device: same answer as the whole matrix."""
    from paper_2503_18974_b200.distributed import GpuBackend, decode_key, slice_rows
    rng = np.random.default_rng(world)
    for it in range(6):
        rows = int(rng.integers(world * 8, 900))
        cols = int(rng.choice([64, 300, 1024, 4096]))
        a = (rng.random((rows, cols)) < [0.99, 0.999, 1.0][it % 3]).astype(np.uint8)
        k = min(rows, cols) // 2
        a[rows // 2 - k // 2:rows // 2 - k // 2 + k, 3:3 + k] = 1  # crosses rank boundaries
        for fmt in (N.FMT_U8, N.FMT_BITS):
            full = a if fmt == N.FMT_U8 else grid.pack_bits(a).view(np.int32)
            bes, srcs = [], []
            rank_rows = [slice_rows(rows, world, q)[1] for q in range(world)]
            for q in range(world):
                r0, n = slice_rows(rows, world, q)
                src = torch.from_numpy(np.ascontiguousarray(full[r0:r0 + n])).cuda()
                be = GpuBackend(fmt, n, cols, r0, nbands=int(rng.integers(1, 6)))
                be.pass1(src)
                bes.append(be)
                srcs.append(src)
            gathered = torch.stack([be.rank_summary().clone() for be in bes])
            keys = []
            for q, be in enumerate(bes):
                base = be.compose(gathered, rank_rows, q) if q > 0 else None
                be.fixup(base)
                keys.append(be.key_status())
            ks = torch.stack(keys).max(dim=0).values.cpu().numpy()
            got = decode_key(int(ks[0]), int(ks[1]), rows, cols)
            _same(got, oracle.freq(a))


@pytest.mark.parametrize("fmt", ["u8", "bits"])
def test_seed_lower_bound_keeps_ties_exact(torch, fmt):
    """Matrices big enough for the lower-bound seed (strip-top climbs before
    pass 1): the seed may equal the answer, and the reported location must
    still be the lexicographically smallest maximal square."""
    rng = np.random.default_rng(11 if fmt == "u8" else 12)
    rows, cols = 2048, 1024
    cases = [
        [(0, 900, 60), (0, 100, 60)],      # both hang from the strip top: left decides
        [(0, 500, 60), (5, 20, 60)],       # seed square is the answer (top 0)
        [(0, 500, 60), (300, 20, 61)],     # a larger square elsewhere
        [(700, 40, 75), (0, 200, 75), (1900, 900, 75)],
        [(0, 0, 128)],                     # climb runs to the strip height
    ]
    for squares in cases:
        a = (rng.random((rows, cols)) < 0.9).astype(np.uint8)
        for (t_, l_, k) in squares:
            a[t_:t_ + k, l_:l_ + k] = 1
        want = oracle.freq(a)
        if fmt == "u8":
            got = freq_square(a)
        else:
            got = freq_square_bits(grid.pack_bits(a), cols)
        _same(got, want)


def test_team_engine_single_matrices(torch):
    """Team engine (forced by the plan's engine choice) on one matrix at a
    time: odd widths, strides, both formats."""
    rng = np.random.default_rng(31)
    for it in range(400):
        rows = int(rng.integers(1, 1200))
        cols = int(rng.integers(1, 1025)) if it % 4 else int(rng.choice([32, 64, 256, 512, 1024]))
        p = float(rng.choice([0.3, 0.7, 0.9, 0.97, 0.995, 1.0]))
        a = _planted(rng, rows, cols, p, int(rng.integers(0, 200)))
        want = oracle.freq(a)
        pad = int(rng.choice([0, 0, 16, 5]))
        wide = np.zeros((rows, cols + pad), np.uint8)
        wide[:, :cols] = a
        s = Solver(N.FMT_U8, rows, cols, ld=cols + pad, engine=1)
        assert int(s.plan.engine) == 1
        _same(s.solve(torch.from_numpy(wide).cuda())[0], want)
        if it % 2 == 0:
            w = grid.pack_bits(a)
            sb = Solver(N.FMT_BITS, rows, cols, ld=w.shape[1], engine=1)
            assert int(sb.plan.engine) == 1
            _same(sb.solve(torch.from_numpy(w.view(np.int32)).cuda())[0], want)


def test_team_engine_batches(torch):
    """Batched solves (team engine by default) for every team width and both plane counts."""
    rng = np.random.default_rng(32)
    for rows, cols in ((7, 3), (40, 33), (100, 64), (256, 256), (300, 130), (511, 512), (600, 1000),
                       (1500, 96), (2040, 40)):
        batch = int(rng.integers(2, 70))
        p = float(rng.choice([0.5, 0.9, 0.99]))
        cells = np.stack([_planted(rng, rows, cols, p, int(rng.integers(0, min(rows, cols) + 1)))
                          for _ in range(batch)])
        got = solve_batch(cells)
        for g_, w_ in zip(got, oracle.freq_batch(cells)):
            _same(g_, w_)
        words = (cols + 31) // 32
        wb = np.stack([grid.pack_bits(c) for c in cells]).reshape(batch, rows, words)
        s = Solver(N.FMT_BITS, rows, cols, batch=batch)
        assert int(s.plan.engine) == 1
        for g_, w_ in zip(s.solve(torch.from_numpy(wb.view(np.int32)).cuda()), oracle.freq_batch(cells)):
            _same(g_, w_)


def test_team_engine_invalid_cells(torch):
    cells = np.ones((5, 64, 64), np.uint8)
    cells[3, 10, 7] = 3
    with pytest.raises(ValueError):
        solve_batch(cells)


@pytest.mark.parametrize("floor", [96, 120, 150, 200])
def test_strip_pass_bits(torch, floor):
    """Strip band pass (msq_strip.cuh): bit-packed, several bands, start threshold in its range.

    The plan's test_floor presets the shared best side (a lower bound <= the
    answer, as the seed provides on large inputs) so the strip pass runs on
    moderate sizes; planted sides above 222 exercise its hand-back to
    pass1_kernel; floor 200 runs the 5-word run filter (t in 191..222)."""
    rng = np.random.default_rng(40 + floor)
    for it in range(14):
        rows = int(rng.integers(300, 2500))
        cols = int(rng.choice([8192, 9000, 16384, 40000, 65536]))
        p = float(rng.choice([0.99, 0.997, 0.999, 0.9995]))
        k = int(rng.integers(floor, 260 if it % 4 == 0 else max(200, floor + 20)))
        a = _planted(rng, rows, cols, p, min(k, rows))
        if it % 5 == 1:  # a second square of the same side further down-left: ties
            kk = min(k, rows)
            t0, l0 = int(rng.integers(0, rows - kk + 1)), int(rng.integers(0, cols - kk + 1))
            a[t0:t0 + kk, l0:l0 + kk] = 1
        want = oracle.freq(a)
        if want.side < floor:
            continue
        w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
        nb = int(rng.integers(2, min(rows // 8, 150) + 1))
        _same(Solver(N.FMT_BITS, rows, cols, nbands=nb, test_floor=floor).solve(w)[0], want)


@pytest.mark.parametrize("world", [2, 4])
def test_row_band_ranks_pooled_seed(torch, world):
    """RowBandSolver's multi-rank flow with the seeds pooled: msq_rank_seed on
    every virtual rank, max of their best sides written back (the all-reduce),
    msq_rank_band_pass (strip pass on bit-packed bands), summaries, carries,
    fix-ups: same answer as the whole matrix, squares crossing rank bounds."""
    from paper_2503_18974_b200.distributed import GpuBackend, decode_key, slice_rows
    rng = np.random.default_rng(100 + world)
    for it in range(3):
        rows, cols = world * 2048, 8192 + 32 * int(rng.integers(0, 64))
        a = (rng.random((rows, cols)) < 0.999).astype(np.uint8)
        k = int(rng.integers(100, 200))
        r0k = 2048 - k // 2  # crosses the first rank boundary
        c0k = int(rng.integers(0, cols - k))
        a[r0k:r0k + k, c0k:c0k + k] = 1
        full = grid.pack_bits(a).view(np.int32)
        rank_rows = [slice_rows(rows, world, q)[1] for q in range(world)]
        bes, srcs = [], []
        for q in range(world):
            r0, n = slice_rows(rows, world, q)
            srcs.append(torch.from_numpy(np.ascontiguousarray(full[r0:r0 + n])).cuda())
            bes.append(GpuBackend(N.FMT_BITS, n, cols, r0))
        for be, src in zip(bes, srcs):
            be.seed(src)
        best = torch.stack([be.best_side().clone() for be in bes]).max()
        for be, src in zip(bes, srcs):
            be.best_side().copy_(best.reshape(1))
            be.band_pass(src)
        gathered = torch.stack([be.rank_summary().clone() for be in bes])
        keys = []
        for q, be in enumerate(bes):
            base = be.compose(gathered, rank_rows, q) if q > 0 else None
            be.fixup(base)
            keys.append(be.key_status())
        ks = torch.stack(keys).max(dim=0).values.cpu().numpy()
        _same(decode_key(int(ks[0]), int(ks[1]), rows, cols), oracle.freq(a))


def test_team_engine_row_bands(torch):
    """Single matrices with cols <= 1024 on the team engine's row-band mode
    (a team per band, carry scan + fix-up): tall shapes, squares crossing band
    boundaries, strides, both formats."""
    rng = np.random.default_rng(33)
    for it in range(40):
        rows = int(rng.integers(128, 6000))
        cols = int(rng.integers(200, 1025))
        p = float(rng.choice([0.5, 0.9, 0.99, 0.999, 1.0]))
        k = int(rng.integers(0, min(rows, cols) + 1))
        a = _planted(rng, rows, cols, p, k)
        want = oracle.freq(a)
        pad = int(rng.choice([0, 16]))
        wide = np.zeros((rows, cols + pad), np.uint8)
        wide[:, :cols] = a
        s = Solver(N.FMT_U8, rows, cols, ld=cols + pad)
        assert int(s.plan.engine) == 1 and s.nbands > 1
        _same(s.solve(torch.from_numpy(wide).cuda())[0], want)
        w = grid.pack_bits(a)
        _same(Solver(N.FMT_BITS, rows, cols, ld=w.shape[1]).solve(torch.from_numpy(w.view(np.int32)).cuda())[0], want)


def test_fixup_climb_large_squares(torch):
    """Squares far taller than a band: the fix-up climbs one side per depth;
    the speculative last-depth test of a climbing tile must keep the exact
    side and location (ties included), for every band count."""
    rng = np.random.default_rng(44)
    for it in range(16):
        rows, cols = int(rng.integers(800, 3000)), int(rng.integers(800, 3000))
        a = (rng.random((rows, cols)) < float(rng.choice([0.9, 0.97, 0.995]))).astype(np.uint8)
        k = int(rng.integers(200, min(rows, cols)))
        t0, l0 = int(rng.integers(0, rows - k + 1)), int(rng.integers(0, cols - k + 1))
        a[t0:t0 + k, l0:l0 + k] = 1
        if it % 3 == 0:  # an equal square elsewhere: the first one in row-major order wins
            t1, l1 = int(rng.integers(0, rows - k + 1)), int(rng.integers(0, cols - k + 1))
            a[t1:t1 + k, l1:l1 + k] = 1
        want = oracle.freq(a)
        nb = int(rng.integers(2, 60))
        _same(Solver(N.FMT_U8, rows, cols, nbands=nb).solve(torch.from_numpy(a).cuda())[0], want)
        w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
        _same(Solver(N.FMT_BITS, rows, cols, nbands=nb).solve(w)[0], want)
        _same(Solver(N.FMT_U8, rows, cols, nbands=nb, deterministic=True).solve(torch.from_numpy(a).cuda())[0], want)
