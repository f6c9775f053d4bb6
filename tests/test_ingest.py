"""GPU text ingest (paper_2503_18974_b200.ingest) against the
reference's parser semantics (grid.py:172-206, mirrored by grid.parse_matrix)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2503_18974_b200 import build
    build.build()
    from paper_2503_18974_b200 import grid, ingest
    return grid, ingest


def _text(a, trailing=True):
    s = "\n".join("".join("1" if x else "0" for x in row) for row in a)
    return s + ("\n" if trailing else "")


def test_valid_texts_bits_and_u8(mods):
    grid, ingest = mods
    import oracle
    rng = np.random.default_rng(3)
    for it in range(40):
        rows = int(rng.integers(1, 120))
        cols = int(rng.choice([1, 5, 31, 32, 33, 100, 1000, 8191, 8192, 8193, 20000]))
        a = (rng.random((rows, cols)) < float(rng.choice([0.5, 0.9, 0.99]))).astype(np.uint8)
        t = _text(a, trailing=bool(it % 2))
        w, r, c = ingest.parse_matrix_device(t, "bits")
        assert (r, c) == (rows, cols)
        assert np.array_equal(w.cpu().numpy().view(np.uint32), grid.pack_bits(a))
        u, r, c = ingest.parse_matrix_device(t.encode(), "u8")
        assert np.array_equal(u.cpu().numpy(), a)
        got, want = ingest.freq_square_text(t), oracle.freq(a)
        assert (got.side, got.area, got.cells_visited, got.top, got.left) == (
            want.side, want.area, want.cells_visited, want.top, want.left)


@pytest.mark.parametrize("bad", [
    "0101\n011\n1111\n",         # short line
    "0101\n01011\n1111\n",       # long line
    "0101\n0101\n\n",            # blank last line
    "0101\n0121\n1111\n",        # invalid digit
    "0101\n0101\n11 1\n",        # space
    "0101\r\n0101\r\n",          # CRLF
    "01é1\n0101\n",              # non-ASCII, first line
    "0101\n0é01\n",              # non-ASCII, same length in characters
    "0101\n0101\n0101",          # fine (no trailing newline) -- control
])
def test_malformed_texts_raise_like_the_reference(mods, bad):
    grid, ingest = mods
    try:
        want = grid.parse_matrix(bad)
    except grid.MatrixParseError as e:
        with pytest.raises(type(e)) as got:
            ingest.parse_matrix_device(bad)
        assert str(got.value) == str(e)
        return
    w, r, c = ingest.parse_matrix_device(bad)
    assert (r, c) == (want.rows, want.cols)


def test_empty_and_newline_only(mods):
    grid, ingest = mods
    assert ingest.parse_matrix_device("")[1:] == (0, 0)
    r = ingest.freq_square_text("")
    assert (r.side, r.area, r.cells_visited) == (0, 0, 0)
