"""GPU-batched verification campaigns (paper_2503_18974_b200.verify).

CPU: the random case stream equals the reference's (verify.py:196-207) as
recorded in tests/golden/random_campaign.npz; the enumeration cap.
GPU: both campaigns run clean with the two GPU solvers (frequency algorithm and
the three-way-min DP), and their sides/locations equal the golden vectors."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
DENS = {0.3, 0.5, 0.7, 0.9, 0.99}


def test_campaign_stream_matches_reference_stream():
    from paper_2503_18974_b200.verify import campaign_specs
    rc = np.load(os.path.join(GOLDEN, "random_campaign.npz"))
    specs = campaign_specs(10_000, 64, DENS, 0)
    assert [s.rows for s in specs] == rc["rows"].tolist()
    assert [s.cols for s in specs] == rc["cols"].tolist()
    assert [s.density for s in specs] == rc["density"].tolist()
    assert [s.seed for s in specs] == [int(x) for x in rc["seed"]]


def test_enumeration_cap():
    from paper_2503_18974_b200.verify import EnumerationCapExceededError, exhaustive_sweep
    with pytest.raises(EnumerationCapExceededError):
        exhaustive_sweep(5, 5)


@pytest.fixture(scope="module")
def built():
    from paper_2503_18974_b200 import build
    build.build()


@pytest.mark.gpu
def test_exhaustive_sweep_4x4_gpu(built):
    from paper_2503_18974_b200.verify import exhaustive_sweep
    rep = exhaustive_sweep(4, 4)
    assert rep.clean, (rep.mismatches[:3], rep.invariant_failures[:3])
    assert rep.cases_run == 74_954
    assert rep.launches == 2 * 16  # one launch per shape and solver


@pytest.mark.gpu
def test_random_campaign_gpu_matches_golden(built):
    from paper_2503_18974_b200 import solve_batch, dp_batch
    from paper_2503_18974_b200.verify import campaign_specs, random_campaign
    rep = random_campaign(10_000, 64, DENS, 0)
    assert rep.clean, (rep.mismatches[:3], rep.invariant_failures[:3])
    assert rep.cases_run == 10_000 and rep.launches == 2
    # the DP solver alone against the golden sides/locations
    from paper_2503_18974_b200.grid import generate_matrix
    rc = np.load(os.path.join(GOLDEN, "random_campaign.npz"))
    specs = campaign_specs(10_000, 64, DENS, 0)
    stack = np.zeros((len(specs), 64, 64), np.uint8)
    for k, s in enumerate(specs):
        stack[k, :s.rows, :s.cols] = np.frombuffer(generate_matrix(s).cells, np.uint8).reshape(s.rows, s.cols)
    for name, res in (("dp", dp_batch(stack)), ("freq", solve_batch(stack))):
        assert [r.side for r in res] == rc["side"].tolist(), name
        assert [r.top for r in res] == rc["top"].tolist(), name
        assert [r.left for r in res] == rc["left"].tolist(), name


@pytest.mark.gpu
def test_dp_batch_invalid_and_wide(built):
    from paper_2503_18974_b200 import dp_batch
    import oracle
    rng = np.random.default_rng(5)
    cells = (rng.random((40, 90, 256)) < 0.9).astype(np.uint8)
    for got, want in zip(dp_batch(cells), oracle.freq_batch(cells)):
        assert (got.side, got.top, got.left) == (want.side, want.top, want.left)
    cells[3, 4, 5] = 7
    with pytest.raises(ValueError):
        dp_batch(cells)
