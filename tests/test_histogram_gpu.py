"""GPU histogram maximal rectangle against the reference's
outputs (tests/golden/histogram.json) and the histogram oracle."""
import json
import os

import numpy as np
import pytest

from oracle import histogram as oh

pytestmark = pytest.mark.gpu
G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "histogram.json")))


@pytest.fixture(scope="module")
def hist():
    from paper_2503_18974_b200 import build
    build.build()
    from paper_2503_18974_b200 import histogram as h
    return h


def test_golden(hist):
    from paper_2503_18974_b200.grid import GenSpec, generate_matrix
    for e in G:
        r, c, dens, seed = e["spec"]
        got = hist.maximal_rectangle(generate_matrix(GenSpec(r, c, dens, seed)))
        assert [got.area, got.height, got.width] == e["rect"], e


def test_random_vs_oracle(hist):
    rng = np.random.default_rng(8)
    for it in range(25):
        r, c = int(rng.integers(1, 400)), int(rng.integers(1, 3000))
        a = (rng.random((r, c)) < float(rng.choice([0.5, 0.9, 0.99, 1.0]))).astype(np.uint8)
        got = hist.maximal_rectangle(a)
        assert (got.area, got.height, got.width) == oh.maximal_rectangle(a), it


def test_edges(hist):
    assert hist.maximal_rectangle(np.zeros((0, 0), np.uint8)) == hist.RectResult(0, 0, 0)
    assert hist.maximal_rectangle(np.zeros((5, 7), np.uint8)) == hist.RectResult(0, 0, 0)
    assert hist.maximal_rectangle(np.ones((5, 7), np.uint8)) == hist.RectResult(35, 5, 7)
    a = np.ones((4, 4), np.uint8)
    a[1, 1] = 9
    with pytest.raises(ValueError):
        hist.maximal_rectangle(a)
