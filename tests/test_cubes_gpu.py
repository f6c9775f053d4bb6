"""GPU cube extension (paper_2503_18974_b200.cubes) against the
reference's max_cube outputs (tests/golden/cubes.json) and the cube oracle."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import cubes as oc

pytestmark = pytest.mark.gpu
G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cubes.json")))


@pytest.fixture(scope="module")
def cubes():
    from paper_2503_18974_b200 import build
    build.build()
    from paper_2503_18974_b200 import cubes as c
    return c


def test_golden(cubes):
    for bits, (side, visited) in zip(itertools.product((0, 1), repeat=8), G["enum2"]):
        r = cubes.max_cube(np.array(bits, np.uint8).reshape(2, 2, 2))
        assert (r.side, r.volume_visited) == (side, visited), bits
    for e in G["seeded"]:
        rr, c, dens, seed, d = e["spec"]
        r = cubes.max_cube(oc.generate_volume(rr, c, dens, seed, d))
        assert (r.side, r.volume_visited) == (e["side"], e["visited"]), e
    for e in G["planted"]:
        rr, c, dens, seed, d = e["spec"]
        v = oc.generate_volume(rr, c, dens, seed, d).copy()
        z0, y0, x0, k = e["box"]
        v[z0:z0 + k, y0:y0 + k, x0:x0 + k] = 1
        r = cubes.max_cube(v)
        assert (r.side, r.volume_visited) == (e["side"], e["visited"]), e


def test_larger_volumes_vs_oracle(cubes):
    rng = np.random.default_rng(11)
    for it in range(6):
        d, r, c = int(rng.integers(20, 48)), int(rng.integers(30, 300)), int(rng.integers(30, 1500))
        v = (rng.random((d, r, c)) < 0.9).astype(np.uint8)
        k = int(rng.integers(3, min(d, r, c)))
        z0, y0, x0 = (int(rng.integers(0, n - k + 1)) for n in (d, r, c))
        v[z0:z0 + k, y0:y0 + k, x0:x0 + k] = 1
        got = cubes.max_cube(v)
        assert (got.side, got.volume_visited) == oc.max_cube(v)


def test_invalid_voxel_and_empty(cubes):
    v = np.ones((3, 4, 5), np.uint8)
    v[1, 2, 3] = 2
    with pytest.raises(ValueError):
        cubes.max_cube(v)
    assert cubes.max_cube(np.zeros((0, 0, 0), np.uint8)) == cubes.CubeResult(0, 0)
