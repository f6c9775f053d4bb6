"""The cube oracle (oracle/cubes.py) pinned against the reference's own
max_cube outputs (tests/golden/cubes.json): side and volume_visited."""
import itertools
import json
import os

import numpy as np

from oracle import cubes as oc

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cubes.json")))


def _planted(e):
    r, c, dens, seed, d = e["spec"]
    v = oc.generate_volume(r, c, dens, seed, d).copy()
    z0, y0, x0, k = e["box"]
    v[z0:z0 + k, y0:y0 + k, x0:x0 + k] = 1
    return v


def test_enum_2x2x2():
    for bits, (side, visited) in zip(itertools.product((0, 1), repeat=8), G["enum2"]):
        assert oc.max_cube(np.array(bits, np.uint8).reshape(2, 2, 2)) == (side, visited)


def test_seeded_and_planted():
    for e in G["seeded"]:
        r, c, dens, seed, d = e["spec"]
        assert oc.max_cube(oc.generate_volume(r, c, dens, seed, d)) == (e["side"], e["visited"])
    for e in G["planted"][:8]:
        assert oc.max_cube(_planted(e)) == (e["side"], e["visited"])
