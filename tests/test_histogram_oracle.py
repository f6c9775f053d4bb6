"""The histogram oracle pinned against the reference's maximal_rectangle outputs."""
import json
import os

from oracle import histogram as oh
from paper_2503_18974_b200.grid import GenSpec, generate_array

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "histogram.json")))


def test_golden():
    for e in G:
        r, c, dens, seed = e["spec"]
        assert list(oh.maximal_rectangle(generate_array(GenSpec(r, c, dens, seed)))) == e["rect"]


def test_kats():
    assert oh.largest_rect([2, 1, 5, 6, 2, 3]) == (10, 5, 2)
    assert oh.largest_rect([]) == (0, 0, 0)
    assert oh.largest_rect([3, 3, 3]) == (9, 3, 3)
