"""Golden vectors for the histogram maximal rectangle, made by
importing the reference in this container:

  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_hist_golden.py

maximal_rectangle(m) = (area, height, width) (histogram.py:60-70) on seeded
matrices of the reference generator (GenSpec rows, cols, density, seed).
Output: tests/golden/histogram.json.
"""
import json
import os
import random

from squarelab.grid import GenSpec, generate_matrix
from squarelab.histogram import maximal_rectangle

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = random.Random(70)
    out = []
    for _ in range(60):
        r, c = rng.randint(1, 90), rng.randint(1, 300)
        dens = rng.choice([0.3, 0.5, 0.7, 0.9, 0.97, 1.0])
        seed = rng.getrandbits(32)
        res = maximal_rectangle(generate_matrix(GenSpec(r, c, dens, seed)))
        out.append({"spec": [r, c, dens, seed], "rect": [res.area, res.height, res.width]})
    with open(os.path.join(HERE, "histogram.json"), "w") as f:
        json.dump(out, f)
    print(len(out))


if __name__ == "__main__":
    main()
