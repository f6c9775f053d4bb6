"""Golden vectors for the cube extension, made by importing the
reference (this container only; the GPU box never reads /root/reference):

  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cube_golden.py

Records max_cube(v) = (side, volume_visited) (cubes.py:105-125) for
  * the all-2x2x2 enumeration (tests/test_cubes.py:119-126),
  * the seeded stream of tests/test_cubes.py:129-136 (random.Random(17)),
  * larger seeded volumes with planted cubes (specs + planted boxes recorded).
Output: tests/golden/cubes.json.
"""
import itertools
import json
import os
import random

from squarelab.cubes import max_cube
from squarelab.grid import BinaryMatrix, BinaryVolume, GenSpec, generate_volume

HERE = os.path.dirname(os.path.abspath(__file__))


def vol_from_bits(d, r, c, bits):
    return BinaryVolume(d, r, c, bytes(bits))


def main():
    out = {"enum2": [], "seeded": [], "planted": []}
    for bits in itertools.product((0, 1), repeat=8):
        v = vol_from_bits(2, 2, 2, bits)
        res = max_cube(v)
        out["enum2"].append([res.side, res.volume_visited])
    rng = random.Random(17)
    for _ in range(150):
        d, r, c = rng.randint(1, 6), rng.randint(1, 6), rng.randint(1, 6)
        dens, seed = rng.random(), rng.getrandbits(32)
        res = max_cube(generate_volume(GenSpec(r, c, dens, seed, depth=d)))
        out["seeded"].append({"spec": [r, c, dens, seed, d], "side": res.side, "visited": res.volume_visited})
    prng = random.Random(2503)
    for _ in range(24):
        d, r, c = prng.randint(4, 28), prng.randint(4, 40), prng.randint(4, 70)
        dens, seed = prng.choice([0.6, 0.8, 0.9, 0.97]), prng.getrandbits(32)
        v = generate_volume(GenSpec(r, c, dens, seed, depth=d))
        k = prng.randint(1, min(d, r, c))
        z0, y0, x0 = prng.randint(0, d - k), prng.randint(0, r - k), prng.randint(0, c - k)
        cells = bytearray(v.cells)
        for z in range(z0, z0 + k):
            for y in range(y0, y0 + k):
                for x in range(x0, x0 + k):
                    cells[(z * r + y) * c + x] = 1
        res = max_cube(BinaryVolume(d, r, c, bytes(cells)))
        out["planted"].append({"spec": [r, c, dens, seed, d], "box": [z0, y0, x0, k],
                               "side": res.side, "visited": res.volume_visited})
    with open(os.path.join(HERE, "cubes.json"), "w") as f:
        json.dump(out, f)
    print(len(out["enum2"]), len(out["seeded"]), len(out["planted"]))


if __name__ == "__main__":
    main()
