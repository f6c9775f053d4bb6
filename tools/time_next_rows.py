"""Timing of the SURVEY §8(f) rows on the GPU (device events; CPU oracle beside where cheap).

F1 campaigns (exhaustive 4x4, random 10k x 64^2), F2 text ingest (GB/s of text),
F3 max_cube (a 64 x 512 x 512 volume with a planted 40-cube), F4 maximal
rectangle (4096^2).  Prints one JSON line per row."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2503_18974_b200 import build
build.build()
from paper_2503_18974_b200 import cubes, histogram, ingest, verify  # noqa: E402


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


out = []
t = ev_time(lambda: verify.exhaustive_sweep(4, 4), 2)
out.append({"row": "F1 exhaustive_sweep(4,4)", "cases": 74954, "s": t, "cases_per_s": 74954 / t})
t = ev_time(lambda: verify.random_campaign(10000, 64, {0.3, 0.5, 0.7, 0.9, 0.99}, 0), 2)
out.append({"row": "F1 random_campaign(10000, 64)", "cases": 10000, "s": t, "cases_per_s": 10000 / t,
            "note": "includes host-side generation of the 10k matrices (reference generator)"})

rng = np.random.default_rng(1)
a = (rng.random((8192, 8192)) < 0.99).astype(np.uint8)
text = "\n".join("".join(map(str, row)) for row in a[:, :]) + "\n"
raw = text.encode()
d_text = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
import ctypes
from paper_2503_18974_b200 import _native as N
words = torch.empty((8192, 256), dtype=torch.int32, device="cuda")
bad = ctypes.c_int64()
lib = N.load()
def parse():
    N.check(lib.msq_parse_text(ctypes.c_void_p(d_text.data_ptr()), len(raw), 8192, 8192, N.FMT_BITS,
                               ctypes.c_void_p(words.data_ptr()), 256, ctypes.byref(bad), None))
t = ev_time(parse, 10)
out.append({"row": "F2 msq_parse_text 8192^2 -> bits (device text)", "bytes": len(raw), "s": t,
            "GB_per_s": len(raw) / t / 1e9})
t = ev_time(lambda: ingest.freq_square_text(raw), 3)
out.append({"row": "F2 freq_square_text 8192^2 (host text: H2D + parse + solve)", "s": t,
            "Gcells_per_s": 8192 * 8192 / t / 1e9})

v = (rng.random((64, 512, 512)) < 0.97).astype(np.uint8)
v[10:50, 100:140, 200:240] = 1
dv = torch.from_numpy(v).cuda()
r = cubes.max_cube(dv)
t = ev_time(lambda: cubes.max_cube(dv), 3)
out.append({"row": "F3 max_cube 64x512x512", "side": r.side, "volume_visited": r.volume_visited, "s": t,
            "Gvoxels_read_per_s": r.volume_visited / t / 1e9})

m = torch.from_numpy((rng.random((4096, 4096)) < 0.95).astype(np.uint8)).cuda()
rr = histogram.maximal_rectangle(m)
t = ev_time(lambda: histogram.maximal_rectangle(m), 3)
out.append({"row": "F4 maximal_rectangle 4096^2", "area": rr.area, "s": t, "Gcells_per_s": 4096 * 4096 / t / 1e9})
for o in out:
    print(json.dumps(o), flush=True)
