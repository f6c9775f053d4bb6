"""Per-warp timeline of 8 mode-L tiles of band 0 (debug trace written by
pass1_kernel when profiling is on): when each warp reaches each phase point,
relative to the tile start of warp 0."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_18974_b200 import _native as N  # noqa: E402
from paper_2503_18974_b200 import build, configs  # noqa: E402
from paper_2503_18974_b200.squares import Solver  # noqa: E402

build.build()
src = configs.cfg4_device()
spec = configs.CONFIGS["cfg4"]
s = Solver(N.FMT_BITS, spec["rows"], spec["cols"])
units = s.nbands
NW = 16
buf = torch.zeros(units * 16 + 8 * NW * 16, dtype=torch.int64, device="cuda")
s.solve(src)
N.load().msq_debug_set_profile(ctypes.c_void_p(buf.data_ptr()))
s.solve(src)
N.load().msq_debug_set_profile(None)
torch.cuda.synchronize()
tr = buf[units * 16:].cpu().numpy().reshape(8, NW, 16).astype(np.int64)
names = ["start", "rowloop", "preA", "postA", "tma", "scan", "check", "preB", "postB", "endB", "endC", "rows", "slotw", "Fdone", "Bexit"]
for t in range(8):
    base = tr[t, 0, 0]
    print(f"tile {40 + t}: (cycles from warp-0 tile start; '-' = not reached)")
    print("warp " + " ".join(f"{n:>7s}" for n in names))
    for w in range(NW):
        row = tr[t, w, :15]
        print(f"{w:4d} " + " ".join(f"{(v - base):7d}" if v else "      -" for v in row))
