"""Per-phase cycle breakdown of pass 1 (clock64 in thread 0 of every band CTA)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_18974_b200 import _native as N  # noqa: E402
from paper_2503_18974_b200 import build, configs  # noqa: E402
from paper_2503_18974_b200.squares import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
build.build()
spec = configs.CONFIGS[cfg]
src = {"cfg4": lambda: configs.cfg4_device(), "cfg5": lambda: configs.cfg5_device(),
       "cfg3": lambda: configs.cfg3_device()}[cfg]()
fmt = N.FMT_BITS if cfg == "cfg4" else N.FMT_U8
s = Solver(fmt, spec["rows"], spec["cols"])
units = s.nbands
buf = torch.zeros(units * 16, dtype=torch.int64, device="cuda")
s.solve(src)
N.load().msq_debug_set_profile(ctypes.c_void_p(buf.data_ptr()))
r = s.solve(src)
N.load().msq_debug_set_profile(None)
torch.cuda.synchronize()
pc = buf.cpu().numpy().reshape(units, 16).astype(np.float64)
names = ["A(work+waits)", "barrierA", "tma issue", "B climb", "maxwarp C", "B modeL", "C", "L rounds",
         "tiles climb", "maxwarp Cend->barA", "issuer TMA total", "raises", "maxwarp rowloop", "L max work", "maxwarp Cend->rowloop", "L max scan"]
tot = pc[:, [0, 1, 2, 3, 5, 6]].sum(axis=1)
print(cfg, r[0], "bands", units)
print("total cycles per band: mean %.0f max %.0f" % (tot.mean(), tot.max()))
for i, n in enumerate(names):
    if n == "-":
        continue
    col = pc[:, i]
    extra = f" ({100 * col.mean() / tot.mean():5.1f}%)" if i < 7 else ""
    print(f"{n:16s} mean {col.mean():12.1f} max {col.max():12.0f}{extra}")
