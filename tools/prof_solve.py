"""Run one config solve (generation + 2 solves) -- the command profiled under ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_18974_b200 import _native as N  # noqa: E402
from paper_2503_18974_b200 import build, configs  # noqa: E402
from paper_2503_18974_b200.squares import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
build.build()
spec = configs.CONFIGS[cfg]
if cfg in ("cfg4_p99", "cfg4_planted"):
    src, fmt = configs.cfg4_variant_device(cfg), N.FMT_BITS
elif cfg == "cfg4":
    src, fmt = configs.cfg4_device(), N.FMT_BITS
elif cfg == "cfg5":
    src, fmt = configs.cfg5_device(), N.FMT_U8
elif cfg == "cfg3":
    src, fmt = configs.cfg3_device(), N.FMT_U8
elif cfg == "cfg2":
    src, fmt = torch.from_numpy(configs.cfg2_array()).cuda(), N.FMT_U8
else:
    src, fmt = torch.from_numpy(configs.cfg1_array()).cuda(), N.FMT_U8
s = Solver(fmt, spec["rows"], spec["cols"], batch=spec["batch"])
for _ in range(2):
    r = s.solve(src)
torch.cuda.synchronize()
print(cfg, r[0])
