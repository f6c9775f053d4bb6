"""Time one config's solve (msq_launch) under plan variants; print answer, ms and the seeded best side.
usage: python tools/time_variants.py cfg5 [variant ...]   variant: noseed | floor=K | nostrip | climb"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import Solver
build.build()
cfg = sys.argv[1]
src = {"cfg3": configs.cfg3_device, "cfg4": configs.cfg4_device, "cfg5": configs.cfg5_device}[cfg]()
fmt = N.FMT_BITS if cfg == "cfg4" else N.FMT_U8
spec = configs.CONFIGS[cfg]
for v in ["base"] + sys.argv[2:]:
    kw = {"flags": 0}
    for part in v.split("+"):
        if part == "noseed":
            kw["flags"] |= N.PLAN_NO_SEED
        elif part == "nostrip":
            kw["flags"] |= N.PLAN_NO_STRIP
        elif part == "climb":
            kw["flags"] |= N.PLAN_CLIMB_FIXUP
        elif part.startswith("floor="):
            kw["test_floor"] = int(part[6:])
    s = Solver(fmt, spec["rows"], spec["cols"], **kw)
    for _ in range(3):
        s.launch(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        s.launch(src)
    e1.record()
    torch.cuda.synchronize()
    r = s.result()[0]
    print(cfg, v, round(e0.elapsed_time(e1) / 20, 4), "ms", (r.side, r.top, r.left), flush=True)
