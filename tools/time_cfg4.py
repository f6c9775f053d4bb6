"""Time the cfg4 solve (msq_launch) under plan variants (flags / test floor); print answer + ms."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import Solver
build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
src = configs.cfg4_device() if cfg == "cfg4" else configs.cfg5_device()
fmt = N.FMT_BITS if cfg == "cfg4" else N.FMT_U8
spec = configs.CONFIGS[cfg]
VARIANTS = ({"flags": N.PLAN_NO_STRIP}, {}, {"test_floor": 100}, {"test_floor": 120}, {"test_floor": 133},
            {"test_floor": 96, "flags": N.PLAN_NO_SEED}, {"test_floor": 120, "flags": N.PLAN_NO_SEED},
            {"test_floor": 133, "flags": N.PLAN_NO_SEED})
for env in VARIANTS:
    s = Solver(fmt, spec["rows"], spec["cols"], **env)
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
    host = s.res.cpu().numpy().view("int32")
    print(env, round(e0.elapsed_time(e1) / 20, 4), "ms", (r.side, r.top, r.left), "best_side", host[5], flush=True)
