"""cfg3 / cfg5 solve time with and without the lower-bound seed (MSQ_NO_SEED=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import Solver
build.build()
for cfg in ("cfg3", "cfg5"):
    src = configs.cfg3_device() if cfg == "cfg3" else configs.cfg5_device()
    r, c = src.shape
    for env in ("0", "1"):
        os.environ["MSQ_NO_SEED"] = env
        s = Solver(N.FMT_U8, r, c)
        for _ in range(2): s.launch(src)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): s.launch(src)
        e1.record(); torch.cuda.synchronize()
        print(cfg, "no_seed" if env == "1" else "seed", round(e0.elapsed_time(e1) / 10, 4), "ms", s.result()[0], flush=True)
