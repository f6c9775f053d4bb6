"""Time msq_launch for small single matrices with each engine (MSQ_ENGINE=0/1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import Solver
build.build()
for rows, cols, fmt in ((512, 512, N.FMT_U8), (256, 256, N.FMT_U8), (1024, 1024, N.FMT_U8), (2000, 1000, N.FMT_U8),
                        (1024, 1024, N.FMT_BITS)):
    a = (np.random.default_rng(0).random((rows, cols)) < 0.7).astype(np.uint8)
    src = torch.from_numpy(a).cuda() if fmt == N.FMT_U8 else torch.from_numpy(
        __import__("paper_2503_18974_b200.grid", fromlist=["x"]).pack_bits(a).view(np.int32)).cuda()
    out = []
    for eng in ("0", "1"):
        os.environ["MSQ_ENGINE"] = eng
        s = Solver(fmt, rows, cols)
        for _ in range(5):
            s.launch(src)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            s.launch(src)
        e1.record()
        torch.cuda.synchronize()
        out.append((eng, int(s.plan.engine), round(e0.elapsed_time(e1) / 200 * 1000, 1), s.result()[0]))
    print(rows, cols, "bits" if fmt else "u8", out, flush=True)
