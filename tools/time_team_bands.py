"""Latency of single small matrices on the team engine's row bands, by band height."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import Solver
import oracle
build.build()
lib = N.load()
rng = np.random.default_rng(0)
shapes = [("cfg1", configs.cfg1_array())]
for r, c in [(1024, 1024), (2000, 1000), (4096, 512), (600, 300)]:
    shapes.append((f"{r}x{c}", (rng.random((r, c)) < 0.9).astype(np.uint8)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, a in shapes:
    src = torch.from_numpy(a).cuda()
    want = oracle.freq(a)
    for hb in (64, 32, 16, 8, 4):
        lib.msq_debug_set_team_band_rows(hb)
        s = Solver(N.FMT_U8, a.shape[0], a.shape[1])
        got = s.solve(src)[0]
        ok = (got.side, got.top, got.left) == (want.side, want.top, want.left)
        ts = []
        for _ in range(30):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); s.launch(src); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(name, "band_rows", hb, "nbands", s.nbands, "engine", s.plan.engine, round(float(np.median(ts)), 4), "ms", "ok" if ok else "MISMATCH", flush=True)
