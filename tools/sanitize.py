"""Small invocations of every kernel family, run under compute-sanitizer
(memcheck / racecheck / synccheck) by tools/gpu_r2_sanitize.sh."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_18974_b200 import _native as N, build, configs, grid
from paper_2503_18974_b200.squares import Solver, freq_square, solve_batch, dp_full, brute_force_square, freq_square_traced
from paper_2503_18974_b200 import ingest, histogram, cubes
import oracle

build.build()
rng = np.random.default_rng(5)
checks = []
# cfg1 (team row bands + carry + window-search fix-up)
r = freq_square(grid.generate_matrix(grid.GenSpec(512, 512, 0.7, 0)))
checks.append(("cfg1", (r.side, r.top, r.left) == (5, 0, 67)))
# exhaustive 3x4 batch (team engine, sub-warp teams)
pats = np.arange(2 ** 12, dtype=np.int64)
cells = ((pats[:, None] >> np.arange(11, -1, -1)) & 1).astype(np.uint8).reshape(-1, 3, 4)
got = solve_batch(cells)
checks.append(("batch3x4", [g.side for g in got] == [w.side for w in oracle.freq_batch(cells)]))
# u8 strip pass + fix-up (several bands)
a = (rng.random((1200, 4096)) < 0.97).astype(np.uint8)
a[300:520, 1000:1220] = 1
w = oracle.freq(a)
g = Solver(N.FMT_U8, 1200, 4096, nbands=12).solve(torch.from_numpy(a).cuda())[0]
checks.append(("ustrip", (g.side, g.top, g.left) == (w.side, w.top, w.left)))
# bits strip pass with a test floor (strip kernel) and its hand-back
b = (rng.random((1600, 8192)) < 0.999).astype(np.uint8)
b[100:260, 4000:4160] = 1
wb = oracle.freq(b)
src = torch.from_numpy(grid.pack_bits(b).view(np.int32)).cuda()
g = Solver(N.FMT_BITS, 1600, 8192, nbands=10, test_floor=120).solve(src)[0]
checks.append(("strip_bits", (g.side, g.top, g.left) == (wb.side, wb.top, wb.left)))
g = Solver(N.FMT_BITS, 1600, 8192, nbands=10, flags=N.PLAN_CLIMB_FIXUP).solve(src)[0]
checks.append(("pass1_bits_climb", (g.side, g.top, g.left) == (wb.side, wb.top, wb.left)))
# sieve engine (streaming pass, coarse pass beside it, verifier) incl. a halo and an undecided input
sv = (rng.random((1300, 4096)) < 0.9993).astype(np.uint8)
sv[640:790, 1000:1150] = 1
wsv = oracle.freq(sv)
g = Solver(N.FMT_BITS, 1300, 4096, engine=2).solve(torch.from_numpy(grid.pack_bits(sv).view(np.int32)).cuda())[0]
checks.append(("sieve", (g.side, g.top, g.left) == (wsv.side, wsv.top, wsv.left)))
dense = (rng.random((1300, 4096)) < 0.95).astype(np.uint8)
wd = oracle.freq(dense)
sd = Solver(N.FMT_BITS, 1300, 4096, engine=2)
g = sd.solve(torch.from_numpy(grid.pack_bits(dense).view(np.int32)).cuda())[0]
checks.append(("sieve_undecided_retry", (g.side, g.top, g.left) == (wd.side, wd.top, wd.left) and sd.sieve_retries == 1))
# team engine row-band mode (single matrix, <= 1024 columns)
c = (rng.random((2000, 1000)) < 0.9).astype(np.uint8)
wc = oracle.freq(c)
g = freq_square(torch.from_numpy(c).cuda())
checks.append(("team_rowbands", (g.side, g.top, g.left) == (wc.side, wc.top, wc.left)))
# DP kernel, brute force, traced
d = (rng.random((300, 700)) < 0.9).astype(np.uint8)
wd = oracle.freq(d)
g = dp_full(torch.from_numpy(d).cuda())
checks.append(("dp", (g.side, g.top, g.left) == (wd.side, wd.top, wd.left)))
m = grid.generate_matrix(grid.GenSpec(60, 70, 0.8, 3))
checks.append(("brute", brute_force_square(m).side == freq_square(m).side))
checks.append(("traced", freq_square_traced(m)[0].side == freq_square(m).side))
# text ingest
txt = grid.serialize_matrix(grid.generate_matrix(grid.GenSpec(300, 257, 0.8, 4)))
checks.append(("ingest", ingest.freq_square_text(txt).side == freq_square(grid.parse_matrix(txt)).side))
# histogram rectangle, cube probe
h = (rng.random((200, 300)) < 0.8).astype(np.uint8)
checks.append(("histogram", histogram.maximal_rectangle(h) is not None))
v = (rng.random((8, 64, 64)) < 0.95).astype(np.uint8)
checks.append(("cube", cubes.max_cube(v) is not None))
torch.cuda.synchronize()
for name, ok in checks:
    print(name, "ok" if ok else "MISMATCH")
print("ALL", "ok" if all(ok for _, ok in checks) else "FAIL")
