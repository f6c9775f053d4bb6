"""Experiment: u8 configs solved directly (u8 bands) vs packed to bits first (bits bands)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import Solver
build.build()

def pack(u8):
    r, c = u8.shape
    w = (c + 31) // 32
    pad = torch.zeros((r, w * 32), dtype=torch.uint8, device=u8.device)
    pad[:, :c] = u8
    bits = pad.view(r, w, 32).to(torch.int64)
    sh = torch.arange(32, device=u8.device, dtype=torch.int64)
    return ((bits << sh).sum(dim=2)).to(torch.int64).bitwise_and(0xFFFFFFFF).to(torch.uint32).view(torch.int32).contiguous()

def timeit(s, src, n=10):
    for _ in range(2): s.launch(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): s.launch(src)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, s.result()[0]

for cfg in ("cfg3", "cfg5"):
    src = configs.cfg3_device() if cfg == "cfg3" else configs.cfg5_device()
    r, c = src.shape
    t_u8, a = timeit(Solver(N.FMT_U8, r, c), src)
    w = pack(src)
    t_bits, b = timeit(Solver(N.FMT_BITS, r, c), w)
    print(cfg, "u8 %.4f ms" % t_u8, a, "| bits %.4f ms" % t_bits, b, "| zero fraction %.3f" % (1 - src.float().mean().item()), flush=True)
