"""Device time of one rank's sieve solve on an 8192-row slice of cfg4 (+ 256-row halo) for forced sweep
counts (msq_debug_set_sieve_phases): is overlapping the coarse pass worth it on short slices?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.distributed import GpuBackend
build.build()
lib = N.load()
full = configs.cfg4_device()
for rows in (8192, 16384, 32768):
    src = full[rows:2 * rows].contiguous()
    halo = full[rows - 256:rows].contiguous()
    for ph in (0, 1, 2, 3, 4):
        lib.msq_debug_set_sieve_phases(ph)
        be = GpuBackend(N.FMT_BITS, rows, 65536, rows)
        for _ in range(3):
            be.sieve(src, halo)
        torch.cuda.synchronize()
        torch.cuda._sleep(4_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            be.sieve(src, halo)
        b.record()
        torch.cuda.synchronize()
        print(rows, "phases", ph, round(a.elapsed_time(b) / 50, 4), "ms", be.key_status().cpu().numpy(), flush=True)
lib.msq_debug_set_sieve_phases(0)
