"""e2e of freq_square_bits on a pageable 512 MiB cfg4 array under staging shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.squares import freq_square_bits
build.build()
host = np.array(configs.cfg4_device().cpu().numpy().view(np.uint32), copy=True)
lib = N.load()
print("cores", os.cpu_count(), flush=True)
for w, b, mb in [(8, 2, 8), (8, 3, 8), (8, 4, 4), (12, 3, 4), (16, 3, 4), (16, 2, 8), (12, 2, 16), (6, 3, 8), (16, 4, 2), (4, 4, 16)]:
    lib.msq_debug_set_staging(w, b, mb << 20)
    freq_square_bits(host, 65536)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        r = freq_square_bits(host, 65536)
    dt = (time.perf_counter() - t0) / 5
    print(w, b, mb, round(dt * 1e3, 2), "ms", round(host.nbytes / dt / 1e9, 1), "GB/s", r.side, flush=True)
# pinned reference
pin = torch.from_numpy(host).pin_memory()
t0 = time.perf_counter()
for _ in range(5):
    d = pin.cuda(non_blocking=True)
    torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print("pinned H2D", round(dt * 1e3, 2), "ms", round(host.nbytes / dt / 1e9, 1), "GB/s", flush=True)
