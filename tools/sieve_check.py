"""Sieve engine on the GPU: random cases against the oracle, then cfg4 timing
(streaming pass alone and whole solve).  usage: sieve_check.py [quick|cfg4|all] [wpc]"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2503_18974_b200 import _native as N  # noqa: E402
from paper_2503_18974_b200 import build, configs, grid  # noqa: E402
from paper_2503_18974_b200.distributed import GpuBackend  # noqa: E402
from paper_2503_18974_b200.squares import Solver  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "all"
build.build()
oracle.build()
lib = N.load()
if len(sys.argv) > 2:
    lib.msq_debug_set_sieve_wpc(int(sys.argv[2]))


def random_cases():
    rng = np.random.default_rng(7)
    bad = 0
    stats = {"decided": 0, "retried": 0}
    for it in range(60):
        rows = int(rng.integers(64, 2600))
        cols = 128 * int(rng.integers(1, 28))
        p = [0.999, 0.9995, 0.998, 0.9999, 0.995][it % 5]
        a = (rng.random((rows, cols)) < p).astype(np.uint8)
        k = int(rng.integers(40, 250))
        if it % 4 != 3 and min(rows, cols) > k:  # planted square around the decidable range
            top, left = int(rng.integers(0, rows - k + 1)), int(rng.integers(0, cols - k + 1))
            a[top:top + k, left:left + k] = 1
        want = oracle.freq(a)
        w = torch.from_numpy(grid.pack_bits(a).view(np.int32)).cuda()
        s = Solver(N.FMT_BITS, rows, cols, engine=2)
        got = s.solve(w)[0]
        retried = getattr(s, "sieve_retries", 0)
        stats["retried" if retried else "decided"] += 1
        ok = (got.side, got.top, got.left) == (want.side, want.top, want.left)
        if not ok:
            bad += 1
        print(f"case {it}: {rows}x{cols} p={p} planted={k if it % 4 != 3 else 0} want=({want.side},{want.top},{want.left}) "
              f"got=({got.side},{got.top},{got.left}) retried={retried} {'ok' if ok else 'MISMATCH'}", flush=True)
    print("random cases:", stats, "mismatches:", bad, flush=True)
    return bad


def time_cfg4():
    src = configs.cfg4_device()
    rows = cols = 65536
    be = GpuBackend(N.FMT_BITS, rows, cols, 0)
    print("plan engine", int(be.plan.engine), "sv_bands", int(be.plan.sv_bands), "ws MB", int(be.plan.ws_bytes) >> 20, flush=True)
    for _ in range(3):
        be.sieve(src)
    torch.cuda.synchronize()
    ks = be.key_status().cpu().numpy()
    res = be.res.cpu().numpy()
    print("key/status", ks, "best_side", res.view(np.int32)[5], flush=True)
    from paper_2503_18974_b200.distributed import decode_key
    print("answer", decode_key(int(ks[0]), 0, rows, cols), "status", int(ks[1]), flush=True)
    ctl = be.ws[int(be.plan.sv_ws_off):int(be.plan.sv_ws_off) + 16].cpu().numpy().view(np.int32)
    print("ctl best/count/abort", ctl[:3], flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        be.sieve(src)
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / n
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        be.sieve_pass(src)
        b.record()
        be.sieve_finish(src)
        ts.append((a, b))
    torch.cuda.synchronize()
    p1 = sum(a.elapsed_time(b) for a, b in ts) / n
    gb = rows * cols / 8 / 1e9
    print(json.dumps({"cfg4_step_ms": round(step, 4), "pass_ms": round(p1, 4), "pass_GBs": round(gb / (p1 * 1e-3), 1),
                      "Gcells_s": round(rows * cols / (step * 1e-3) / 1e9, 1)}), flush=True)


bad = 0
if mode in ("quick", "all"):
    bad = random_cases()
if mode in ("cfg4", "all"):
    time_cfg4()
sys.exit(1 if bad else 0)
