"""Row-band sharding logic under gloo (world sizes 2, 3 and 4, CPU, no GPU).

RowBandSolver (paper_2503_18974_b200/distributed.py) runs the same exchange it
runs over NCCL on the GPU box -- all-gather of per-rank bottom runs, carry
composition, key all-reduce -- with the per-rank steps done by the oracle
(tests/cpu_band_backend.py).  The answer must equal Algorithm 1 on the whole
matrix (side and location), including squares that cross rank boundaries and
columns that are all ones across whole ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2503_18974_b200 import grid


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cases():
    rng = np.random.default_rng(123)
    cases = []
    for it in range(12):
        rows = int(rng.integers(6, 120))
        cols = int(rng.integers(1, 90))
        p = [0.7, 0.95, 0.99, 1.0][it % 4]
        a = (rng.random((rows, cols)) < p).astype(np.uint8)
        if it % 3 == 0 and min(rows, cols) >= 8:  # square straddling the middle rows
            k = min(rows, cols) * 2 // 3
            top = max(0, rows // 2 - k // 2)
            a[top:top + k, :k] = 1
        cases.append(a)
    return cases


def _worker(rank, world, port, fmt, results):
    import torch.distributed as dist

    from cpu_band_backend import CpuBandBackend
    from paper_2503_18974_b200.distributed import RowBandSolver, slice_rows
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    out = []
    for a in _cases():
        rows, cols = a.shape
        r0, n = slice_rows(rows, world, rank)
        local = a[r0:r0 + n] if fmt == 0 else grid.pack_bits(a[r0:r0 + n])
        be = CpuBandBackend(local, fmt, cols, r0, nbands=3)
        res = RowBandSolver(rows, cols, rank, world, be).solve(local)
        out.append((res.side, res.area, res.cells_visited, res.top, res.left))
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fmt", [(2, 0), (3, 0), (4, 0), (2, 1), (4, 1)])
def test_row_band_sharding_matches_whole_matrix(world, fmt):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = here + os.pathsep + os.path.dirname(here) + os.pathsep + os.environ.get("PYTHONPATH", "")
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), fmt, results), nprocs=world, join=True)
    want = [oracle.freq(a) for a in _cases()]
    for rank in range(world):
        got = results[rank]
        for g_, w_ in zip(got, want):
            assert g_ == (w_.side, w_.area, w_.cells_visited, w_.top, w_.left)
