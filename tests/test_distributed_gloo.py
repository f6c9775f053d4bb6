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


def _sieve_cases():
    rng = np.random.default_rng(321)
    cases = []
    for it in range(10):
        rows = int(rng.integers(80, 160))
        cols = int(rng.integers(40, 100))
        a = (rng.random((rows, cols)) < 0.97).astype(np.uint8)
        k = [6, 12, 16, 17, 30, 3, 10, 14, 40, 8][it]  # decided: 4..16 (the halo is 16 rows)
        top = [rows // 2 - k // 2, rows // 4, rows // 2 - 3, 5, rows // 2, 9, rows * 3 // 4 - 5, rows // 2 - k + 1,
               rows // 3, rows - k][it]
        a[top:top + k, 3:3 + k] = 1
        cases.append(a)
    return cases


def _sieve_worker(rank, world, port, fmt, results):
    import torch
    import torch.distributed as dist

    from cpu_band_backend import CpuSieveBackend
    from paper_2503_18974_b200.distributed import RowBandSolver, slice_rows
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    out = []
    for a in _sieve_cases():
        rows, cols = a.shape
        r0, n = slice_rows(rows, world, rank)
        local = a[r0:r0 + n] if fmt == 0 else grid.pack_bits(a[r0:r0 + n]).view(np.int32)
        be = CpuSieveBackend(local, fmt, cols, r0, nbands=3)
        solver = RowBandSolver(rows, cols, rank, world, be)
        src = torch.from_numpy(np.ascontiguousarray(local))
        res = solver.solve(src)
        again = solver.solve(src)  # an undecided input stays on the band protocol
        assert (again.side, again.top, again.left) == (res.side, res.top, res.left)
        out.append((res.side, res.area, res.cells_visited, res.top, res.left, solver.sieve_retries,
                    be.sieve_calls))
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fmt", [(2, 0), (3, 1), (4, 1)])
def test_sieve_protocol_halo_exchange_and_fallback(world, fmt):
    """RowBandSolver on a sieve backend: one halo send/recv per solve, every rank
    solves (halo, local rows) alone, all-reduce of [key, status]; answers the
    sieve cannot decide (here > 16 = the halo, or < 4) take the band protocol on
    every rank together, once, and stay there."""
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["PYTHONPATH"] = here + os.pathsep + os.path.dirname(here) + os.pathsep + os.environ.get("PYTHONPATH", "")
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_sieve_worker, args=(world, _free_port(), fmt, results), nprocs=world, join=True)
    cases = _sieve_cases()
    want = [oracle.freq(a) for a in cases]
    for rank in range(world):
        for g_, w_ in zip(results[rank], want):
            assert g_[:5] == (w_.side, w_.area, w_.cells_visited, w_.top, w_.left)
            decided = 4 <= w_.side <= 16
            assert g_[5] == (0 if decided else 1)          # one collective fall-back, or none
            assert g_[6] == 2 if decided else g_[6] == 1   # the sieve is not tried again after it
