"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/msq.h declares, and plans shapes the way DESIGN.md says."""
import ctypes

import pytest

from paper_2503_18974_b200 import _native as N
from paper_2503_18974_b200 import build as B


@pytest.fixture(scope="module")
def lib():
    B.build()
    return N.load()


def test_every_header_symbol_is_exported(lib):
    names = N.header_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_strerror_and_version(lib):
    assert lib.msq_strerror(N.MSQ_EVALUE).decode() == "cells must contain only 0 or 1"
    assert b"sm_100a" in lib.msq_version()


def test_plan_shapes(lib):
    p = N.plan(N.FMT_BITS, 1, 65536, 65536, 2048)
    assert (p.words, p.wpt, p.team) == (2048, 4, 512)
    assert p.threads == 512
    assert (p.fix_wpt, p.fix_threads) == (4, 512)
    assert p.nstage >= 8 and p.smem_pass1 <= 232448 and p.smem_fixup <= 232448
    assert 1 <= p.nbands <= 148
    p = N.plan(N.FMT_U8, 1, 32768, 32768, 32768)
    assert (p.words, p.wpt, p.team) == (1024, 2, 512)
    assert p.nstage >= 2
    p = N.plan(N.FMT_U8, 4096, 256, 256, 256)
    assert (p.nbands, p.team, p.batch) == (1, 8, 4096)  # sub-warp teams of 8 lanes
    assert p.teams_per_cta * p.team == p.threads and p.threads % 32 == 0
    assert p.grid * p.teams_per_cta >= 4096
    assert p.smem_pass1 <= 232448
    # odd width: no TMA staging (rows are not 16-byte multiples)
    p = N.plan(N.FMT_U8, 1, 7, 13, 13)
    assert p.nstage == 0 and p.nbands == 1


def test_plan_rejects_bad_shapes(lib):
    with pytest.raises(ValueError):
        N.plan(N.FMT_U8, 1, 10, 70000, 70000)  # wider than 65536 columns
    with pytest.raises(ValueError):
        N.plan(N.FMT_U8, 1, 10, 10, 5)  # ld < cols
    with pytest.raises(ValueError):
        N.plan(N.FMT_U8, 1, 0, 10, 10)


def test_bands_respect_uint16_heights(lib):
    p = N.plan(N.FMT_BITS, 1, 2**20, 64, 2, nbands=1)
    assert p.nbands >= 17  # every band <= 65535 rows


def test_decode_empty_key(lib):
    r = N.MsqDevResult()
    out = N.MsqResult()
    assert lib.msq_decode(ctypes.byref(r), 3, 4, ctypes.byref(out)) == 0
    assert (out.side, out.area, out.cells_visited, out.top, out.left) == (0, 0, 12, -1, -1)
    r.status = 1
    assert lib.msq_decode(ctypes.byref(r), 3, 4, ctypes.byref(out)) == N.MSQ_EVALUE


def test_engine_selection(lib):
    """Which engine a plan picks: team engine for batches and
    for single matrices up to 1024 columns (row bands when the plan has
    several), band engine otherwise or when bands are requested explicitly."""
    assert N.plan(N.FMT_U8, 4096, 256, 256, 256).engine == 1           # cfg2
    p = N.plan(N.FMT_U8, 1, 512, 512, 512)                              # cfg1
    assert p.engine == 1 and p.nbands > 1 and p.ws_bytes > 0
    assert N.plan(N.FMT_U8, 1, 100, 64, 64).engine == 1                 # one band, one team
    p4 = N.plan(N.FMT_BITS, 1, 65536, 65536, 2048)                      # cfg4: sieve engine first
    assert p4.engine == 2 and p4.sv_bands >= 1 and p4.ws_bytes > p4.sv_ws_off > 0
    assert N.plan(N.FMT_BITS, 1, 65536, 65536, 2048, engine=0).engine == 0
    assert N.plan(N.FMT_BITS, 1, 65536, 65536, 2048, deterministic=True).engine == 0
    assert N.plan(N.FMT_BITS, 1, 2048, 65536, 2048).engine == 0         # below 4096 rows: band engine
    assert N.plan(N.FMT_BITS, 1, 700, 768, 24, engine=2).engine == 2    # any shape the sieve can stream
    assert N.plan(N.FMT_BITS, 1, 700, 800, 28, engine=2).engine == 2    # 25 words in a 16-byte-multiple stride
    with pytest.raises(ValueError):
        N.plan(N.FMT_BITS, 1, 700, 800, 25, engine=2)                   # stride of 25 words: not 16-byte rows
    with pytest.raises(ValueError):
        N.plan(N.FMT_U8, 1, 4096, 4096, 4096, engine=2)                 # bit-packed only
    assert N.plan(N.FMT_U8, 1, 512, 512, 512, nbands=4).engine == 0     # explicit bands
    assert N.plan(N.FMT_U8, 1, 512, 2048, 2048).engine == 0             # wider than 1024
    assert N.plan(N.FMT_U8, 3, 4000, 64, 64).engine == 0                # batch rows > 2040


def test_sieve_entry_points_reject_bad_arguments(lib):
    p = N.plan(N.FMT_BITS, 1, 4096, 4096, 128)
    assert p.engine == 2
    band = N.plan(N.FMT_BITS, 1, 4096, 4096, 128, engine=0)
    ptr = ctypes.c_void_p(4096)  # aligned, never dereferenced: every check fails first
    for fn in (lib.msq_rank_sieve, lib.msq_rank_sieve_pass, lib.msq_rank_sieve_finish):
        assert fn(None, ptr, None, 0, 0, ptr, ptr, None) == N.MSQ_EINVAL
        assert fn(ctypes.byref(band), ptr, None, 0, 0, ptr, ptr, None) == N.MSQ_EINVAL      # not a sieve plan
        assert fn(ctypes.byref(p), None, None, 0, 0, ptr, ptr, None) == N.MSQ_EINVAL
        assert fn(ctypes.byref(p), ctypes.c_void_p(4100), None, 0, 0, ptr, ptr, None) == N.MSQ_EINVAL  # misaligned
        assert fn(ctypes.byref(p), ptr, None, 256, 128, ptr, ptr, None) == N.MSQ_EINVAL     # halo rows, no halo
        assert fn(ctypes.byref(p), ptr, ptr, 12, 128, ptr, ptr, None) == N.MSQ_EINVAL       # not a multiple of 8
        assert fn(ctypes.byref(p), ptr, ptr, 512, 128, ptr, ptr, None) == N.MSQ_EINVAL      # more than 256
        assert fn(ctypes.byref(p), ptr, ptr, 256, 64, ptr, ptr, None) == N.MSQ_EINVAL       # halo stride < words
        assert fn(ctypes.byref(p), ptr, ptr, 256, 128, ptr, ptr, None) == N.MSQ_EINVAL      # row_base 0 with a halo
    assert lib.msq_strerror(N.MSQ_EAGAIN).decode().startswith("the sieve engine could not decide")


def test_new_entry_points_reject_bad_arguments(lib):
    out = N.MsqResult()
    bad = ctypes.c_int64()
    assert lib.msq_parse_text(None, 10, 1, 4, N.FMT_BITS, None, 1, ctypes.byref(bad), None) == N.MSQ_EINVAL
    assert lib.msq_dp_batch_u8(None, 1, 4, 300, ctypes.byref(out), None) == N.MSQ_EINVAL  # cols > 256
    first = ctypes.c_int64()
    assert lib.msq_cube_probe(None, 2, 2, 2, 1, None, ctypes.byref(first), None) == N.MSQ_EINVAL
    a, h, w = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    assert lib.msq_max_rectangle_u8(None, 0, 0, 0, None, ctypes.byref(a), ctypes.byref(h), ctypes.byref(w), None) == N.MSQ_OK
    assert (a.value, h.value, w.value) == (0, 0, 0)
