"""ctypes binding of libmsq.so (include/msq.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every solver raises.  Loading the library itself needs no
GPU (the CPU test-suite checks that every symbol of include/msq.h resolves).
"""
from __future__ import annotations

import ctypes
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libmsq.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "msq.h")

MSQ_OK, MSQ_EINVAL, MSQ_EVALUE, MSQ_ECUDA, MSQ_ENOMEM, MSQ_EAGAIN = 0, 1, 2, 3, 4, 5
ENGINE_BAND, ENGINE_TEAM, ENGINE_SIEVE = 0, 1, 2
FMT_U8, FMT_BITS = 0, 1
PLAN_NO_STRIP, PLAN_NO_SEED, PLAN_SINGLE_TEAM, PLAN_CLIMB_FIXUP, PLAN_PASS1 = 1, 2, 4, 8, 16


class MsqResult(ctypes.Structure):
    _fields_ = [("side", ctypes.c_int64), ("area", ctypes.c_int64),
                ("cells_visited", ctypes.c_int64), ("top", ctypes.c_int64),
                ("left", ctypes.c_int64)]


class MsqDevResult(ctypes.Structure):
    _fields_ = [("key_pass1", ctypes.c_uint64), ("key_fix", ctypes.c_uint64),
                ("status", ctypes.c_uint32), ("best_side", ctypes.c_int32),
                ("reserved", ctypes.c_uint64)]


class MsqPlan(ctypes.Structure):
    _fields_ = [("fmt", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("words", ctypes.c_int32), ("wpt", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("tile_rows", ctypes.c_int32), ("nbands", ctypes.c_int32),
                ("nstage", ctypes.c_int32), ("row_stage_bytes", ctypes.c_int32),
                ("smem_pass1", ctypes.c_int32), ("smem_fixup", ctypes.c_int32),
                ("deterministic", ctypes.c_int32), ("row_base", ctypes.c_int64),
                ("ws_bytes", ctypes.c_int64), ("team", ctypes.c_int32),
                ("teams_per_cta", ctypes.c_int32), ("tile_rows_l", ctypes.c_int32),
                ("tl", ctypes.c_int32), ("grid", ctypes.c_int32), ("fix_threads", ctypes.c_int32),
                ("fix_wpt", ctypes.c_int32), ("engine", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("test_floor", ctypes.c_int32),
                ("col_chunks", ctypes.c_int32), ("sv_bands", ctypes.c_int32),
                ("sv_ws_off", ctypes.c_int64)]


_lib = None


def header_symbols() -> list[str]:
    """Every function declared in include/msq.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(msq_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load libmsq.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python -m paper_2503_18974_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    RP = ctypes.POINTER(MsqResult)
    PP = ctypes.POINTER(MsqPlan)
    sig = {
        "msq_plan_make": ([I32, I32, I64, I64, I64, I32, I32, PP], ctypes.c_int),
        "msq_plan_make_ex": ([I32, I32, I64, I64, I64, I32, I32, I32, PP], ctypes.c_int),
        "msq_launch": ([PP, P, P, P, P], ctypes.c_int),
        "msq_decode": ([ctypes.POINTER(MsqDevResult), I64, I64, RP], ctypes.c_int),
        "msq_solve_u8": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_solve_bits": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_solve_batch_u8": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_dp_batch_u8": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_dp_solve": ([I32, P, I64, I64, I64, P, P, RP, P], ctypes.c_int),
        "msq_brute_u8": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_parse_text": ([P, I64, I64, I64, I32, P, I64, ctypes.POINTER(I64), P], ctypes.c_int),
        "msq_cube_probe": ([P, I64, I64, I64, I64, P, ctypes.POINTER(I64), P], ctypes.c_int),
        "msq_max_rectangle_scratch_bytes": ([I64, I64], I64),
        "msq_max_rectangle_u8": ([P, I64, I64, I64, P, ctypes.POINTER(I64), ctypes.POINTER(I64),
                                  ctypes.POINTER(I64), P], ctypes.c_int),
        "msq_solve_u8_host": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_solve_bits_host": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_solve_batch_u8_host": ([P, I64, I64, I64, RP, P], ctypes.c_int),
        "msq_rank_pass1": ([PP, P, P, P, P], ctypes.c_int),
        "msq_rank_seed": ([PP, P, P, P], ctypes.c_int),
        "msq_rank_band_pass": ([PP, P, P, P, P], ctypes.c_int),
        "msq_rank_summary": ([PP, P, P, P], ctypes.c_int),
        "msq_compose_carry": ([P, P, I32, I32, I64, P, P], ctypes.c_int),
        "msq_rank_fixup": ([PP, P, P, P, P], ctypes.c_int),
        "msq_rank_key_status": ([P, P, P], ctypes.c_int),
        "msq_rank_sieve": ([PP, P, P, I64, I64, P, P, P], ctypes.c_int),
        "msq_rank_sieve_pass": ([PP, P, P, I64, I64, P, P, P], ctypes.c_int),
        "msq_rank_sieve_finish": ([PP, P, P, I64, I64, P, P, P], ctypes.c_int),
        "msq_debug_set_sieve_wpc": ([I32], None),
        "msq_debug_set_sieve_phases": ([I32], None),
        "msq_ws_views": ([PP, P, P, P, P, P], ctypes.c_int),
        "msq_gen_hash": ([I32, U64, U64, I64, I64, I64, I64, P, P], ctypes.c_int),
        "msq_last_launch_count": ([], I32),
        "msq_debug_set_profile": ([P], None),
        "msq_debug_set_staging": ([I32, I32, I64], None),
        "msq_debug_set_team_band_rows": ([I32], None),
        "msq_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "msq_last_cuda_error": ([], ctypes.c_char_p),
        "msq_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


class MsqError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map a status code to the reference's error behaviour (ValueError for bad cells)."""
    if rc == MSQ_OK:
        return
    msg = load().msq_strerror(rc).decode()
    if rc in (MSQ_EVALUE, MSQ_EINVAL):
        raise ValueError(msg)
    detail = load().msq_last_cuda_error().decode() if rc == MSQ_ECUDA else ""
    raise MsqError(f"libmsq: {msg} (code {rc}) {detail}")


def plan(fmt: int, batch: int, rows: int, cols: int, ld: int, nbands: int = 0,
         deterministic: bool = False, engine: int = -1) -> MsqPlan:
    p = MsqPlan()
    check(load().msq_plan_make_ex(fmt, batch, rows, cols, ld, nbands, int(deterministic), engine,
                                  ctypes.byref(p)))
    return p
