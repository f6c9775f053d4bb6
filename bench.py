#!/usr/bin/env python
"""Benchmark: maximal-square Gcells/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

One step = one full solve of the workload (all band passes, band-boundary
fix-ups and, for N > 1, the NCCL exchange + key all-reduce) with the input
already resident in HBM.  Default workload: cfg4 (65536^2 bit-packed,
Bernoulli(0.999)), the matrix BASELINE.json's scaling target names; it is row-
band sharded across the N ranks (strong scaling: the matrix is fixed).

Rank 0 prints ONE JSON line.  Extra keys: roofline (dominant kernel = band
pass, algorithmic bytes = input bytes per launch), cpu_baseline (the
reference's own Python freq_square and dp_full from baseline/_ref, single
threaded as its contract says, reference bench semantics, bounded sample), e2e
(the public API -- freq_square_bits / freq_square / solve_batch -- on a
pageable numpy array, H2D copy and result read-back inside the timed region),
clocks (NVML sampled during the timed region), gpu_launches.  Inputs smaller
than L2 get a 256 MiB flush before every step, outside the step's events.

--impl reference solves the WHOLE configured matrix every step with the
reference algorithm's CPU implementation (the C restatement in oracle/ -- the
reference being pure Python -- per row band on all host threads plus the band
combine), on the same bytes for cfg1-cfg4.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Gcells/s for maximal-square side at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gcells/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def env_dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join()

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ workload
def build_input(cfg: str, torch, rank: int, world: int):
    """Device input for this rank (its row slice for row-band sharding)."""
    from paper_2503_18974_b200 import configs
    from paper_2503_18974_b200 import _native as N
    spec = configs.CONFIGS[cfg]
    if cfg == "cfg4":
        full = configs.cfg4_device()
        fmt = N.FMT_BITS
    elif cfg in ("cfg4_p99", "cfg4_planted"):
        full = configs.cfg4_variant_device(cfg)
        fmt = N.FMT_BITS
    elif cfg == "cfg5":
        full = configs.cfg5_device()
        fmt = N.FMT_U8
    elif cfg == "cfg3":
        full = configs.cfg3_device()
        fmt = N.FMT_U8
    elif cfg == "cfg1":
        full = torch.from_numpy(configs.cfg1_array()).cuda()
        fmt = N.FMT_U8
    elif cfg == "cfg2":
        full = torch.from_numpy(configs.cfg2_array()).cuda()
        fmt = N.FMT_U8
    else:
        raise SystemExit(f"unknown config {cfg}")
    if spec["batch"] > 1:
        b0 = spec["batch"] * rank // world
        b1 = spec["batch"] * (rank + 1) // world
        return full[b0:b1].contiguous(), fmt, spec
    r0 = spec["rows"] * rank // world
    r1 = spec["rows"] * (rank + 1) // world
    return full[r0:r1].contiguous(), fmt, spec


def _trimmed_mean(xs, trim=0.1):
    """bench.py:98-147 of the reference: drop floor(n * trim) runs per tail."""
    xs = sorted(xs)
    k = int(len(xs) * trim)
    xs = xs[k:len(xs) - k] if len(xs) > 2 * k else xs
    return sum(xs) / len(xs)


def _squarelab():
    """The reference package (pip-installed into baseline/_ref), or None."""
    for cand in (os.environ.get("SQUARELAB_REF"), os.path.join(ROOT, "baseline", "_ref")):
        if cand and os.path.isdir(os.path.join(cand, "squarelab")):
            if cand not in sys.path:
                sys.path.insert(0, cand)
            import squarelab.squares
            import squarelab.grid
            return squarelab
    return None


def _sample_rows(host_full, spec, cells_budget):
    """First rows of the workload (all columns) up to ~cells_budget cells, as u8."""
    cols = spec["cols"]
    rows = int(max(1, min(spec["rows"], cells_budget // cols)))
    sub = host_full[:rows]
    if spec["fmt"] == "bits":
        from paper_2503_18974_b200.grid import unpack_bits
        sub = unpack_bits(sub, cols)
    return np.ascontiguousarray(sub, dtype=np.uint8), rows


def cpu_baseline_reference(cfg: str, host_full, spec):
    """The reference's own CPU path, single-threaded as its contract states
    (SPEC.md:469), timed with its bench semantics (bench.py:98-147: warmup 1,
    trimmed mean, one instance reused, generation excluded): squarelab's
    freq_square and its default DP baseline dp_full (bench.py:61), on a bounded
    sample of this workload.  Falls back to the oracle C port if the reference
    package is not installed."""
    cores = len(os.sched_getaffinity(0))
    sl = _squarelab()
    runs = 30 if cfg == "cfg1" else 3
    if spec["batch"] > 1:
        n = 16
        mats = [np.ascontiguousarray(host_full[k]) for k in range(n)]
        unit = f"first {n} of {spec['batch']} matrices ({spec['rows']}x{spec['cols']})"
        cells = n * spec["rows"] * spec["cols"]
        dp_mats, dp_unit, dp_cells = mats[:4], f"first 4 of {spec['batch']} matrices", 4 * spec["rows"] * spec["cols"]
    else:
        a, r = _sample_rows(host_full, spec, 8_000_000)
        mats, unit, cells = [a], f"first {r} rows x {spec['cols']} cols", a.size
        d, rd = _sample_rows(host_full, spec, 2_000_000)
        dp_mats, dp_unit, dp_cells = [d], f"first {rd} rows x {spec['cols']} cols", d.size
    if sl is None:
        import oracle
        ts = []
        for _ in range(runs + 1):
            t0 = time.perf_counter()
            for m in mats:
                oracle.freq(m)
            ts.append(time.perf_counter() - t0)
        v = cells / _trimmed_mean(ts[1:]) / 1e9
        return {"value": v, "unit": UNIT, "cores": 1, "host_cores": cores, "kind": "port",
                "sample": unit + " (reference package not installed: oracle C port, 1 thread)"}
    BM = sl.grid.BinaryMatrix
    objs = [BM(m.shape[0], m.shape[1], m.tobytes()) for m in mats]  # construction excluded
    dobjs = [BM(m.shape[0], m.shape[1], m.tobytes()) for m in dp_mats]

    def timed(fn, ob, n):
        ts = []
        for it in range(n + 1):  # warmup 1
            t0 = time.perf_counter()
            for o in ob:
                fn(o)
            ts.append(time.perf_counter() - t0)
        return _trimmed_mean(ts[1:])

    fv = cells / timed(sl.squares.freq_square, objs, runs) / 1e9
    dv = dp_cells / timed(sl.squares.dp_full, dobjs, 3 if runs > 3 else 1) / 1e9
    return {"value": fv, "unit": UNIT, "cores": 1, "host_cores": cores, "kind": "reference",
            "impl": "squarelab.freq_square (the reference's Python, 1 of %d host cores)" % cores,
            "sample": unit + f"; warmup 1, trimmed mean of {runs} (reference bench.py:98-147)",
            "dp_full": {"value": dv, "unit": UNIT, "sample": dp_unit,
                        "impl": "squarelab.dp_full (the reference's default DP baseline, bench.py:61)"}}


def host_workload(cfg: str, spec):
    """The configured matrix on the host, generated on the CPU: the same bytes as
    the GPU arm for cfg1-4 (MT19937 mirror, counter hash); cfg5 is the same recipe
    (N(0,1) noise, periodic Gaussian blur sigma 64, 40th percentile) drawn from
    numpy's generator, so a different instance of the same distribution."""
    from paper_2503_18974_b200 import configs
    import oracle
    cores = len(os.sched_getaffinity(0))
    if cfg == "cfg1":
        return configs.cfg1_array(), "same bytes as the GPU arm"
    if cfg == "cfg2":
        return configs.cfg2_array(), "same bytes as the GPU arm"
    if cfg in ("cfg3", "cfg4", "cfg4_p99", "cfg4_planted"):
        n, thr = spec["rows"], configs.thr53(spec["p"])
        words = (spec["cols"] + 31) // 32
        out = (np.empty((n, spec["cols"]), np.uint8) if cfg == "cfg3" else np.empty((n, words), np.uint32))
        step = -(-n // cores)

        def gen(k):
            r0, r1 = k * step, min(n, (k + 1) * step)
            if r0 < r1:
                fn = oracle.gen_hash_u8 if cfg == "cfg3" else oracle.gen_hash_bits
                out[r0:r1] = fn(spec["seed"], thr, r0, r1 - r0, spec["cols"])

        ths = [threading.Thread(target=gen, args=(k,)) for k in range(cores)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if cfg == "cfg3":
            k = spec["square"]
            top, left = configs.cfg3_square_pos(spec["seed"], n, k)
            out[top:top + k, left:left + k] = 1
        elif "square" in spec:  # bit-packed planted square
            k = spec["square"]
            top, left = configs.planted_pos(spec["seed"], n, k)
            for c in range(left, left + k):
                out[top:top + k, c >> 5] |= np.uint32(1 << (c & 31))
        return out, "same bytes as the GPU arm"
    import scipy.fft as sfft
    n, sigma, q = spec["rows"], spec["sigma"], spec["q"]
    rng = np.random.default_rng(spec["seed"])
    x = rng.standard_normal((n, n), dtype=np.float32)
    X = sfft.rfft2(x, workers=-1)
    del x
    fy = np.fft.fftfreq(n).astype(np.float32)
    fx = np.fft.rfftfreq(n).astype(np.float32)
    c = np.float32(-2.0 * np.pi ** 2 * sigma * sigma)
    X *= np.exp(c * fy * fy)[:, None]
    X *= np.exp(c * fx * fx)[None, :]
    y = sfft.irfft2(X, s=(n, n), workers=-1)
    del X
    k = int(q * n * n)
    thr = np.partition(y.ravel(), k)[k]
    return (y > thr).astype(np.uint8), "same recipe as the GPU arm, numpy noise (another instance)"


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The reference algorithm's CPU implementation on the WHOLE configured
    matrix, every step: the oracle's C restatement of Algorithm 1
    (squares.py:84-103; the reference itself is pure Python) run per row band
    on all host threads plus the band combine (carry fold, data-free fix-up),
    so each step returns the exact whole-matrix answer.  Batches: the
    matrices split over the threads."""
    if rank != 0:
        return 0
    from paper_2503_18974_b200 import configs
    import oracle
    oracle.lib()
    spec = configs.CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    host, same = host_workload(args.config, spec)
    fmt_bits = spec["fmt"] == "bits"
    cells = spec["batch"] * spec["rows"] * spec["cols"]

    def solve():
        if spec["batch"] > 1:
            res = [None] * cores
            step = -(-len(host) // cores)

            def part(k):
                res[k] = oracle.freq_batch(host[k * step:(k + 1) * step]) if k * step < len(host) else []

            ths = [threading.Thread(target=part, args=(k,)) for k in range(cores)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            return [r for p in res for r in p][0]
        return oracle.solve_banded_mt(host, 1 if fmt_bits else 0, spec["cols"], cores)

    for _ in range(args.warmup):
        ans = solve()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ans = solve()
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    value = cells * args.steps / total / 1e9
    sample = (f"whole matrix every step ({spec['rows']}x{spec['cols']}"
              f"{' x %d' % spec['batch'] if spec['batch'] > 1 else ''}, {same})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u32" if fmt_bits else "u8", "data": "synthetic",
        "config": {"workload": spec["workload"], "rows": spec["rows"], "cols": spec["cols"],
                   "batch": spec["batch"], "format": spec["fmt"],
                   "impl": ("oracle C port of Algorithm 1 (squares.py:84-103) per row band on "
                            f"{cores} host threads + band combine (carry fold, fix-up)"
                            if spec["batch"] == 1 else
                            f"oracle C port of Algorithm 1, matrices split over {cores} host threads"),
                   "answer": {"side": ans.side, "top": ans.top, "left": ans.left}},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults: 200 timed solves (~20 ms of device time on cfg4: the clocks are sampled
    # every millisecond, and a 2 ms region right after the synchronize still shows the
    # clock ramp: 0.108 ms per solve at 20 steps, 0.104 at 100 and 400); the CPU arm's
    # steps are whole-matrix solves of ~1 s each, so it defaults to 20
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--config", default="cfg4",
                    choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "cfg4_p99", "cfg4_planted"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 20 if args.impl == "reference" else 200
    if args.warmup is None:
        args.warmup = 5 if args.impl == "reference" else 10
    rank, world, local = env_dist()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2503_18974_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    from paper_2503_18974_b200 import _native as N
    from paper_2503_18974_b200.distributed import GpuBackend, RowBandSolver
    from paper_2503_18974_b200.squares import Solver

    src, fmt, spec = build_input(args.config, torch, rank, world)
    rows, cols = spec["rows"], spec["cols"]
    batch = spec["batch"]
    stream = torch.cuda.current_stream()
    lib = N.load()

    # ---- solver for this rank
    # batches, and single matrices the plan gives to the register team engine,
    # go through msq_launch (one kernel); larger single matrices through the
    # row-band pipeline (pass 1 + carry scan + fix-up, NCCL between ranks)
    use_solver = batch > 1 or (world == 1 and int(Solver(fmt, rows, cols).plan.engine) == 1)
    if use_solver:
        local_batch = src.shape[0] if batch > 1 else 1
        solver = Solver(fmt, rows, cols, batch=local_batch)
        band_solver = None
        cells_per_step_local = local_batch * rows * cols
        cells_total = batch * rows * cols
        bytes_per_cell = 0.125 if fmt == N.FMT_BITS else 1.0
    else:
        local_rows = src.shape[0]
        if world > 1:
            be = GpuBackend(fmt, local_rows, cols, rows * rank // world)
            band_solver = RowBandSolver(rows, cols, rank, world, be)
        else:
            be = GpuBackend(fmt, local_rows, cols, 0)
            band_solver = RowBandSolver(rows, cols, 0, 1, be)
        solver = None
        cells_per_step_local = local_rows * cols
        cells_total = rows * cols
        bytes_per_cell = 0.125 if fmt == N.FMT_BITS else 1.0

    # L2 policy: flush between steps when the per-rank input fits in L2
    in_bytes = src.numel() * src.element_size()
    flush = None
    if in_bytes < 256 * 2**20:
        flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")

    p1_ev = []

    def step(instrument=False):
        if flush is not None and instrument:
            flush.fill_(1)
        if use_solver:
            if instrument:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            solver.launch(src)
            if instrument:
                e1.record(stream)
                p1_ev.append((e0, e1))
            return 1
        if instrument and band_solver.sieve:
            # as RowBandSolver.launch on the sieve engine, with events around its
            # streaming pass (the kernel that reads the matrix)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            be_ = band_solver.backend
            halo = band_solver._exchange_halo(src) if world > 1 else None
            e0.record(stream)
            be_.sieve_pass(src, halo)
            e1.record(stream)
            p1_ev.append((e0, e1))
            be_.sieve_finish(src, halo)
            if world > 1:
                ks = be_.key_status()
                dist.all_reduce(ks, op=dist.ReduceOp.MAX)
                band_solver._ks = ks
            else:
                band_solver._ks = None
            return 0
        if instrument:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            be_ = band_solver.backend
            e0.record(stream)
            if world > 1:  # as RowBandSolver.launch: pooled seed, then the band passes
                be_.seed(src)
                dist.all_reduce(be_.best_side(), op=dist.ReduceOp.MAX)
                be_.band_pass(src)
            else:
                be_.pass1(src)
            e1.record(stream)
            p1_ev.append((e0, e1))
            # finish the solve exactly as RowBandSolver.launch does
            base = None
            if world > 1:
                summary = be_.rank_summary()
                dist.all_gather_into_tensor(band_solver.gathered, summary)
                if rank > 0:
                    base = be_.compose(band_solver.gathered, band_solver.rank_rows, rank)
            be_.fixup(base)
            if world > 1:
                ks = be_.key_status()
                dist.all_reduce(ks, op=dist.ReduceOp.MAX)
                band_solver._ks = ks
            else:
                band_solver._ks = None
            return 0
        band_solver.launch(src)
        return 0

    def result():
        if use_solver:
            return solver.result()
        return [band_solver.result()]

    # ---- warm-up (also the parity answer of this run)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    answer = result()

    # ---- timed region: K steps, barrier + sync on both sides, device events
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches_before = be.launches if not use_solver else 0
    # inputs < L2 are flushed before every step, OUTSIDE the step's events:
    # the step time is the sum of the K per-step event intervals
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps if flush is not None else 1)]
    with ClockSampler(local) as clk:
        if flush is None:
            evs[0][0].record(stream)
            for _ in range(args.steps):
                step()
            evs[0][1].record(stream)
        else:
            for e0, e1 in evs:
                flush.fill_(1)
                e0.record(stream)
                step()
                e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_per_step = ms_total / args.steps
    if not use_solver:
        gpu_launches = be.launches - launches_before
    else:
        gpu_launches = args.steps * int(lib.msq_last_launch_count())  # msq_launch kernels per step
    value = cells_total / (ms_per_step * 1e-3) / 1e9

    # ---- dominant kernel duration (band pass), measured separately with events
    p1_ev.clear()
    for _ in range(min(args.steps, 50)):
        step(instrument=True)
    torch.cuda.synchronize()
    p1_ms = statistics.mean(a.elapsed_time(b) for a, b in p1_ev)
    peak, peak_kind = load_peaks()
    alg_bytes = cells_per_step_local * bytes_per_cell
    achieved = alg_bytes / (p1_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": ("msq::team_kernel" if use_solver and int(solver.plan.engine) == 1 else
                           "msq::sieve_pass_kernel (the sieve engine's streaming pass: every input byte once, "
                           "block bitmap out)" if not use_solver and band_solver.sieve else
                           "band pass: msq::strip_kernel (+ ubits_kernel for the bands it hands back), "
                           "timed with the seed_climb_kernel before it" if fmt == N.FMT_BITS else
                           "band pass: msq::ustrip_kernel, timed with the seed_climb_kernel before it"),
                "kernel_ms": round(p1_ms, 5),
                "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": int(alg_bytes)}
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                roofline["traffic"] = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            pass

    # ---- e2e: the public API on a pageable numpy array (what a caller of
    # freq_square / freq_square_bits / solve_batch passes); the library's H2D
    # copy and the result read-back are inside the timed region
    e2e = None
    if world == 1:
        from paper_2503_18974_b200.squares import freq_square, freq_square_bits, solve_batch
        host = src.cpu().numpy()
        if fmt == N.FMT_BITS:
            host = host.view(np.uint32)
        host = np.array(host, copy=True)  # plain pageable memory
        if batch > 1:
            call, path = (lambda: solve_batch(host)), "solve_batch(numpy) -> msq_solve_batch_u8_host"
        elif fmt == N.FMT_BITS:
            call, path = (lambda: [freq_square_bits(host, cols)]), "freq_square_bits(numpy) -> msq_solve_bits_host"
        else:
            call, path = (lambda: [freq_square(host)]), "freq_square(numpy) -> msq_solve_u8_host"
        got = call()  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            got = call()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": cells_total / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(in_bytes),
               "d2h_bytes_per_step": int(32 * batch), "ms_per_step": dt * 1e3, "path": path,
               "host_memory": "pageable"}
        assert [(g.side, g.top, g.left) for g in got] == [(a.side, a.top, a.left) for a in answer]

    # ---- parity of this run's answer against the oracle (rank 0, cheap configs / sample)
    parity = None
    cpu = None
    if rank == 0 and world == 1:
        import oracle
        host_np = src.cpu().numpy()
        if fmt == N.FMT_BITS:
            host_np = host_np.view(np.uint32)
        if not args.no_verify:
            if batch > 1:
                want = oracle.freq_batch(host_np)  # every matrix of the batch
                got = answer
            elif fmt == N.FMT_BITS:
                want = [oracle.freq_bits(host_np, cols)]
                got = answer
            else:
                want = [oracle.freq(host_np)]
                got = answer
            parity = all((g.side, g.top, g.left) == (w.side, w.top, w.left)
                         for g, w in zip(got, want))
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_reference(args.config, host_np, spec)

    if rank == 0:
        a0 = answer[0]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32" if fmt == N.FMT_BITS else "u8", "data": "synthetic",
            "config": {"workload": spec["workload"], "rows": rows, "cols": cols, "batch": batch,
                       "format": "bits" if fmt == N.FMT_BITS else "u8",
                       "parallelism": (f"matrices x{world}" if batch > 1 else
                                       "one team (register engine)" if use_solver else
                                       f"sieve engine, row slices x{world}" if band_solver.sieve else
                                       f"row-bands x{world}"),
                       "engine": ("team" if use_solver and int(solver.plan.engine) == 1 else
                                  "batch teams" if use_solver else
                                  "sieve" if band_solver.sieve else
                                  "band" + (" (sieve undecided on this input: %d retry)" % band_solver.sieve_retries
                                            if band_solver.sieve_retries else "")),
                       "nbands_per_rank": int(be.plan.nbands) if not use_solver else 1,
                       "l2": ("input > 126 MB L2, no flush" if flush is None
                              else "256 MiB L2 flush between steps"),
                       "answer": {"side": a0.side, "top": a0.top, "left": a0.left}},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": int(gpu_launches),
            "parity_vs_oracle": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
