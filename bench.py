#!/usr/bin/env python
"""Benchmark: maximal-square Gcells/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

One step = one full solve of the workload (all band passes, band-boundary
fix-ups and, for N > 1, the NCCL exchange + key all-reduce) with the input
already resident in HBM.  Default workload: cfg4 (65536^2 bit-packed,
Bernoulli(0.999)), the matrix BASELINE.json's scaling target names; it is row-
band sharded across the N ranks (strong scaling: the matrix is fixed).

Rank 0 prints ONE JSON line.  Extra keys: roofline (dominant kernel = band
pass, algorithmic bytes = input bytes per launch), cpu_baseline (the oracle
port on the host, bounded sample), e2e (host buffers through the C ABI with the
H2D copy inside the timed region), clocks (NVML sampled during the timed
region), gpu_launches.

--impl reference times the reference algorithm's CPU implementation (the C
restatement in oracle/, the reference being pure Python) on the host cores.
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


def cpu_baseline_sample(cfg: str, host_full, spec, budget_s: float = 12.0, threads: int = 1):
    """Time the oracle port (Algorithm 1 restated in C) on a bounded sample."""
    import oracle
    if spec["batch"] > 1:
        unit_cells = spec["rows"] * spec["cols"]
        t0 = time.perf_counter()
        oracle.freq_batch(host_full[:4])
        per = (time.perf_counter() - t0) / 4
        n = max(1, min(len(host_full), int(budget_s / max(per, 1e-9))))
        t0 = time.perf_counter()
        oracle.freq_batch(host_full[:n])
        dt = time.perf_counter() - t0
        return n * unit_cells / dt / 1e9, f"first {n} of {spec['batch']} matrices", 1
    cols = spec["cols"]
    fmt_bits = spec["fmt"] == "bits"

    def run(rows):
        sub = host_full[:rows]
        t0 = time.perf_counter()
        if fmt_bits:
            oracle.freq_bits(sub, cols)
        else:
            oracle.freq(sub)
        return time.perf_counter() - t0

    probe = min(spec["rows"], 64)
    per_row = run(probe) / probe
    rows = int(max(probe, min(spec["rows"], budget_s / max(per_row, 1e-12))))
    if threads <= 1:
        dt = run(rows)
        return rows * cols / dt / 1e9, f"first {rows} rows x {cols} cols (1 solve)", 1
    # independent solves of distinct row slices, one per thread (ctypes drops the GIL)
    rows_t = max(1, min(rows, len(host_full) // threads))
    ts = []

    def worker(k):
        sub = host_full[k * rows_t:(k + 1) * rows_t]
        if fmt_bits:
            oracle.freq_bits(sub, cols)
        else:
            oracle.freq(sub)

    t0 = time.perf_counter()
    for k in range(threads):
        th = threading.Thread(target=worker, args=(k,))
        th.start()
        ts.append(th)
    for th in ts:
        th.join()
    dt = time.perf_counter() - t0
    return (threads * rows_t * cols / dt / 1e9,
            f"{threads} concurrent solves of {rows_t} x {cols} row slices", threads)


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_2503_18974_b200 import configs
    import oracle
    oracle.lib()
    spec = configs.CONFIGS[args.config]
    cores = len(os.sched_getaffinity(0))
    # host copy of the workload (generated with the oracle's own generator on CPU)
    if args.config == "cfg4":
        rows = min(spec["rows"], 4096 * cores)
        host = oracle.gen_hash_bits(spec["seed"], configs.thr53(spec["p"]), 0, rows, spec["cols"])
    elif args.config == "cfg3":
        rows = min(spec["rows"], 2048 * cores)
        host = oracle.gen_hash_u8(spec["seed"], configs.thr53(spec["p"]), 0, rows, spec["cols"])
    elif args.config == "cfg1":
        host = configs.cfg1_array()
    elif args.config == "cfg2":
        host = configs.cfg2_array(count=256)
    else:  # cfg5: blob mask recipe on CPU at reduced size (same statistics per row)
        host = configs.blob_mask_numpy(4096, spec["sigma"], spec["q"], spec["seed"])
        spec = dict(spec, rows=4096, cols=4096)
    vals = []
    sample = ""
    for it in range(args.warmup + args.steps):
        v, sample, used = cpu_baseline_sample(args.config, host, spec, budget_s=args.ref_budget,
                                              threads=cores)
        if it >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": {"workload": spec["workload"], "impl": "oracle C port"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=6.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    args = ap.parse_args()
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
        if flush is not None:
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
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = start.elapsed_time(end)
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
                           "band pass: msq::strip_kernel (+ pass1_kernel for bands it hands back), "
                           "timed with the seed_climb_kernel before it" if fmt == N.FMT_BITS else
                           "msq::pass1_kernel (timed with the seed_climb_kernel before it)"),
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

    # ---- e2e: host buffers through the C ABI, H2D inside the timed region
    e2e = None
    if world == 1 and batch == 1:
        host = src.cpu().pin_memory()
        out = N.MsqResult()
        hptr = ctypes.c_void_p(host.data_ptr())
        sh = ctypes.c_void_p(stream.cuda_stream)
        ld = src.shape[1]
        fn = lib.msq_solve_bits_host if fmt == N.FMT_BITS else lib.msq_solve_u8_host
        N.check(fn(hptr, rows, cols, ld, ctypes.byref(out), sh))  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            N.check(fn(hptr, rows, cols, ld, ctypes.byref(out), sh))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": cells_total / dt / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": 32,
               "ms_per_step": dt * 1e3, "path": fn.__name__}
        assert (out.side, out.top, out.left) == (answer[0].side, answer[0].top, answer[0].left)
    elif world == 1:
        host = src.cpu().pin_memory()
        dev = host.to("cuda", non_blocking=True)  # warm: device buffer, pinned path
        solver.launch(dev)
        solver.res.cpu()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            dev = host.to("cuda", non_blocking=True)
            solver.launch(dev)
            solver.res.cpu()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": cells_total / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(in_bytes),
               "d2h_bytes_per_step": int(32 * src.shape[0]), "ms_per_step": dt * 1e3,
               "path": "Solver.launch (msq_launch)"}

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
            v, sample, used = cpu_baseline_sample(args.config, host_np, spec,
                                                  budget_s=args.cpu_budget)
            cpu = {"value": v, "unit": UNIT, "cores": used, "kind": "port", "sample": sample}

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
                                       "one team (register engine)" if use_solver else f"row-bands x{world}"),
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
