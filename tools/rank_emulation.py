"""One-GPU emulation of the N-rank row-band split of cfg4 (no kernel waits on another).

For N in 1/2/4/8, the 65536^2 matrix is cut into N row slices; each slice is
solved by the rank API exactly as rank r of an N-GPU job would (msq_rank_seed
-> [all-reduce of the best side: here the max of the ranks' seeds, written
back] -> msq_rank_band_pass -> msq_rank_summary -> [all-gather] ->
msq_compose_carry -> msq_rank_fixup -> msq_rank_key_status), one rank after
another, each phase timed with CUDA events.  Per-rank time = what one GPU of
the N-GPU job spends on device work; the collectives (8 B all-reduce, cols*4 B
all-gather, 16 B all-reduce) are not included.  Prints one JSON line per N.

Bit-packed slices whose plan is a sieve plan (cfg4) take the sieve protocol
instead, as RowBandSolver does: rank r gets the last 256 rows of rank r-1 (the
halo send/recv, 2 MB, is not timed) and runs msq_rank_sieve_pass +
msq_rank_sieve_finish over (halo, local rows); `rank_emulation.py cfg4 band`
forces the band protocol for comparison.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_18974_b200 import _native as N, build, configs
from paper_2503_18974_b200.distributed import GpuBackend, decode_key, slice_rows

build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
spec = configs.CONFIGS[cfg]
full = configs.cfg4_device() if cfg == "cfg4" else configs.cfg5_device()
fmt = N.FMT_BITS if cfg == "cfg4" else N.FMT_U8
rows, cols = spec["rows"], spec["cols"]
REPS = 10
FORCE_BAND = len(sys.argv) > 2 and sys.argv[2] == "band"
HALO = 256
for world in (1, 2, 4, 8):
    rank_rows = [slice_rows(rows, world, q)[1] for q in range(world)]
    bes, srcs = [], []
    for q in range(world):
        r0, n = slice_rows(rows, world, q)
        srcs.append(full[r0:r0 + n].contiguous())
        bes.append(GpuBackend(fmt, n, cols, r0, engine=0 if FORCE_BAND else -1))
    if bes[0].is_sieve:
        halos = [None] + [srcs[q - 1][-HALO:].contiguous() for q in range(1, world)]
        ph = {q: {"sieve_pass": 0.0, "coarse+verify": 0.0} for q in range(world)}
        whole = {q: 0.0 for q in range(world)}
        for it in range(REPS + 2):
            marks, keys = {}, []
            # keep the GPU busy while the host enqueues, so the events see device time
            # and not the host's launch rate (a rank's kernels are ~10 us long)
            torch.cuda._sleep(4_000_000)
            for q, be in enumerate(bes):
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                c = torch.cuda.Event(enable_timing=True)
                a.record(); be.sieve_pass(srcs[q], halos[q]); b.record(); be.sieve_finish(srcs[q], halos[q]); c.record()
                keys.append(be.key_status().clone())
                marks[q] = (a, b, c)
            # the same again without the event in the middle (the coarse pass and the
            # verifier then run beside the streaming pass, as in a real solve)
            for q, be in enumerate(bes):
                d = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
                d.record(); be.sieve(srcs[q], halos[q]); e.record()
                marks[q] += (d, e)
            torch.cuda.synchronize()
            if it >= 2:
                for q in range(world):
                    a, b, c, d, e = marks[q]
                    ph[q]["sieve_pass"] += a.elapsed_time(b) / REPS
                    ph[q]["coarse+verify"] += b.elapsed_time(c) / REPS
                    whole[q] += d.elapsed_time(e) / REPS
        ks = torch.stack(keys).max(dim=0).values.cpu().numpy()
        r = decode_key(int(ks[0]), 0, rows, cols)
        per_rank = [whole[q] for q in range(world)]
        slowest = max(per_rank)
        print(json.dumps({"config": cfg, "protocol": "sieve", "world": world, "rows_per_rank": rank_rows[0],
                          "halo_rows": HALO if world > 1 else 0, "status": int(ks[1]),
                          "per_rank_ms": [round(x, 4) for x in per_rank],
                          "phases_ms_rank0": {k: round(v, 4) for k, v in ph[0].items()},
                          "phases_ms_last": {k: round(v, 4) for k, v in ph[world - 1].items()},
                          "projected_gcells_s": round(rows * cols / (slowest * 1e-3) / 1e9, 1),
                          "answer": [r.side, r.top, r.left]}), flush=True)
        continue
    gathered = torch.empty((world, cols), dtype=torch.int32, device="cuda")
    phases = {q: {"seed": 0.0, "band_pass": 0.0, "summary": 0.0, "compose+carry+fixup": 0.0} for q in range(world)}

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    for it in range(REPS + 2):
        marks = {}
        torch.cuda._sleep(4_000_000)  # the host enqueues ahead of the device
        for q, be in enumerate(bes):
            a = ev(); be.seed(srcs[q]); b = ev()
            marks[q] = [a, b]
        best = torch.stack([be.best_side() for be in bes]).max()
        for be in bes:
            be.best_side().copy_(best.reshape(1))
        for q, be in enumerate(bes):
            a = ev(); be.band_pass(srcs[q]); b = ev(); s = be.rank_summary(); c = ev()
            gathered[q].copy_(s)
            marks[q] += [a, b, c]
        keys = []
        for q, be in enumerate(bes):
            a = ev()
            base = be.compose(gathered, rank_rows, q) if q > 0 else None
            be.fixup(base)
            keys.append(be.key_status())
            b = ev()
            marks[q] += [a, b]
        torch.cuda.synchronize()
        if it >= 2:
            for q in range(world):
                m = marks[q]
                phases[q]["seed"] += m[0].elapsed_time(m[1]) / REPS
                phases[q]["band_pass"] += m[2].elapsed_time(m[3]) / REPS
                phases[q]["summary"] += m[3].elapsed_time(m[4]) / REPS
                phases[q]["compose+carry+fixup"] += m[5].elapsed_time(m[6]) / REPS
    ks = torch.stack(keys).max(dim=0).values.cpu().numpy()
    r = decode_key(int(ks[0]), int(ks[1]), rows, cols)
    per_rank = [sum(phases[q].values()) for q in range(world)]
    slowest = max(per_rank)
    print(json.dumps({"config": cfg, "world": world, "rows_per_rank": rank_rows[0],
                      "per_rank_ms": [round(x, 4) for x in per_rank],
                      "phases_ms_rank0": {k: round(v, 4) for k, v in phases[0].items()},
                      "phases_ms_last": {k: round(v, 4) for k, v in phases[world - 1].items()},
                      "projected_gcells_s": round(rows * cols / (slowest * 1e-3) / 1e9, 1),
                      "answer": [r.side, r.top, r.left]}), flush=True)
