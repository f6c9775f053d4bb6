"""The five BASELINE.json configurations as seeded synthetic inputs.

No public dataset is involved: the paper's own inputs are random matrices
(PAPER.md:298).  Each config is restated here as a deterministic recipe
(SURVEY.md section 8(d)):

cfg1  single 512x512 u8, squarelab.grid.generate_matrix(GenSpec(512,512,0.7,0))
      (MT19937, bit-identical to the reference generator, grid.py:274-286)
cfg2  4096 x 256x256 u8, per-matrix density drawn from {.3,.5,.7,.9,.99} and a
      64-bit seed from random.Random(seed) (the verify.py:201-209 stream shape)
cfg3  16384^2 u8 Bernoulli(.95) counter-hash background + planted 2048^2
      all-ones square at a seeded position; plus all-zeros / all-ones
cfg4  65536^2 bit-packed u32 (LSB = lowest column) Bernoulli(.999) counter hash
cfg5  32768^2 u8: seeded N(0,1) noise, periodic Gaussian blur sigma=64 (FFT),
      thresholded at its 40th percentile (bisection) -> ~60% ones in blobs

Counter hash: cell(i,j) = (mix64(seed + (i*cols+j+1)*0x9E3779B97F4A7C15) >> 11)
< thr53(p); restated in C (oracle), CUDA (msq_gen_hash) and numpy (below).
"""
from __future__ import annotations

import random

import numpy as np

from .grid import GenSpec, generate_array

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1

CFG2_DENSITIES = (0.3, 0.5, 0.7, 0.9, 0.99)

CONFIGS = {
    "cfg1": {"workload": "cfg1: 512x512 u8 Bernoulli(0.7) seed 0", "rows": 512, "cols": 512,
             "fmt": "u8", "batch": 1},
    "cfg2": {"workload": "cfg2: 4096 x 256x256 u8, p in {.3,.5,.7,.9,.99}", "rows": 256,
             "cols": 256, "fmt": "u8", "batch": 4096, "seed": 2},
    "cfg3": {"workload": "cfg3: 16384^2 u8 Bernoulli(0.95) + planted 2048^2", "rows": 16384,
             "cols": 16384, "fmt": "u8", "batch": 1, "seed": 3, "p": 0.95, "square": 2048},
    "cfg4": {"workload": "cfg4: 65536^2 bit-packed u32 Bernoulli(0.999)", "rows": 65536,
             "cols": 65536, "fmt": "bits", "batch": 1, "seed": 4, "p": 0.999},
    # extra bit-packed workloads (not BASELINE configs): answers outside the strip
    # pass's window -- a sparser background, and a planted square far above it
    "cfg4_p99": {"workload": "extra: 65536^2 bit-packed u32 Bernoulli(0.99)", "rows": 65536,
                 "cols": 65536, "fmt": "bits", "batch": 1, "seed": 41, "p": 0.99},
    "cfg4_planted": {"workload": "extra: 65536^2 bit-packed u32 Bernoulli(0.999) + planted 4096^2",
                     "rows": 65536, "cols": 65536, "fmt": "bits", "batch": 1, "seed": 42, "p": 0.999,
                     "square": 4096},
    "cfg5": {"workload": "cfg5: 32768^2 u8 Gaussian-blob mask (sigma 64, 60% ones)",
             "rows": 32768, "cols": 32768, "fmt": "u8", "batch": 1, "seed": 5,
             "sigma": 64.0, "q": 0.4},
}


def thr53(p: float) -> int:
    return min(int(p * (1 << 53)), 1 << 53)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def hash_u8(seed: int, thr: int, row0: int, nrows: int, cols: int) -> np.ndarray:
    """numpy restatement of the counter-hash generator (uint8 cells)."""
    with np.errstate(over="ignore"):
        idx = (np.arange(row0 * cols, (row0 + nrows) * cols, dtype=np.uint64) + np.uint64(1))
        z = np.uint64(seed & M64) + idx * np.uint64(GOLDEN)
        return ((_mix64(z) >> np.uint64(11)) < np.uint64(thr)).astype(np.uint8).reshape(nrows, cols)


def cfg1_array() -> np.ndarray:
    return generate_array(GenSpec(512, 512, 0.7, 0))


def cfg2_specs(seed: int = 2, count: int = 4096) -> list[GenSpec]:
    master = random.Random(seed)
    specs = []
    for _ in range(count):
        p = master.choice(CFG2_DENSITIES)
        s = master.getrandbits(64)
        specs.append(GenSpec(256, 256, p, s))
    return specs


def cfg2_array(seed: int = 2, count: int = 4096) -> np.ndarray:
    out = np.empty((count, 256, 256), np.uint8)
    for k, spec in enumerate(cfg2_specs(seed, count)):
        out[k] = generate_array(spec)
    return out


def cfg3_square_pos(seed: int = 3, n: int = 16384, k: int = 2048) -> tuple[int, int]:
    r = random.Random(seed)
    return r.randint(0, n - k), r.randint(0, n - k)


# ------------------------------------------------------------ device builders
def _lib():
    from . import _native
    return _native


def device_hash(fmt: str, seed: int, p: float, rows: int, cols: int, device="cuda"):
    """Counter-hash matrix generated on the GPU (msq_gen_hash)."""
    import ctypes

    import torch
    N = _lib()
    if fmt == "u8":
        out = torch.empty((rows, cols), dtype=torch.uint8, device=device)
        ld = cols
        f = N.FMT_U8
    else:
        words = (cols + 31) // 32
        out = torch.empty((rows, words), dtype=torch.int32, device=device)
        ld = words
        f = N.FMT_BITS
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    N.check(N.load().msq_gen_hash(f, seed, thr53(p), 0, rows, cols, ld,
                                  ctypes.c_void_p(out.data_ptr()), stream))
    return out


def cfg3_device(seed: int = 3, n: int = 16384, k: int = 2048, p: float = 0.95, device="cuda"):
    m = device_hash("u8", seed, p, n, n, device)
    top, left = cfg3_square_pos(seed, n, k)
    m[top:top + k, left:left + k] = 1
    return m


def cfg4_device(seed: int = 4, n: int = 65536, p: float = 0.999, device="cuda"):
    return device_hash("bits", seed, p, n, n, device)


def planted_pos(seed: int, n: int, k: int) -> tuple[int, int]:
    r = random.Random(seed)
    return r.randint(0, n - k), r.randint(0, n - k)


def cfg4_variant_device(name: str, device="cuda"):
    """The extra bit-packed workloads (cfg4_p99, cfg4_planted) on the device."""
    c = CONFIGS[name]
    w = device_hash("bits", c["seed"], c["p"], c["rows"], c["cols"], device)
    if "square" in c:
        k = c["square"]
        top, left = planted_pos(c["seed"], c["rows"], k)
        # whole words inside the square at once, the two partial words bit by bit
        a0, a1 = (left + 31) // 32, (left + k) // 32
        w[top:top + k, a0:a1] = -1
        for cc in list(range(left, min(left + k, 32 * a0))) + list(range(max(32 * a1, left), left + k)):
            w[top:top + k, cc >> 5] |= (1 << (cc & 31)) if (cc & 31) != 31 else -(1 << 31)
    return w


def blob_mask_torch(n: int, sigma: float, q: float, seed: int, device="cuda"):
    """Gaussian-blurred white noise thresholded at its q-quantile (cfg5)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.randn((n, n), generator=g, device=device, dtype=torch.float32)
    X = torch.fft.rfft2(x)
    del x
    fy = torch.fft.fftfreq(n, device=device)
    fx = torch.fft.rfftfreq(n, device=device)
    c = -2.0 * (np.pi ** 2) * sigma * sigma
    X *= torch.exp(c * fy * fy)[:, None]
    X *= torch.exp(c * fx * fx)[None, :]
    y = torch.fft.irfft2(X, s=(n, n))
    del X
    k = int(q * n * n)
    lo, hi = float(y.min()), float(y.max())
    for _ in range(48):  # bisection for the k-th order statistic
        mid = 0.5 * (lo + hi)
        if int((y <= mid).sum()) >= k:
            hi = mid
        else:
            lo = mid
    cells = (y > hi).to(torch.uint8)
    del y
    return cells


def cfg5_device(seed: int = 5, n: int = 32768, sigma: float = 64.0, q: float = 0.4, device="cuda"):
    return blob_mask_torch(n, sigma, q, seed, device)


def blob_mask_numpy(n: int, sigma: float, q: float, seed: int) -> np.ndarray:
    """CPU version of the cfg5 recipe for small n (tests)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, n)).astype(np.float32)
    X = np.fft.rfft2(x)
    fy = np.fft.fftfreq(n)
    fx = np.fft.rfftfreq(n)
    c = -2.0 * (np.pi ** 2) * sigma * sigma
    X *= np.exp(c * fy * fy)[:, None] * np.exp(c * fx * fx)[None, :]
    y = np.fft.irfft2(X, s=(n, n))
    thr = np.partition(y.ravel(), int(q * n * n))[int(q * n * n)]
    return (y > thr).astype(np.uint8)
