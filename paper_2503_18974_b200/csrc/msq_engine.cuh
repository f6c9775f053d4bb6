// msq_engine.cuh -- sm_100a kernels for the maximal-square hot path.
//
// Reference semantics: /root/reference/pkg/src/squarelab/squares.py:68-114
// (Algorithm 1 / _freq_core): per row, column one-run heights ("freq") are
// updated and ONE threshold test is made -- do t consecutive columns have
// height >= t, t = best side so far + 1.  On success the side grows by one and
// the location is the cell where the t-run closes (squares.py:93-97).
//
// B200 design (DESIGN.md has the full argument and the measurements):
//  * One CTA ("team") per row band of one matrix; for batches of small
//    matrices a team is a sub-warp (8/16/32 lanes) and one matrix is one band.
//    Thread tau owns WPT consecutive 32-column words.  Rows stream through a
//    TMA bulk-copy ring in shared memory (one cp.async.bulk per row).
//  * Work per word-row is divergence free.  Two regimes, switched per tile:
//      mode S (t < tl): heights kept as 7-plane bit-sliced saturating
//        counters (min(h,127)); the eligibility mask E = {h >= t} is a
//        bit-sliced compare against the warp-uniform t.  The row test walks
//        E words (clz/ffs) from the smem E history.
//      mode L (t >= tl >= 63): a run of >= t eligible columns must contain a
//        whole word whose 32 columns are all eligible.  Per word we keep only
//        Zw = last row with any zero; F = {rho - Zw >= t} is one compare.  The
//        test scans the tile's F bitmap (rare runs) and checks the two
//        boundary words exactly from per-column last-zero rows in smem.
//    Per-column last-zero rows are written in a deferred per-tile phase (C)
//    from the rows still resident in the TMA ring, so the hot loop never
//    branches per bit.
//  * B rows are tested per barrier; a raise inside a tile re-tests later rows
//    at t+1 with X_b(t+1) = X_b(t) & X_{b-1}(t) (X = E or F).
//  * Bands run standalone; squares crossing a band top are recovered by a
//    data-free fix-up on virtual heights c_j + d while d <= e_j (P5/P6).
//  * Result: one 64-bit key per unit, (side, -bottom, -right), max-reduced.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace msq {

constexpr int KEY_DIM_BITS = 21;
constexpr unsigned long long KEY_DIM_MASK = (1ull << KEY_DIM_BITS) - 1ull;
constexpr uint32_t RES_INF = 0xFFFFFFFFu;
constexpr int NPLANES = 7;   // mode S counters saturate at 127
#ifndef MSQ_ABLATE
#define MSQ_ABLATE 0  // experiments: bit 0 = no zero events, bit 1 = no mode-L candidates, bit 2 = no F build, bit 3 = no climb tests, bit 4 = seed t=120, bit 5 = no band-end summaries
#endif
constexpr int BMAX = 8;      // max rows per tile
constexpr int FIX_TL = 63;   // fix-up mode L threshold (runs then contain a full word)
constexpr int MAXP = 12;     // last-zero bit planes: bands are <= 4095 rows

__host__ __device__ __forceinline__ unsigned long long pack_key(long long side, long long bottom,
                                                                long long right) {
    if (side <= 0) return 0ull;
    return ((unsigned long long)side << (2 * KEY_DIM_BITS)) |
           ((KEY_DIM_MASK - (unsigned long long)bottom) << KEY_DIM_BITS) |
           (KEY_DIM_MASK - (unsigned long long)right);
}

// rows < 2^21 and nbands <= 2048, so the product fits in 32 unsigned bits
__host__ __device__ __forceinline__ int band_row0(int rows, int nbands, int band) {
    return (int)(((unsigned)rows * (unsigned)band) / (unsigned)nbands);
}

__host__ __device__ __forceinline__ int r16(int x) { return (x + 15) & ~15; }

struct Misc {
    uint32_t res[3];
    int g;
    int cres[BMAX];  // climb: leftmost window start per tile row (-1 = none)
    int pad[8];
    alignas(16) unsigned char ex[128];  // Pass1Exact of the team (smem: no local-memory stack)
};

// ------------------------------------------------------------ smem layouts
struct P1Layout {
    int ring, bars, pcs, zp, za, nzm, ab, hist, fmap, misc, total;
};
// per team; zp holds P bit-planes of the last-zero rows, hist bs rows of E
// words, fmap 2 x BMAX rows of F bits; pcs = optional phase-cycle counters
// (CTA teams only)
__host__ __device__ inline P1Layout p1_layout(int NT, int WPT, int nstage, int rs, int bs, int P, bool tma,
                                              bool pcs) {
    P1Layout L;
    const int wpad = NT * WPT, nfw = (wpad + 31) / 32;
    int off = 0;
    L.ring = off;
    if (tma) off += nstage * rs;
    L.bars = off;
    if (tma) off += r16(nstage * 8);
    L.pcs = off;
    if (pcs) off += 16 * 8;
    L.zp = off;
    off += P * wpad * 4;
    L.za = off;  // global-z mode: last all-zero row per word
    off += r16(wpad * 2);
    L.nzm = off;  // global-z mode: never-zeroed column masks
    off += wpad * 4;
    L.ab = off;  // prefix-AND of the band top at the row above the tile (climb tiles)
    off += wpad * 4;
    L.hist = off;
    off += bs * wpad * 4;
    L.fmap = off;
    off += 2 * BMAX * r16(nfw * 4);
    off = r16(off);  // Misc holds 8/16-byte members
    L.misc = off;
    off += r16((int)sizeof(Misc));
    L.total = (off + 127) & ~127;
    return L;
}

struct FixLayout {
    int us, e8, wmin, hist, fmap, dmark, misc, total;
};
__host__ __device__ inline FixLayout fix_layout(int NT, int WPT, int bs) {
    FixLayout L;
    const int wpad = NT * WPT, nfw = (wpad + 31) / 32;
    int off = 0;
    L.us = off;
    off += wpad * 32 * 2;
    L.e8 = off;
    off += wpad * 32;
    L.wmin = off;  // per word: min carry, min leading-ones depth (uint16 pairs)
    off += wpad * 4;
    L.hist = off;
    off += bs * wpad * 4;
    L.fmap = off;
    off += 2 * BMAX * r16(nfw * 4);
    L.dmark = off;  // depth filter bitmap (band heights <= 4095)
    off += r16((4096 / 32 + 1) * 4);
    off = r16(off);  // Misc holds 8/16-byte members
    L.misc = off;
    off += r16((int)sizeof(Misc));
    L.total = (off + 127) & ~127;
    return L;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
// streaming rows are read once: evict them first so the band summaries stay in L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ uint32_t mbar_test_s(uint32_t bar_s, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar_s), "r"(parity)
        : "memory");
    return ok;
}
// shared-window (32-bit) address forms for the hot row loop
__device__ int g_spin_dbg;  // debug: failed barrier polls (profiling builds only)
__device__ __forceinline__ void mbar_wait_s(uint32_t bar_s, uint32_t parity, int* spins = nullptr) {
    uint32_t ok;
    do {
        if (spins) ++*spins;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar_s), "r"(parity)
            : "memory");
    } while (!ok);
}
template <int N>
__device__ __forceinline__ void lds_words(uint32_t addr, uint32_t (&w)[N]) {
    if (N == 4) {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[0]), "=r"(w[(1) % N]), "=r"(w[(2) % N]), "=r"(w[(3) % N])
                     : "r"(addr));
    } else if (N == 2) {
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[(1) % N]) : "r"(addr));
    } else {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(addr));
    }
}
__device__ __forceinline__ int ld_volatile(const int* p) { return *(const volatile int*)p; }

template <bool SUB>
__device__ __forceinline__ void tsync(unsigned mask) {
    if (SUB)
        __syncwarp(mask);
    else
        __syncthreads();
}

// 4 bytes in {0,1} -> 4 bits (byte i -> bit i).  The partial products of
// x * 0x01020408 land on distinct bit positions, so there are no carries.
__device__ __forceinline__ uint32_t nib4(uint32_t x) { return ((x * 0x01020408u) >> 24) & 0xFu; }
// 16 u8 cells (bytes 0/1) -> 16 bits: (x0 + 16 x1) * 0x01020408 has the 8
// cells of x0, x1 in column order in its top byte; one byte permute joins two
__device__ __forceinline__ uint32_t bits16(uint4 v) {
    const uint32_t p0 = (v.x + (v.y << 4)) * 0x01020408u;
    const uint32_t p1 = (v.z + (v.w << 4)) * 0x01020408u;
    return __byte_perm(p0, p1, 0x0073) & 0xFFFFu;
}
// 32 u8 cells -> 32 bits (two 16-byte vectors): three byte permutes join the four products
__device__ __forceinline__ uint32_t bits32(uint4 a, uint4 b) {
    const uint32_t p0 = (a.x + (a.y << 4)) * 0x01020408u;
    const uint32_t p1 = (a.z + (a.w << 4)) * 0x01020408u;
    const uint32_t p2 = (b.x + (b.y << 4)) * 0x01020408u;
    const uint32_t p3 = (b.z + (b.w << 4)) * 0x01020408u;
    return __byte_perm(__byte_perm(p0, p1, 0x0073), __byte_perm(p2, p3, 0x0073), 0x5410);
}

// windows of length t (1..32) inside a word: bit p set iff bits p..p+t-1 set
__device__ __forceinline__ uint32_t windows_in_word(uint32_t x, int t) {
    uint32_t y = x;
    int len = 1;
    while (2 * len <= t) {
        y &= y >> len;
        len *= 2;
    }
    if (len < t) y &= y >> (t - len);
    return y;
}

__device__ __forceinline__ uint32_t enc_res(int b, int col) { return ((uint32_t)b << 20) | (uint32_t)col; }

// X word at tile row b for threshold t+m: AND of rows b-m..b (P7)
__device__ __forceinline__ uint32_t x_at(const uint32_t* hist, int stride, int b, int m, int x) {
    uint32_t v = hist[b * stride + x];
    for (int q = 1; q <= m; ++q) v &= hist[(b - q) * stride + x];
    return v;
}

__device__ __forceinline__ int run_right(const uint32_t* hist, int Wpad, int W, int b, int m, int y,
                                         int L, int t) {
    while (L < t && y < W) {
        const uint32_t nx = x_at(hist, Wpad, b, m, y);
        if (nx == 0xFFFFFFFFu) {
            L += 32;
            ++y;
        } else {
            L += __ffs(~nx) - 1;
            break;
        }
    }
    return L;
}

// E test, every run that STARTS in word a
__device__ __forceinline__ void test_word_full(const uint32_t* hist, int Wpad, int W, int b, int m,
                                               int a, int t, uint32_t& best) {
    const uint32_t x = x_at(hist, Wpad, b, m, a);
    if (x == 0) return;
    if (t <= 32) {
        const uint32_t y = windows_in_word(x, t);
        if (y) best = min(best, enc_res(b, 32 * a + __ffs(y) - 1));
    }
    const int s = __clz(~x);
    if (s == 0) return;
    if (s == 32 && a > 0 && (x_at(hist, Wpad, b, m, a - 1) >> 31)) return;  // continuation
    const int L = run_right(hist, Wpad, W, b, m, a + 1, s, t);
    if (L >= t) best = min(best, enc_res(b, 32 * a + 32 - s));
}

// E test, every run intersecting word a (a gained eligible bits this row)
__device__ __forceinline__ void test_word_incr(const uint32_t* hist, int Wpad, int W, int b, int m,
                                               int a, int t, uint32_t& best) {
    const uint32_t x = x_at(hist, Wpad, b, m, a);
    if (x == 0) return;
    if (t <= 32) {
        const uint32_t y = windows_in_word(x, t);
        if (y) best = min(best, enc_res(b, 32 * a + __ffs(y) - 1));
    }
    if (x & 1u) {
        int start = 32 * a;
        for (int y = a - 1; y >= 0; --y) {
            const uint32_t px = x_at(hist, Wpad, b, m, y);
            if (px == 0xFFFFFFFFu) {
                start -= 32;
            } else {
                start -= __clz(~px);
                break;
            }
        }
        int L = 32 * a - start;
        if (x == 0xFFFFFFFFu)
            L = run_right(hist, Wpad, W, b, m, a + 1, L + 32, t);
        else
            L += __ffs(~x) - 1;
        if (L >= t) best = min(best, enc_res(b, start));
    }
    if (x != 0xFFFFFFFFu) {
        const int s = __clz(~x);
        if (s > 0) {
            const int L = run_right(hist, Wpad, W, b, m, a + 1, s, t);
            if (L >= t) best = min(best, enc_res(b, 32 * a + 32 - s));
        }
    }
}

// ------------------------------------------------------------------ params
struct Pass1Params {
    const uint8_t* src;
    long long ld_bytes;
    long long batch_stride;
    int rows, cols, W, nbands, cols_pad;
    long long row_base;
    int nstage, rs, row_bytes;  // TMA ring: one row per stage
    int bs, bl;                 // rows per tile in mode S / mode L
    int tl;                     // mode L threshold
    int share, write_summaries;
    int team;                   // threads per team
    int teams_per_cta;
    int zplanes;                // bit planes of the last-zero rows (2^P > band height)
    int units;                  // nbands * batch
    int layout_bytes;           // per-team smem bytes
    uint16_t* zb;               // [units][cols_pad] bottom runs (band outputs)
    uint16_t* e_out;
    uint32_t* ao_out;
    unsigned long long* band_keys;
    unsigned char* results;
    unsigned long long* prof;  // optional [units][16] phase-cycle counters (thread 0)
    const int* redo;           // optional [nbands]: bands the strip pass left over (0 = done)
};

struct FixParams {
    int rows, cols, W, nbands, cols_pad;
    long long row_base;
    int band_begin;
    int bs, bl;
    const uint16_t* e_in;
    const uint16_t* carry_in;  // [nbands][cols_pad] carry-in heights (clamped 65535)
    int share;
    unsigned long long* fix_keys;
    unsigned char* results;
};

__device__ __forceinline__ unsigned long long* res_key1(unsigned char* r) {
    return (unsigned long long*)(r + 0);
}
__device__ __forceinline__ unsigned long long* res_keyfix(unsigned char* r) {
    return (unsigned long long*)(r + 8);
}
__device__ __forceinline__ unsigned int* res_status(unsigned char* r) { return (unsigned int*)(r + 16); }
__device__ __forceinline__ int* res_best(unsigned char* r) { return (int*)(r + 20); }


// bit-sliced saturating increment (reset on zero): planes h[0..P-1]
template <int P>
__device__ __forceinline__ void planes_step(uint32_t (&h)[P], uint32_t w) {
    uint32_t c = w;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const uint32_t tmp = h[p] & c;
        h[p] ^= c;
        c = tmp;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) h[p] = (h[p] | c) & w;
}

// bit-sliced compare h >= t for a warp-uniform t in [0, 2^P)
template <int P>
__device__ __forceinline__ uint32_t planes_ge(const uint32_t (&h)[P], int t) {
    uint32_t ge = 0, eq = 0xFFFFFFFFu;
#pragma unroll
    for (int p = P - 1; p >= 0; --p) {
        if ((t >> p) & 1)
            eq &= h[p];
        else
            ge |= eq & h[p];
    }
    return ge | eq;
}

__device__ __forceinline__ uint32_t valid_mask(int a, int W, int cols) {
    if (a >= W) return 0u;
    const int rem = cols - 32 * a;
    return rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
}

// row words for the thread's WPT words from a staged row (TMA) or global
template <int WPT, bool U8, bool TMA>
__device__ __forceinline__ void fetch_words(const uint8_t* stage_row, const uint8_t* grow, int tau, int W,
                                            int cols, int rs, const uint32_t (&VAL)[WPT], uint32_t (&w)[WPT],
                                            uint32_t& bad_or) {
    if (U8) {
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            uint32_t word = 0;
            if (a < W) {
                if (TMA) {
                    const uint8_t* rp = stage_row + (size_t)a * 32;
                    const uint4 v0 = *(const uint4*)rp;
                    uint4 v1 = make_uint4(0, 0, 0, 0);
                    if (a * 32 + 16 < rs) v1 = *(const uint4*)(rp + 16);
                    bad_or |= v0.x | v0.y | v0.z | v0.w | v1.x | v1.y | v1.z | v1.w;
                    word = bits32(v0, v1);
                } else {
                    const int c0 = 32 * a;
                    const int n = min(32, cols - c0);
                    for (int j = 0; j < n; ++j) {
                        const uint32_t cb = grow[c0 + j];
                        bad_or |= cb;
                        word |= (cb & 1u) << j;
                    }
                }
            }
            w[k] = word & VAL[k];
        }
    } else {
        if (TMA) {
            const uint32_t* rp = (const uint32_t*)stage_row + tau * WPT;
            if (tau * WPT < W) {
                if (WPT >= 4) {
#pragma unroll
                    for (int q = 0; q < WPT / 4; ++q) {
                        const uint4 v = ((const uint4*)rp)[q];
                        w[(4 * q + 0) % WPT] = v.x;
                        w[(4 * q + 1) % WPT] = v.y;
                        w[(4 * q + 2) % WPT] = v.z;
                        w[(4 * q + 3) % WPT] = v.w;
                    }
                } else if (WPT == 2) {
                    const uint2 v = *(const uint2*)rp;
                    w[0] = v.x;
                    w[1 % WPT] = v.y;
                } else {
                    w[0] = rp[0];
                }
            } else {
#pragma unroll
                for (int k = 0; k < WPT; ++k) w[k] = 0;
            }
        } else {
            const uint32_t* rp = (const uint32_t*)grow;
#pragma unroll
            for (int k = 0; k < WPT; ++k) {
                const int a = tau * WPT + k;
                w[k] = a < W ? rp[a] : 0u;
            }
        }
#pragma unroll
        for (int k = 0; k < WPT; ++k) w[k] &= VAL[k];
    }
}

// one word of one staged/global row (any owner), for phase C / exact checks
template <bool U8, bool TMA>
__device__ __forceinline__ uint32_t word_of_row(const uint8_t* stage_row, const uint8_t* grow, int a,
                                                int cols, int rs) {
    if (U8) {
        uint32_t word = 0;
        if (TMA) {
            const uint8_t* rp = stage_row + (size_t)a * 32;
            const uint4 v0 = *(const uint4*)rp;
            uint4 v1 = make_uint4(0, 0, 0, 0);
            if (a * 32 + 16 < rs) v1 = *(const uint4*)(rp + 16);
            word = bits32(v0, v1);
        } else {
            const int c0 = 32 * a;
            const int n = min(32, cols - c0);
            for (int j = 0; j < n; ++j) word |= ((uint32_t)grow[c0 + j] & 1u) << j;
        }
        return word;
    }
    if (TMA) return ((const uint32_t*)stage_row)[a];
    return ((const uint32_t*)grow)[a];
}

// scan one F-bitmap word (32 words of the row) at tile row b, threshold T =
// t+m: every maximal F run that STARTS here and whose upper bound
// 32*len + 31 + 32 reaches T is handed to on_cand(b, a0, len).  A qualifying
// run = suffix(a0-1) + 32*len + prefix(a0+len); the boundary words are checked
// exactly by the caller.
template <class OnCand>
__device__ __forceinline__ void scan_fword(const uint32_t* fm, int nfw, int W, int b, int m, int fw,
                                           int T, OnCand&& on_cand) {
    const uint32_t x = x_at(fm, nfw, b, m, fw);
    if (!x) return;
    const uint32_t prev = fw > 0 ? (x_at(fm, nfw, b, m, fw - 1) >> 31) : 0u;
    uint32_t starts = x & ~((x << 1) | prev);
    const int nwords_f = (W + 31) / 32;
    while (starts) {
        const int i = __ffs(starts) - 1;
        starts &= starts - 1;
        const uint32_t rest = x >> i;
        int len = (~rest == 0u) ? 32 : (__ffs(~rest) - 1);
        if (i + len == 32) {
            for (int y = fw + 1; y < nwords_f; ++y) {
                const uint32_t nx = x_at(fm, nfw, b, m, y);
                if (nx == 0xFFFFFFFFu) {
                    len += 32;
                } else {
                    len += __ffs(~nx) - 1;
                    break;
                }
            }
        }
        const int a0 = fw * 32 + i;
        const int ub = 32 * len + (a0 > 0 ? 31 : 0) + (a0 + len < W ? 32 : 0);
        if (ub >= T) on_cand(b, a0, len);
    }
}

__device__ __forceinline__ int suffix_ones(uint32_t m) { return __clz(~m); }
__device__ __forceinline__ int prefix_ones(uint32_t m) { return m == 0xFFFFFFFFu ? 32 : __ffs(~m) - 1; }

// pass-1 exact eligibility of word a at tile row b, threshold T (T > BMAX):
// column j is eligible iff no zero in the tile rows <= b and its last zero
// before the tile, z_j, is <= rho_b - T.  z is kept bit-sliced in smem
// (zp[p*Wpad + k*NT + tau] = bit p of z for the 32 columns of word
// a = tau*WPT + k; z = 0 means "no zero in the band yet"), so the test is a
// bit-sliced compare with a warp-uniform constant.
__device__ __forceinline__ int zp_index(int a, int p, int WPT, int NT, int Wpad) {
    const int tau = a / WPT, k = a - tau * WPT;
    return p * Wpad + k * NT + tau;
}

// z_j = rho for the columns in `cols` (bit-sliced, P planes); loads first for ILP
template <int P>
__device__ __forceinline__ void zplanes_set_t(uint32_t* zp, int base, int stride, uint32_t cols, int rho) {
    uint32_t v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = zp[base + q * stride];
#pragma unroll
    for (int q = 0; q < P; ++q) zp[base + q * stride] = (v[q] & ~cols) | (((rho >> q) & 1) ? cols : 0u);
}
__device__ __forceinline__ void zplanes_set(uint32_t* zp, int base, int stride, int P, uint32_t cols, int rho) {
    switch (P) {
#define MSQ_ZS(n) \
    case n: zplanes_set_t<n>(zp, base, stride, cols, rho); break;
        MSQ_ZS(1) MSQ_ZS(2) MSQ_ZS(3) MSQ_ZS(4) MSQ_ZS(5) MSQ_ZS(6)
        MSQ_ZS(7) MSQ_ZS(8) MSQ_ZS(9) MSQ_ZS(10) MSQ_ZS(11) MSQ_ZS(12)
#undef MSQ_ZS
        default: break;
    }
}

// bit-sliced "Z <= c" over P planes (0 <= c < 2^P)
template <int P>
__device__ __forceinline__ uint32_t planes_le_t(const uint32_t* zp, int base, int stride, int c) {
    uint32_t v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = zp[base + q * stride];
    uint32_t lt = 0, eq = 0xFFFFFFFFu;
#pragma unroll
    for (int q = P - 1; q >= 0; --q) {
        if ((c >> q) & 1) {
            lt |= eq & ~v[q];
            eq &= v[q];
        } else {
            eq &= ~v[q];
        }
    }
    return lt | eq;
}
__device__ __forceinline__ uint32_t planes_le(const uint32_t* zp, int base, int stride, int P, int c) {
    switch (P) {
#define MSQ_LE(n) \
    case n: return planes_le_t<n>(zp, base, stride, c);
        MSQ_LE(1) MSQ_LE(2) MSQ_LE(3) MSQ_LE(4) MSQ_LE(5) MSQ_LE(6)
        MSQ_LE(7) MSQ_LE(8) MSQ_LE(9) MSQ_LE(10) MSQ_LE(11) MSQ_LE(12)
#undef MSQ_LE
        default: return 0u;
    }
}

// Per-column last-zero rows z_j (0 = no zero in the band yet) live either in
// smem bit planes (u8 inputs: dense zero events, updated with P-plane
// read-modify-writes) or, for bit-packed inputs (sparse zero events), as
// uint16 in L2-resident global scratch with one store per zero bit, a lazy
// all-zero row per word (za) and the never-zeroed masks (nzm) in smem.
template <bool U8, bool TMA>
struct Pass1Exact {
    const uint32_t* zp;
    const uint16_t* zg;   // global z (bits inputs)
    const uint16_t* za;
    const uint32_t* nzm;
    const uint8_t* ring;
    const uint8_t* mbase;
    long long ld_bytes;
    int W, cols, rs, nstage, P, WPT, NT, Wpad;
    int tile_row0;  // band-relative 0-based row of tile row 0
    int r0;         // band top row (matrix)
    int st0;        // ring stage of tile row 0
    __device__ __forceinline__ const uint8_t* srow(int b) const {
        return TMA ? ring + (size_t)(st0 + b) * rs : nullptr;  // a tile never wraps the ring (slots)
    }
    __device__ __forceinline__ const uint8_t* grow(int b) const {
        return mbase + (size_t)(r0 + tile_row0 + b) * ld_bytes;
    }
    // columns of word a whose last zero (before the current tile) is <= lim (lim >= 0)
    __device__ __forceinline__ uint32_t z_le(int a, int lim) const {
        if (U8) return (lim >= (1 << P)) ? 0xFFFFFFFFu : planes_le(zp, zp_index(a, 0, WPT, NT, Wpad), Wpad, P, lim);
        if ((int)za[a] > lim) return 0u;
        uint32_t m = nzm[a];
        const uint4* zq = (const uint4*)(zg + (size_t)a * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = zq[q];
            const uint32_t pr[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                m |= ((int)(pr[h] & 0xFFFFu) <= lim ? 1u : 0u) << (8 * q + 2 * h);
                m |= ((int)(pr[h] >> 16) <= lim ? 1u : 0u) << (8 * q + 2 * h + 1);
            }
        }
        return m;
    }
    __device__ __noinline__ uint32_t mask(int a, int b, int T) const {
        const uint32_t val = valid_mask(a, W, cols);
        const int lim = tile_row0 + b + 1 - T;
        if (lim < 0) return 0u;
        uint32_t zin = 0;
        for (int q = 0; q <= b; ++q) zin |= ~word_of_row<U8, TMA>(srow(q), grow(q), a, cols, rs);
        return z_le(a, lim) & val & ~zin;
    }
    // suffix of word a (a >= 0) and prefix of word c (c < W) at row b,
    // threshold T, packed as suffix | prefix << 8
    __device__ __noinline__ int boundary_len(int a, int c, int b, int T) const {
        const int lim = tile_row0 + b + 1 - T;
        if (lim < 0) return 0;
        uint32_t zina = 0, zinc = 0;
        for (int q = 0; q <= b; ++q) {
            if (a >= 0) zina |= ~word_of_row<U8, TMA>(srow(q), grow(q), a, cols, rs);
            if (c < W) zinc |= ~word_of_row<U8, TMA>(srow(q), grow(q), c, cols, rs);
        }
        const uint32_t ma = a >= 0 ? z_le(a, lim) & ~zina : 0u;
        const uint32_t mc = c < W ? z_le(c, lim) & valid_mask(c, W, cols) & ~zinc : 0u;
        return (a >= 0 ? suffix_ones(ma) : 0) | ((c < W ? prefix_ones(mc) : 0) << 8);
    }
};

// leftmost window of T consecutive ones in row X (smem, W words) starting at
// column >= s0; one full warp; returns the start column or -1.  Segmented
// warp scan of run lengths (R = full ? R_prev + 32 : suffix), chunk by chunk.
template <class Fetch>
__device__ __forceinline__ int warp_first_window(const Fetch& X, int W, int s0, int T, int lane) {
    int carry = 0;
    const int w0 = s0 >> 5;
    const uint32_t first_mask = ~((1u << (s0 & 31)) - 1u);
    for (int base = w0; base < W; base += 32) {
        const int w = base + lane;
        uint32_t x = (w < W) ? X(w) : 0u;
        if (w == w0) x &= first_mask;
        const bool full = x == 0xFFFFFFFFu;
        const int pre = prefix_ones(x);
        int v = full ? 32 : suffix_ones(x);
        int f = full ? 1 : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v2 = __shfl_up_sync(0xFFFFFFFFu, v, o);
            const int f2 = __shfl_up_sync(0xFFFFFFFFu, f, o);
            if (lane >= o) {
                if (f) v = v2 + v;
                f = f & f2;
            }
        }
        const int R = f ? carry + v : v;  // run ending at bit 31 of my word
        int Rin = __shfl_up_sync(0xFFFFFFFFu, R, 1);
        if (lane == 0) Rin = carry;
        int end = 64;
        if (Rin < T && Rin + pre >= T) end = T - Rin - 1;
        if (T <= 32 && x) {
            const uint32_t y = windows_in_word(x, T);
            if (y) end = min(end, __ffs(y) - 1 + T - 1);
        }
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, end < 64);
        if (bal) {
            const int src = __ffs(bal) - 1;
            const int e = __shfl_sync(0xFFFFFFFFu, end, src);
            return 32 * (base + src) + e - T + 1;
        }
        carry = __shfl_sync(0xFFFFFFFFu, R, 31);
    }
    return -1;
}

// climb tile row b: prefix-AND of the band top = ab & tile rows 0..b
template <bool U8, bool TMA>
struct ClimbRow {
    const uint32_t* ab;
    const Pass1Exact<U8, TMA>* ex;
    int b;
    __device__ __forceinline__ uint32_t operator()(int w) const {
        uint32_t x = ab[w];
        for (int q = 0; q <= b; ++q) x &= word_of_row<U8, TMA>(ex->srow(q), ex->grow(q), w, ex->cols, ex->rs);
        return x;
    }
};

template <bool U8, bool TMA>
__device__ __noinline__ int climb_scan(const uint32_t* ab, const Pass1Exact<U8, TMA>* ex, int b, int W, int s0, int T,
                                       int lane) {
    const ClimbRow<U8, TMA> f{ab, ex, b};
    return warp_first_window(f, W, s0, T, lane);
}

// exact eligibility of word a at tile row b for any threshold T (rows after a
// climb failure): last zero <= rho_b - T, from the planes (row above the tile)
// and the zeros of tile rows 0..b that are later than rho_b - T
template <bool U8, bool TMA>
__device__ __noinline__ uint32_t exact_row_mask(const Pass1Exact<U8, TMA>* ex, int a, int b, int T) {
    const uint32_t val = valid_mask(a, ex->W, ex->cols);
    const int rho_b = ex->tile_row0 + b + 1;
    const int lim = rho_b - T;
    if (lim < 0) return 0u;
    uint32_t late = 0;
    for (int q = 0; q <= b; ++q)
        if (ex->tile_row0 + q + 1 > lim) late |= ~word_of_row<U8, TMA>(ex->srow(q), ex->grow(q), a, ex->cols, ex->rs);
    return ex->z_le(a, lim) & ~late & val;
}

// Mode-L candidate check by a whole warp (bits inputs): candidate = F run
// [a0, a0+len) of tile row cb (packed cb | a0 << 3 | len << 14).  Lanes 0-7 /
// 8-15 read the tile-row words of the left / right boundary word, lane j tests
// column j of both boundary words against the last-zero rows (one coalesced
// 64-byte read per word), ballots give the exact masks.  Returns the encoded
// leftmost window start or RES_INF.
template <bool U8, bool TMA>
__device__ __noinline__ uint32_t coop_check(const Pass1Exact<U8, TMA>* ex, uint32_t cand, int T, int lane) {
    const int cb = (int)(cand & 7u), a0 = (int)((cand >> 3) & 0x7FFu), len = (int)(cand >> 14);
    const int W = ex->W;
    const int a = a0 - 1, c = a0 + len;
    const int lim = ex->tile_row0 + cb + 1 - T;
    if (lim < 0) return RES_INF;
    const int q = lane & 7;
    const int wsel = lane < 8 ? a : c;
    uint32_t zin = 0u;
    if (lane < 16 && q <= cb && wsel >= 0 && wsel < W)
        zin = ~word_of_row<U8, TMA>(ex->srow(q), ex->grow(q), wsel, ex->cols, ex->rs);
    const uint32_t zina = __reduce_or_sync(0xFFFFFFFFu, lane < 8 ? zin : 0u);
    const uint32_t zinc = __reduce_or_sync(0xFFFFFFFFu, lane < 8 ? 0u : zin);
    bool ea = false, ec = false;
    if (a >= 0 && (int)ex->za[a] <= lim)
        ea = ((ex->nzm[a] >> lane) & 1u) || (int)ex->zg[(size_t)a * 32 + lane] <= lim;
    if (c < W && (int)ex->za[c] <= lim)
        ec = ((ex->nzm[c] >> lane) & 1u) || (int)ex->zg[(size_t)c * 32 + lane] <= lim;
    const uint32_t ma = __ballot_sync(0xFFFFFFFFu, ea);
    const uint32_t mc = __ballot_sync(0xFFFFFFFFu, ec);
    const int suf = a >= 0 ? suffix_ones(ma & ~zina) : 0;
    const int pre = c < W ? prefix_ones(mc & ~zinc & valid_mask(c, W, ex->cols)) : 0;
    return suf + pre + 32 * len >= T ? enc_res(cb, 32 * a0 - suf) : RES_INF;
}

// bits inputs, small threshold: columns of word a whose last zero is <= lim
// (outlined: the cold path of the bits format)
__device__ __noinline__ uint32_t bits_small_e(const uint16_t* zg, int zaa, int a, uint32_t nz, uint32_t val, int lim) {
    if (!val || lim < 0 || zaa > lim) return 0u;
    uint32_t e = nz;
    for (int j = 0; j < 32; ++j)
        if (!((nz >> j) & 1u) && (int)zg[(size_t)a * 32 + j] <= lim) e |= 1u << j;
    return e & val;
}

// mode-S row tests of one thread's words (outlined: keeps the hot loop's
// register pressure down)
__device__ __noinline__ uint32_t test_rows_s(const uint32_t* hist, int Wpad, int W, int WPT, int tau, int start_b,
                                             int lastb, int full_from, uint32_t dirty, int m, int T) {
    uint32_t best = RES_INF;
    for (int b = start_b; b <= lastb; ++b) {
        const bool full = b >= full_from;
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            if (a < W) {
                if (full)
                    test_word_full(hist, Wpad, W, b, m, a, T, best);
                else if ((dirty >> (b * WPT + k)) & 1u)
                    test_word_incr(hist, Wpad, W, b, m, a, T, best);
            }
        }
    }
    return best;
}

// band outputs: bottom run b_j = H - z_j from the last-zero planes
__device__ __noinline__ void band_bottom_runs(const uint32_t* zp, int zbase, int Wpad, int P, int H, uint16_t* bo) {
    // the 32 last-zero rows as packed uint16 pairs, plane by plane; 4 vector stores
    uint32_t v[16];
#pragma unroll
    for (int h = 0; h < 16; ++h) v[h] = 0u;
    for (int q = 0; q < P; ++q) {
        const uint32_t zq = zp[zbase + q * Wpad];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j >> 1] |= ((zq >> j) & 1u) << (q + 16 * (j & 1));
    }
    const uint32_t HH = (uint32_t)H | ((uint32_t)H << 16);
#pragma unroll
    for (int h = 0; h < 16; ++h) v[h] = HH - v[h];  // per half: H - z (z <= H, no borrow)
    uint4* bq = (uint4*)bo;
#pragma unroll
    for (int q = 0; q < 4; ++q) bq[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

// Rows b < nrows of a tile (ring stages st0.., already waited for): loads of
// RG rows first, then their zero tests.  Returns the word-major zero flags
// (bit k*BMAX + b: row b has a zero in word k); optionally folds the rows
// into the prefix-AND AL and records it per row in hist (sub-warp climbs).
template <int WPT, bool U8, bool TMA>
__device__ __forceinline__ uint32_t tile_zero_flags(const Pass1Params& p, const uint8_t* ring,
                                                    const uint8_t* rows_base, int st0, int nrows, int tau, int W,
                                                    const uint32_t (&VAL)[WPT], uint32_t (&AL)[WPT], bool do_al,
                                                    uint32_t* hist, int Wpad, uint32_t& bad_or) {
    constexpr int RG = 4;
    uint32_t zflag = 0;
#pragma unroll
    for (int h = 0; h < BMAX; h += RG) {
        if (h < nrows) {
            uint32_t w[RG][WPT];
#pragma unroll
            for (int g = 0; g < RG; ++g) {
                const int b = h + g;
                if (b < nrows) {
                    const uint8_t* srow = TMA ? ring + (size_t)(st0 + b) * p.rs : nullptr;
                    fetch_words<WPT, U8, TMA>(srow, rows_base + (size_t)b * p.ld_bytes, tau, W, p.cols, p.rs, VAL,
                                              w[g], bad_or);
                } else {
#pragma unroll
                    for (int k = 0; k < WPT; ++k) w[g][k] = VAL[k];
                }
            }
#pragma unroll
            for (int g = 0; g < RG; ++g) {
                const int b = h + g;
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    zflag |= w[g][k] != VAL[k] ? (1u << (k * BMAX + b)) : 0u;  // word-major
                    if (do_al) {
                        AL[k] &= w[g][k];
                        if (hist && b < nrows) hist[b * Wpad + tau * WPT + k] = AL[k];
                    }
                }
            }
        }
    }
    return zflag;
}

// Lean form of tile_zero_flags for bit-packed TMA-staged rows (CTA teams):
// per row one vector smem load and one "any zero in my words" flag; the
// per-word flags are rebuilt only for the (few) rows that had a zero.
// ring_s = shared address of the thread's words in ring stage 0, inv = ~valid
// mask per word.
template <int WPT, bool DO_AL>
__device__ __forceinline__ uint32_t tile_zero_flags_bits(uint32_t ring_s, int rs, int st0, int nrows, bool active,
                                                         const uint32_t (&inv)[WPT], uint32_t (&AL)[WPT],
                                                         unsigned long long* trp = nullptr) {
    constexpr int RG = 4;
    uint32_t rowflag = 0;
    const uint32_t base = ring_s + (uint32_t)(st0 * rs);
#pragma unroll
    for (int h = 0; h < BMAX; h += RG) {
        if (h < nrows) {
            uint32_t w[RG][WPT];
#pragma unroll
            for (int g = 0; g < RG; ++g) {
                if (h + g < nrows && active) {
                    lds_words<WPT>(base + (uint32_t)((h + g) * rs), w[g]);
                } else {
#pragma unroll
                    for (int k = 0; k < WPT; ++k) w[g][k] = 0xFFFFFFFFu;
                }
            }
#pragma unroll
            for (int g = 0; g < RG; ++g) {
                uint32_t all = 0xFFFFFFFFu;
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    all &= w[g][k] | inv[k];
                    if (DO_AL) AL[k] &= w[g][k];
                }
                rowflag |= all != 0xFFFFFFFFu ? (1u << (h + g)) : 0u;
            }
        }
    }
    if (trp) *trp = (unsigned long long)clock64();
    uint32_t zflag = 0;
    while (rowflag) {  // rows with a zero somewhere in the thread's words
        const int b = __ffs(rowflag) - 1;
        rowflag &= rowflag - 1;
        uint32_t w[WPT];
        lds_words<WPT>(base + (uint32_t)(b * rs), w);
#pragma unroll
        for (int k = 0; k < WPT; ++k) zflag |= (w[k] | inv[k]) != 0xFFFFFFFFu ? (1u << (k * BMAX + b)) : 0u;
    }
    return zflag;
}

// ============================================================= pass 1 kernel
// Tile kinds: CLIMB (t >= rho: heights <= rho, so E = prefix-AND of the band
// top when t == rho; 1 row per tile, one warp finds the leftmost window),
// S (t < tl: bit-sliced counters), L (t >= tl: word-level F filter).
// Rows stream through the TMA ring; refills are issued by lane 0 of the last
// warp of the team right after the tile's first barrier (that warp is idle
// during most of phase B).
template <int WPT, bool U8, bool TMA, bool SUB>
__global__ void __launch_bounds__(512, 1) pass1_kernel(const Pass1Params p) {
    extern __shared__ __align__(128) uint8_t smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the seed / strip pass
    if (!SUB && p.redo && ld_volatile(p.redo + blockIdx.x) == 0) return;  // done by strip_kernel
    const int NT = p.team;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int team_idx = SUB ? tid / NT : 0;
    const int tau = SUB ? tid - team_idx * NT : tid;
    const unsigned tmask =
        SUB ? (unsigned)((NT >= 32 ? 0xFFFFFFFFull : ((1ull << NT) - 1ull)) << (lane - (tau & 31))) : 0xFFFFFFFFu;
    const int teams_per_cta = SUB ? p.teams_per_cta : 1;
    const int unit = blockIdx.x * teams_per_cta + team_idx;
    if (SUB && (team_idx >= teams_per_cta || unit >= p.units)) return;
    const int band = unit % p.nbands;
    const int mat = unit / p.nbands;
    const int W = p.W;
    const int Wpad = NT * WPT;
    const int nfw = (Wpad + 31) / 32;
    const bool nfw_pow2 = (nfw & (nfw - 1)) == 0;
    const int nfw_sh = __ffs(nfw) - 1;
    const int fstride = r16(nfw * 4) / 4;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    const int P = U8 ? p.zplanes : 0;  // bit planes only for u8 inputs
    unsigned char* result = p.results + (size_t)mat * 32;

    const P1Layout Lo = p1_layout(NT, WPT, p.nstage, p.rs, p.bs, P, TMA, !SUB);
    uint8_t* tsm = smem + (size_t)team_idx * p.layout_bytes;
    uint8_t* ring = tsm + Lo.ring;
    uint64_t* bars = (uint64_t*)(tsm + Lo.bars);
    uint32_t* zp = (uint32_t*)(tsm + Lo.zp);  // bit-sliced last-zero rows
    uint32_t* ab = (uint32_t*)(tsm + Lo.ab);  // prefix-AND of the band top, row above the tile
    uint16_t* za = (uint16_t*)(tsm + Lo.za);
    uint32_t* nzm = (uint32_t*)(tsm + Lo.nzm);
    uint16_t* zg = p.zb + (size_t)unit * p.cols_pad;  // bits inputs: global last-zero rows
    uint32_t* hist = (uint32_t*)(tsm + Lo.hist);
    uint32_t* fmap = (uint32_t*)(tsm + Lo.fmap);
    Misc* misc = (Misc*)(tsm + Lo.misc);
    const uint8_t* mbase = p.src + (size_t)mat * p.batch_stride;
    const size_t sum_base = (size_t)band * p.cols_pad;
    const uint64_t pol = TMA ? l2_evict_first_policy() : 0ull;
    // TMA issuer: lane 0 of the last warp of the team (idle during most of phase B)
    const int issuer = SUB ? 0 : NT - 32;
    static_assert(sizeof(Pass1Exact<U8, TMA>) <= sizeof(Misc::ex), "Misc::ex too small");
    Pass1Exact<U8, TMA>* exs = reinterpret_cast<Pass1Exact<U8, TMA>*>(misc->ex);
    if (tau == 0)
        *exs = Pass1Exact<U8, TMA>{zp, zg, za, nzm, ring, mbase, p.ld_bytes, W, p.cols, p.rs, p.nstage, P, WPT, NT,
                                   Wpad, 0, r0, 0};

    // ---- setup
    for (int i = tau; i < P * Wpad; i += NT) zp[i] = 0u;
    for (int i = tau; i < Wpad; i += NT) {
        ab[i] = valid_mask(i, W, p.cols);
        nzm[i] = valid_mask(i, W, p.cols);
        za[i] = 0;
    }
    for (int i = tau; i < 2 * BMAX * fstride; i += NT) fmap[i] = 0u;
    if (tau == 0) {
        misc->res[0] = misc->res[1] = misc->res[2] = RES_INF;
        for (int i = 0; i < 8; ++i) misc->pad[i] = 0;
        misc->g = p.share ? ld_volatile(res_best(result)) : 0;
        if (MSQ_ABLATE & 16) misc->g = max(misc->g, 120);
        if (TMA) {
            for (int s = 0; s < p.nstage / p.bl; ++s) mbar_init(&bars[s], 1);
            fence_mbar_init();
        }
    }
    auto csync = [&]() { tsync<SUB>(tmask); };
    csync();

    // TMA ring of slots: SR = p.bl consecutive band rows per slot, one mbarrier
    // per slot, one bulk copy per slot when the rows are contiguous in memory
    // (else one copy per row, all on the slot's barrier).  Tiles never straddle
    // a slot; a slot is refilled once every row of it went through phase C.
    const int SR = p.bl;
    const int nslots = TMA ? p.nstage / SR : 1;
    auto issue_slot = [&](int first) {
        const int sl = (first / SR) % nslots;
        const int n = min(SR, H - first);
        mbar_expect_tx(&bars[sl], (uint32_t)(n * p.row_bytes));
        uint8_t* dst = ring + (size_t)sl * SR * p.rs;
        const uint8_t* srcp = mbase + (size_t)(r0 + first) * p.ld_bytes;
        if (p.ld_bytes == (long long)p.rs && p.rs == p.row_bytes) {
            tma_row(dst, srcp, (uint32_t)(n * p.row_bytes), &bars[sl], pol);
        } else {
            for (int q = 0; q < n; ++q)
                tma_row(dst + (size_t)q * p.rs, srcp + (size_t)q * p.ld_bytes, (uint32_t)p.row_bytes, &bars[sl], pol);
        }
    };
    int slot_no = 0, slot_idx = 0;  // slot of the current tile: band slot number, ring slot
    uint32_t slot_par = 0u;         // its mbarrier phase parity
    int issued = 0;  // issuer: first band row not yet staged (a multiple of SR)
    if (TMA && tau == issuer)
        for (; issued < H && issued < p.nstage; issued += SR) issue_slot(issued);

    uint32_t VAL[WPT], EPREV[WPT], AL[WPT];  // never-zeroed masks live in smem (nzm)
    int ZW[WPT];
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
        VAL[k] = valid_mask(tau * WPT + k, W, p.cols);
        AL[k] = VAL[k];
        EPREV[k] = 0;
        ZW[k] = 0;
    }

    // side effects of the zeros of own word k at row rho: last-zero rows
    // (optional), first zeros (e_out) and the never-zeroed masks
    auto apply_event = [&](uint32_t& nzk, const uint32_t valk, int zi, int a, int rho, uint32_t zeros, bool do_z) {
        uint32_t newly = nzk & zeros;
        if (do_z) {
            if (U8) {
                zplanes_set(zp, zi, Wpad, P, zeros, rho);
            } else if (zeros == valk) {
                za[a] = (uint16_t)rho;  // whole word zero: lazy row; first zeros read as <= za
                uint32_t nn = newly;
                while (nn) {
                    const int j = __ffs(nn) - 1;
                    nn &= nn - 1;
                    zg[(size_t)a * 32 + j] = 0;
                }
            } else {
                uint32_t zz = zeros;
                while (zz) {
                    const int j = __ffs(zz) - 1;
                    zz &= zz - 1;
                    zg[(size_t)a * 32 + j] = (uint16_t)rho;
                }
            }
        }
        if (newly) {
            if (p.write_summaries) {
                const size_t cb = sum_base + (size_t)a * 32;
                while (newly) {
                    const int j = __ffs(newly) - 1;
                    newly &= newly - 1;
                    p.e_out[cb + j] = (uint16_t)(rho - 1);
                }
            }
            nzk &= ~zeros;
            nzm[a] = nzk;
        }
    };

    uint32_t INV[WPT];  // ~valid mask per word (lean bits row loop)
#pragma unroll
    for (int k = 0; k < WPT; ++k) INV[k] = ~VAL[k];
    const uint32_t ring_s0 = smem_addr(ring);
    const uint32_t ring_s = ring_s0 + (uint32_t)(tau * WPT * 4);
    const uint32_t bars_s = smem_addr(bars);
    const uint32_t lastval = valid_mask(W - 1, W, p.cols);  // the only word that may be partial
    uint32_t fullk = 0;  // words whose 32 columns are all valid (only those can be F)
#pragma unroll
    for (int k = 0; k < WPT; ++k) fullk |= (VAL[k] == 0xFFFFFFFFu ? 1u : 0u) << k;

    int t = max(1, misc->g);
    bool full_next = false;
    bool climbL = false;  // every row of the previous mode-L tile raised
    int climb_s = 0;
    unsigned long long bandkey = 0ull;
    int round_ctr = 0;
    uint32_t bad_or = 0;
    int tile = 0;
    long long tB = p.prof ? clock64() : 0;  // profiling: end of phase B of this warp
    // optional per-phase cycle counters (thread 0): smem for CTA teams, global for sub-warp teams
    unsigned long long* pc = SUB ? (p.prof ? p.prof + (size_t)unit * 16 : nullptr)
                                 : (unsigned long long*)(tsm + Lo.pcs);
    const bool prof = p.prof != nullptr && tau == 0;
    if (prof)
        for (int i = 0; i < 16; ++i) pc[i] = 0;
    long long ck = prof ? clock64() : 0;
    // debug timeline (builds with -DMSQ_TRACE only): band 0, tiles [TR_T0, TR_T0+8),
    // lane 0 of every warp, 16 stamps per tile kept in registers, stored at the tile end
    constexpr int TR_T0 = 40;
#ifdef MSQ_TRACE
    unsigned long long* trace = p.prof ? p.prof + (size_t)p.units * 16 : nullptr;
    long long trv[16];
#define MSQ_TR(i) { trv[i] = clock64(); }
#define MSQ_TR_FLUSH()                                                                                    \
    if (trace && unit == 0 && tile >= TR_T0 && tile < TR_T0 + 8 && lane == 0)                            \
        for (int q = 0; q < 16; ++q)                                                                      \
            trace[(((size_t)(tile - TR_T0) * (NT >> 5) + (tau >> 5)) * 16) + q] = (unsigned long long)trv[q];
#else
    unsigned long long* trace = nullptr;
#define MSQ_TR(i) {}
#define MSQ_TR_FLUSH() {}
#endif
#define MSQ_CK(i)                               \
    if (prof) {                                 \
        const long long c1 = clock64();         \
        pc[i] += (unsigned long long)(c1 - ck); \
        ck = c1;                                \
    }

    for (int row0 = 0; row0 < H; ++tile) {
        MSQ_TR(0)
        const int rho0 = row0 + 1;
        const bool climb = t >= rho0 && (SUB || t < p.tl);  // large t: mode L handles rho == t rows too
        const bool modeL = !climb && t >= p.tl;
        const bool modeS = !climb && !modeL;
        const int slot_row0 = slot_no * SR;  // slot_no = row0 / SR (kept incrementally)
        const int nrows = min(min(climb ? (SUB ? 1 : p.bl) : (modeL ? p.bl : p.bs), H - row0), slot_row0 + SR - row0);
        uint32_t* fm = fmap + (tile & 1) * BMAX * fstride;
        int polled = 0;
        const bool poll = p.share && ((tile & 7) == 7 || (!climb && !modeL));
        if (poll && tau == 0) polled = ld_volatile(res_best(result));

        // ---------------------------------------------------- phase A
        uint32_t dirty = 0, zflag = 0;
        const int st0 = TMA ? slot_idx * SR + (row0 - slot_row0) : 0;  // ring stage of tile row 0
        if (TMA && row0 == slot_row0)  // first tile of a slot: wait for its rows (every thread)
            mbar_wait(&bars[slot_idx], slot_par);
        MSQ_TR(12)
        if (tau == 0) {  // read only after barrier A; the previous tile's readers passed a barrier
            exs->tile_row0 = row0;
            exs->st0 = st0;
        }
        if (!climb && !modeL) {  // ---- mode S (small threshold): E rows for the tests
#pragma unroll
            for (int b = 0; b < BMAX; ++b) {
                if (b < nrows) {
                    const int r = row0 + b;
                    const int rho = r + 1;
                    const uint8_t* srow = nullptr;
                    if (TMA) srow = ring + (size_t)(st0 + b) * p.rs;
                    uint32_t w[WPT];
                    fetch_words<WPT, U8, TMA>(srow, mbase + (size_t)(r0 + r) * p.ld_bytes, tau, W, p.cols, p.rs,
                                              VAL, w, bad_or);
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        const bool z = w[k] != VAL[k];
                        zflag |= (z ? 1u : 0u) << (k * BMAX + b);  // word-major
                        AL[k] &= w[k];
                        const int zi = k * NT + tau;
                        const int lim = rho - t;
                        uint32_t e;
                        if (U8) {
                            if (z) zplanes_set(zp, zi, Wpad, P, VAL[k] & ~w[k], rho);
                            e = (lim >= (1 << P) ? 0xFFFFFFFFu : planes_le(zp, zi, Wpad, P, lim)) & VAL[k];
                        } else {  // bits inputs, small threshold: slow path through global z
                            const int a = tau * WPT + k;
                            uint32_t nzk = nzm[a];
                            if (z) apply_event(nzk, VAL[k], k * NT + tau, a, rho, VAL[k] & ~w[k], true);
                            e = bits_small_e(zg, za[a], a, nzk, VAL[k], lim);
                        }
                        if (e & ~EPREV[k]) dirty |= 1u << (b * WPT + k);
                        EPREV[k] = e;
                        hist[b * Wpad + tau * WPT + k] = e;
                    }
                }
            }
        } else {  // ---- climb / mode L: per word one zero test, the last-zero row, F
            if (!U8 && TMA && !SUB) {
                const long long ta0 = p.prof ? clock64() : 0;
                zflag = modeL ? tile_zero_flags_bits<WPT, false>(ring_s, p.rs, st0, nrows, tau * WPT < W, INV, AL)
                              : tile_zero_flags_bits<WPT, true>(ring_s, p.rs, st0, nrows, tau * WPT < W, INV, AL);
                MSQ_TR(11)
                if (p.prof && lane == 0) {
                    atomicMax(&misc->pad[5], (int)(clock64() - ta0));
                    atomicMax(&misc->pad[6], (int)(ta0 - tB));
                }
                MSQ_TR(1)
            } else {
                zflag = tile_zero_flags<WPT, U8, TMA>(p, ring, mbase + (size_t)(r0 + row0) * p.ld_bytes, st0, nrows,
                                                      tau, W, VAL, AL, true, SUB && !modeL ? hist : nullptr, Wpad,
                                                      bad_or);
            }
            if (modeL && !(MSQ_ABLATE & 4)) {
                // F words of row b: zero-free since rho_b - t, i.e. no zero in
                // the tile up to row b and last zero before the tile <= rho0 + b - t:
                // one row interval [lo, hi) per word
                uint32_t fr[WPT], any = 0;
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    const uint32_t zb = (zflag >> (k * BMAX)) & ((1u << BMAX) - 1u);
                    const int hi = zb ? __ffs(zb) - 1 : nrows;
                    const int lo = max(0, ZW[k] + t - rho0);
                    fr[k] = (fullk >> k) & 1u && lo < hi ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
                    any |= fr[k];
                }
                const int a0 = tau * WPT;
                if (!SUB) {
                    // the 32/WPT lanes that own one F word OR their bits together
                    // and one of them stores it (no atomics, no clearing)
                    constexpr int LPF = 32 / WPT;
                    // WPT == 4: the 4x8 bit matrix (word k, row b) as bytes of X; the
                    // nibble of row b = bits b, 8+b, 16+b, 24+b gathered by one multiply
                    uint32_t X = 0;
                    if (WPT == 4) X = fr[0] | (fr[(1) % WPT] << 8) | (fr[(2) % WPT] << 16) | (fr[(3) % WPT] << 24);
#pragma unroll
                    for (int b = 0; b < BMAX; ++b) {
                        if (b < nrows) {
                            uint32_t v = 0;
                            if (WPT == 4) {
                                v = (((X >> b) & 0x01010101u) * 0x01020408u) >> 24;
                            } else {
#pragma unroll
                                for (int k = 0; k < WPT; ++k) v |= ((fr[k] >> b) & 1u) << k;
                            }
                            v <<= (a0 & 31);
#pragma unroll
                            for (int o = 1; o < LPF; o <<= 1) v |= __shfl_xor_sync(0xFFFFFFFFu, v, o);
                            if ((lane & (LPF - 1)) == 0) fm[b * fstride + (a0 >> 5)] = v;
                        }
                    }
                } else {
                    while (any) {
                        const int b = __ffs(any) - 1;
                        any &= any - 1;
                        uint32_t fn = 0;
#pragma unroll
                        for (int k = 0; k < WPT; ++k) fn |= ((fr[k] >> b) & 1u) << k;
                        atomicOr(&fm[b * fstride + (a0 >> 5)], fn << (a0 & 31));
                    }
                }
            }
        }
        MSQ_TR(13)
        // last zero row of each word after the tile
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const uint32_t zb = (zflag >> (k * BMAX)) & ((1u << BMAX) - 1u);
            if (zb) ZW[k] = rho0 + 31 - __clz(zb);
        }
        if (tau == 0 && poll) misc->g = polled;
        if (p.prof && lane == 0) atomicMax(&misc->pad[4], (int)(clock64() - tB));
        MSQ_TR(2)
        MSQ_CK(0)
        csync();  // (A)
        MSQ_TR(3)
        MSQ_CK(1)
        if (prof) {
            pc[4] += misc->pad[3];
            pc[9] += misc->pad[4];
            pc[12] += misc->pad[5];
            pc[14] += misc->pad[6];
            misc->pad[3] = misc->pad[4] = misc->pad[5] = misc->pad[6] = 0;
        }
        const long long ti0 = p.prof ? clock64() : 0;
        if (TMA && tau == issuer)  // slots below the current one are consumed: refill them
            for (; issued < H && issued < slot_row0 + p.nstage; issued += SR) issue_slot(issued);
        if (p.prof && tau == issuer) atomicAdd(&misc->pad[7], (int)(clock64() - ti0));
        MSQ_TR(4)
        MSQ_CK(2)

        // ---------------------------------------------------- phase B
        const int lastb = nrows - 1;
        int cur_t = t;
        const Pass1Exact<U8, TMA>& ex = *exs;
        if (climb && SUB) {
            if (t == rho0) {  // E = prefix-AND of the band top; leftmost t-window
                uint32_t best = RES_INF;
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    const int a = tau * WPT + k;
                    if (a < W) test_word_full(hist, Wpad, W, 0, 0, a, t, best);
                }
                const int slot = round_ctr % 3;
                if (best != RES_INF) atomicMin(&misc->res[slot], best);
                if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
                csync();  // (B)
                const uint32_t rr = misc->res[slot];
                ++round_ctr;
                if (rr != RES_INF) {
                    const int start = (int)(rr & 0xFFFFFu);
                    if (tau == 0) {
                        bandkey = pack_key(t, p.row_base + r0 + row0, start + t - 1);
                        if (p.share) atomicMax(res_best(result), t);
                    }
                    cur_t = t + 1;
                }
            }
        } else if (climb) {
            // heights are <= rho, so the only rows with a test are rho >= t; a
            // test at rho == t asks for a t-window in the prefix-AND A(rho), and
            // success is monotone in rho: test every row of the tile in parallel
            // (warp w takes row bfirst + w) and keep the last success.
            const int bfirst = (MSQ_ABLATE & 8) ? BMAX : t - rho0;
            if (bfirst <= lastb) {
                // the issuer's warp (last) is busy with the refill: rows go to the others
                const int wid = tid >> 5, nwarps = TMA && NT > 32 ? (NT >> 5) - 1 : (NT >> 5);
                for (int b = bfirst + wid; wid < nwarps && b <= lastb; b += nwarps) {
                    const int st = climb_scan<U8, TMA>(ab, &ex, b, W, climb_s, rho0 + b, lane);
                    if (lane == 0) misc->cres[b - bfirst] = st;
                }
                csync();  // (B)

                int nsucc = 0, last_start = -1;
                for (int w2 = 0; w2 <= lastb - bfirst; ++w2) {
                    const int st = misc->cres[w2];
                    if (st < 0) break;
                    ++nsucc;
                    last_start = st;
                }
                if (nsucc > 0) {
                    cur_t = t + nsucc;  // rows rho0+bfirst .. +nsucc-1 raised once each
                    if (tau == 0) {
                        bandkey = pack_key(cur_t - 1, p.row_base + r0 + row0 + bfirst + nsucc - 1,
                                           last_start + cur_t - 2);
                        if (p.share) atomicMax(res_best(result), cur_t - 1);
                    }
                    climb_s = last_start;
                }
                // rows after the failing row are general rows: exact E at cur_t
                for (int bg = bfirst + nsucc + 1; bg <= lastb; ++bg) {
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        const int a = tau * WPT + k;
                        hist[a] = a < W ? exact_row_mask<U8, TMA>(&ex, a, bg, cur_t) : 0u;
                    }
                    csync();
                    uint32_t best = RES_INF;
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        const int a = tau * WPT + k;
                        if (a < W) test_word_full(hist, Wpad, W, 0, 0, a, cur_t, best);
                    }
                    const int slot = round_ctr % 3;
                    if (best != RES_INF) atomicMin(&misc->res[slot], best);
                    if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
                    csync();
                    const uint32_t rr = misc->res[slot];
                    ++round_ctr;
                    if (rr != RES_INF) {
                        const int col = (int)(rr & 0xFFFFFu);
                        if (tau == 0) {
                            bandkey = pack_key(cur_t, p.row_base + r0 + row0 + bg, col + cur_t - 1);
                            if (p.share) atomicMax(res_best(result), cur_t);
                        }
                        ++cur_t;
                    }
                }
            }
        } else {
            // climbing (the previous mode-L tile raised on every row): test the
            // last row at t + lastb first -- success implies a raise on every
            // row (a square of side t + lastb ending there contains one of side
            // t + b ending at row b), and its window is the last raise
            bool spec = modeL && climbL && lastb > 0;
            int start_b = spec ? lastb : 0, full_from = full_next ? 0 : BMAX;
            if (spec) cur_t = t + lastb;
            bool round_ctr_first = true;
            for (;;) {
                uint32_t best = RES_INF;
                const int m = cur_t - t;
                const long long rc0 = p.prof ? clock64() : 0;
                if (modeL) {
                    // CTA teams with bits inputs (last-zero rows in L2) queue up to
                    // two candidates per lane for the warp-cooperative check (one
                    // L2 round trip per candidate instead of a serial chain per
                    // lane) when the warp has few; otherwise, and for every u8
                    // candidate (smem planes), the lane checks its own
                    constexpr uint32_t NONE = 0xFFFFFFFFu;
                    constexpr bool COOP = !SUB && !U8;
                    uint32_t cq0 = NONE, cq1 = NONE;
                    auto direct = [&](int cb, int a0, int len) {
                        const int bl2 = ex.boundary_len(a0 - 1, a0 + len, cb, cur_t);
                        const int suf = bl2 & 0xFF;
                        if (suf + (bl2 >> 8) + 32 * len >= cur_t) best = min(best, enc_res(cb, 32 * a0 - suf));
                    };
                    const int n = (MSQ_ABLATE & 2) ? 0 : (lastb - start_b + 1) * nfw;
                    const int nscan = TMA && NT > 32 ? NT - 32 : NT;  // not the issuer's warp
                    for (int idx = tau; idx < n && tau < nscan; idx += nscan) {
                        const int b = start_b + (nfw_pow2 ? idx >> nfw_sh : idx / nfw);
                        const int fw = nfw_pow2 ? idx & (nfw - 1) : idx % nfw;
                        scan_fword(fm, fstride, W, b, m, fw, cur_t, [&](int cb, int a0, int len) {
                            if (p.prof) atomicAdd(&misc->pad[0], 1);
                            const uint32_t cand = (uint32_t)cb | ((uint32_t)a0 << 3) | ((uint32_t)len << 14);
                            if (COOP && cq0 == NONE) {
                                cq0 = cand;
                            } else if (COOP && cq1 == NONE) {
                                cq1 = cand;
                            } else {
                                direct(cb, a0, len);
                            }
                        });
                    }
                    if (p.prof && lane == 0) atomicMax(&misc->pad[2], (int)(clock64() - rc0));
                    if (round_ctr_first) MSQ_TR(5)
                    if (COOP) {
                        const uint32_t bal0 = __ballot_sync(0xFFFFFFFFu, cq0 != NONE);
                        const uint32_t bal1 = __ballot_sync(0xFFFFFFFFu, cq1 != NONE);
                        if (__popc(bal0) + __popc(bal1) <= 4) {
#pragma unroll
                            for (int qi = 0; qi < 2; ++qi) {
                                const uint32_t mine = qi ? cq1 : cq0;
                                uint32_t bal = qi ? bal1 : bal0;
                                while (bal) {
                                    const int l = __ffs(bal) - 1;
                                    bal &= bal - 1;
                                    const uint32_t cand = __shfl_sync(0xFFFFFFFFu, mine, l);
                                    const uint32_t r = coop_check<U8, TMA>(exs, cand, cur_t, lane);
                                    if (lane == l) best = min(best, r);
                                }
                            }
                        } else {  // many candidates in this warp: lanes in parallel
#pragma unroll
                            for (int qi = 0; qi < 2; ++qi) {
                                const uint32_t cand = qi ? cq1 : cq0;
                                if (cand != NONE)
                                    direct((int)(cand & 7u), (int)((cand >> 3) & 0x7FFu), (int)(cand >> 14));
                            }
                        }
                    }
                } else {
                    best = test_rows_s(hist, Wpad, W, WPT, tau, start_b, lastb, full_from, dirty, m, cur_t);
                }
                if (round_ctr_first) MSQ_TR(6)
                const int slot = round_ctr % 3;
                if (best != RES_INF) atomicMin(&misc->res[slot], best);
                if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
                if (p.prof && modeL && lane == 0) atomicMax(&misc->pad[1], (int)(clock64() - rc0));
                if (round_ctr_first) MSQ_TR(7)
                if (prof && modeL) pc[7] += 1;
                csync();  // (B)
                if (round_ctr_first) MSQ_TR(8)
                round_ctr_first = false;
                if (prof && modeL) {
                    pc[13] += misc->pad[1];
                    pc[15] += misc->pad[2];
                    misc->pad[1] = misc->pad[2] = 0;
                }
                const uint32_t rr = misc->res[slot];
                ++round_ctr;
                if (spec) {
                    spec = false;
                    if (rr == RES_INF) {  // not a full climb: the tile's normal rounds
                        cur_t = t;
                        start_b = 0;
                        continue;
                    }
                }
                if (rr == RES_INF) break;
                const int bs_ = (int)(rr >> 20), col = (int)(rr & 0xFFFFFu);
                if (tau == 0) {
                    bandkey = pack_key(cur_t, p.row_base + r0 + row0 + bs_, col + cur_t - 1);
                    if (p.share) atomicMax(res_best(result), cur_t);
                }
                ++cur_t;
                start_b = bs_ + 1;
                full_from = bs_ + 1;
                if (start_b > lastb) break;
            }
        }
        if (prof && climb && t - rho0 <= lastb) pc[13] += 0;
        if (prof) {
            const int kind = climb ? 0 : (modeL ? 2 : 1);
            if (kind == 0) pc[8] += 1;
            pc[11] += cur_t - t;
            const long long c1 = clock64();
            if (kind != 1) pc[3 + kind] += (unsigned long long)(c1 - ck);
            ck = c1;
        }
        MSQ_TR(14)
        climbL = modeL && !climb && cur_t - t == nrows;
        const bool raised = cur_t != t;
        t = cur_t;
        bool jumped = false;
        if (p.share) {
            const int g = misc->g;
            if (g > t) {
                t = g;
                jumped = true;
            }
        }
        full_next = raised || jumped || climb;
        if (!climb || !raised) climb_s = 0;
#pragma unroll
        for (int k = 0; k < WPT; ++k) ab[tau * WPT + k] = AL[k];

        // ---------------------------------------------------- phase C
        MSQ_TR(9)
        tB = p.prof ? clock64() : 0;
        // last-zero rows (bit-sliced) and first zeros, in row order per word
        // one loop over all (word, row) events of the thread (word-major, so
        // rows stay in order per word); the word's state is selected with
        // compile-time indices so VAL/NZ stay in registers
        if ((!modeS || U8) && !(MSQ_ABLATE & 1)) {
            uint32_t zf = zflag;
            while (zf) {
                const int bit = __ffs(zf) - 1;
                zf &= zf - 1;
                const int k = bit / BMAX, b = bit % BMAX;
                const int a = tau * WPT + k;
                const uint32_t valk = a == W - 1 ? lastval : 0xFFFFFFFFu;  // events only occur in valid words
                uint32_t nzk = nzm[a];
                const int r = row0 + b, rho = r + 1;
                uint32_t wv;
                if (TMA && !U8) {  // the tile's rows never wrap the ring (slots)
                    uint32_t w1[1];
                    lds_words<1>(ring_s0 + (uint32_t)((st0 + b) * p.rs + a * 4), w1);
                    wv = w1[0];
                } else {
                    const uint8_t* srow = TMA ? ring + (size_t)(st0 + b) * p.rs : nullptr;
                    wv = word_of_row<U8, TMA>(srow, mbase + (size_t)(r0 + r) * p.ld_bytes, a, p.cols, p.rs);
                }
                apply_event(nzk, valk, k * NT + tau, a, rho, valk & ~wv, !modeS);

            }
        }
        if (modeL && SUB)  // sub-warp teams build F with atomics: clear for the reuse
            for (int i = tau; i < BMAX * fstride; i += NT) fm[i] = 0u;
        MSQ_CK(6)
        MSQ_TR(10)
        MSQ_TR_FLUSH()
        if (p.prof && lane == 0) atomicMax(&misc->pad[3], (int)(clock64() - tB));
        if (p.prof) tB = clock64();  // end of phase C
        row0 += nrows;
        if (row0 == slot_row0 + SR) {  // next slot
            ++slot_no;
            if (++slot_idx == nslots) {
                slot_idx = 0;
                slot_par ^= 1u;
            }
        }
    }
#undef MSQ_CK
#undef MSQ_TR
#undef MSQ_TR_FLUSH
    csync();
    if (prof) {
        pc[10] = misc->pad[7];
        if (!SUB)
            for (int i = 0; i < 16; ++i) p.prof[(size_t)unit * 16 + i] = pc[i];
    }
    csync();

    // ---------------------------------------------------------- band outputs
    if (p.write_summaries && !(MSQ_ABLATE & 32)) {
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            if (a < W) {
                const size_t cb = sum_base + (size_t)a * 32;
                const uint32_t nz = nzm[a];
                if (nz) {  // never-zeroed columns: e = H (16-byte merges of the first-zero rows)
                    uint4* eq = (uint4*)(p.e_out + cb);
                    uint4 evs[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {  // all loads first (one round trip)
                        const uint32_t nq = (nz >> (8 * q)) & 0xFFu;
                        evs[q] = nq == 0u || nq == 0xFFu ? make_uint4(0, 0, 0, 0) : eq[q];
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t nq = (nz >> (8 * q)) & 0xFFu;
                        if (!nq) continue;
                        const uint4 ev = evs[q];
                        uint32_t v[4] = {ev.x, ev.y, ev.z, ev.w};
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            if ((nq >> (2 * h)) & 1u) v[h] = (v[h] & 0xFFFF0000u) | (uint32_t)H;
                            if ((nq >> (2 * h + 1)) & 1u) v[h] = (v[h] & 0xFFFFu) | ((uint32_t)H << 16);
                        }
                        eq[q] = make_uint4(v[0], v[1], v[2], v[3]);
                    }
                }
                if (U8) {
                    band_bottom_runs(zp, k * NT + tau, Wpad, P, H, p.zb + (size_t)unit * p.cols_pad + (size_t)a * 32);
                } else {  // bottom runs overwrite the global last-zero rows in place
                    const int zaa = za[a];
                    uint4* zq = (uint4*)(zg + (size_t)a * 32);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 zv = zq[q];
                        const uint32_t pr[4] = {zv.x, zv.y, zv.z, zv.w};
                        uint32_t v[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const int j0 = 8 * q + 2 * h;
                            const int u0 = ((nz >> j0) & 1u) ? 0 : max((int)(pr[h] & 0xFFFFu), zaa);
                            const int u1 = ((nz >> (j0 + 1)) & 1u) ? 0 : max((int)(pr[h] >> 16), zaa);
                            v[h] = (uint32_t)(H - u0) | ((uint32_t)(H - u1) << 16);
                        }
                        zq[q] = make_uint4(v[0], v[1], v[2], v[3]);
                    }
                }
                p.ao_out[(size_t)band * W + a] = nz;
            }
        }
    }
    if (U8 && (bad_or & 0xFEFEFEFEu)) atomicOr(res_status(result), 1u);
    if (tau == 0) {
        if (p.band_keys) p.band_keys[unit] = bandkey;
        if (bandkey) atomicMax(res_key1(result), bandkey);
    }
}

// ============================================================ fix-up kernel
// virtual band top: column j has height c_j + d at depth d while d <= e_j.
// us/e8 are word-major (us[a*32 + j]).
struct FixExact {
    const uint16_t* us;   // c clamped to 65535
    const uint8_t* e8;    // e clamped to 255
    const uint16_t* e_g;  // exact e (global) for this band
    int W, cols;
    int d0;               // depth of tile row 0
    __device__ __forceinline__ bool elig(int idx, int d, int T) const {
        int e = e8[idx];
        if (e == 255 && d > 255) e = e_g[idx];
        return e >= d && (int)us[idx] + d >= T;
    }
    __device__ uint32_t mask(int a, int b, int T) const {
        const uint32_t val = valid_mask(a, W, cols);
        const int d = d0 + b;
        uint32_t m = 0;
        const uint4* up = (const uint4*)(us + (size_t)a * 32);
        const uint4* ep = (const uint4*)(e8 + (size_t)a * 32);
        const uint4 e0 = ep[0], e1 = ep[1];
        const uint32_t ew[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = up[q];
            const uint32_t pr[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int j = 8 * q + 2 * h + s;
                    int e = (int)((ew[j >> 2] >> (8 * (j & 3))) & 0xFFu);
                    if (e == 255 && d > 255) e = e_g[(size_t)a * 32 + j];
                    const int c = (int)((pr[h] >> (16 * s)) & 0xFFFFu);
                    m |= ((e >= d && c + d >= T) ? 1u : 0u) << j;
                }
            }
        }
        return m & val;
    }
    __device__ uint32_t coop_mask(int a, int b, int T, int lane) const {
        const uint32_t val = valid_mask(a, W, cols);
        const bool el = ((val >> lane) & 1u) && elig(a * 32 + lane, d0 + b, T);
        return __ballot_sync(0xFFFFFFFFu, el);
    }
};

template <int WPT>
__global__ void __launch_bounds__(512, 1) fixup_kernel(const FixParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the carry scan
    const int NT = blockDim.x;
    const int tau = threadIdx.x;
    const int lane = tau & 31;
    const int band = p.band_begin + blockIdx.x;
    const int W = p.W;
    const int Wpad = NT * WPT;
    const int nfw = (Wpad + 31) / 32;
    const int fstride = r16(nfw * 4) / 4;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    unsigned char* result = p.results;

    const FixLayout Lo = fix_layout(NT, WPT, p.bs);
    uint16_t* us = (uint16_t*)(smem + Lo.us);
    uint8_t* e8 = smem + Lo.e8;
    uint32_t* hist = (uint32_t*)(smem + Lo.hist);
    uint32_t* fmap = (uint32_t*)(smem + Lo.fmap);
    Misc* misc = (Misc*)(smem + Lo.misc);
    const uint16_t* e_g = p.e_in + (size_t)band * p.cols_pad;

    if (tau == 0) {
        misc->res[0] = misc->res[1] = misc->res[2] = RES_INF;
        int g = (int)(*(volatile unsigned long long*)res_key1(result) >> (2 * KEY_DIM_BITS));
        if (p.share) g = max(g, ld_volatile(res_best(result)));
        misc->g = g;
    }
    for (int i = tau; i < 2 * BMAX * fstride; i += NT) fmap[i] = 0u;

    // ---- prologue: carry-in heights (carry_scan_kernel) and leading-ones
    // depths of the band top, coalesced 16-byte chunks (8 columns) per thread;
    // the 4 chunk-threads of a word combine its minima by shuffles
    uint32_t* wmin = (uint32_t*)(smem + Lo.wmin);
    {
        const uint4* cp4 = (const uint4*)(p.carry_in + (size_t)band * p.cols_pad);
        const uint4* ep4 = (const uint4*)e_g;
        uint4* us4 = (uint4*)us;
        uint2* e82 = (uint2*)e8;
        const int nchunk = Wpad * 4;  // a multiple of 4 * NT: 4 lanes per word, 4 chunks per thread in flight
        constexpr int U = 4;
        for (int i0 = tau; i0 < nchunk; i0 += U * NT) {
          uint4 c4s[U], e4s[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {  // all loads of the group first
              const int i = i0 + u * NT;
              c4s[u] = e4s[u] = make_uint4(0, 0, 0, 0);
              if ((i >> 2) < W) {
                  c4s[u] = cp4[i];
                  e4s[u] = ep4[i];
              }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = i0 + u * NT;
            const int a = i >> 2;
            const uint32_t val = valid_mask(a, W, p.cols) >> (8 * (i & 3));
            const uint4 c4 = c4s[u], e4 = e4s[u];
            us4[i] = c4;
            const uint32_t cw[4] = {c4.x, c4.y, c4.z, c4.w}, ew[4] = {e4.x, e4.y, e4.z, e4.w};
            uint32_t e8w[2] = {0u, 0u};
            int minc = 0xFFFF, mine = 0xFFFF;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = (int)((cw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
                const int e = (int)((ew[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
                const bool v = (val >> j) & 1u;
                e8w[j >> 2] |= (uint32_t)(v ? min(e, 255) : 0) << (8 * (j & 3));
                if (v) {
                    minc = min(minc, c);
                    mine = min(mine, e);
                }
            }
            e82[i] = make_uint2(e8w[0], e8w[1]);
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                minc = min(minc, __shfl_xor_sync(0xFFFFFFFFu, minc, o));
                mine = min(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, o));
            }
            if ((i & 3) == 0) wmin[a] = (uint32_t)minc | ((uint32_t)mine << 16);
          }
        }
    }
    __syncthreads();
    uint32_t VAL[WPT];
    int MINC[WPT], MINE[WPT];
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
        const int a = tau * WPT + k;
        VAL[k] = valid_mask(a, W, p.cols);
        const uint32_t mm = wmin[a];
        const bool full = VAL[k] == 0xFFFFFFFFu;  // a partial word is never F
        MINC[k] = full ? (int)(mm & 0xFFFFu) : -0x3FFFFFFF;
        MINE[k] = full ? (int)(mm >> 16) : -1;
    }
    int t = max(1, misc->g);
    FixExact ex{us, e8, e_g, W, p.cols, 1};

    // Depth filter (t >= FIX_TL): a window at depth d contains a run of at
    // least len_min words whose 32 columns are all eligible, and word a is
    // such an F word exactly on the depths [t - minc_a, mine_a].  Mark the
    // depths covered by the intersection of len_min consecutive intervals;
    // unmarked depths (and the depth-1 probe) need no test.  t only grows, so
    // marks made with the starting t stay a superset.
    const bool dfilt = t >= FIX_TL;
    uint32_t* dmark = (uint32_t*)(smem + Lo.dmark);
    if (dfilt) {
        const int nmw = (H >> 5) + 1;
        for (int i = tau; i < nmw; i += NT) dmark[i] = 0u;
        __syncthreads();
        const int len_min = max(1, (t - 63 + 31) / 32);
        const bool last_full = valid_mask(W - 1, W, p.cols) == 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            if (a >= W || VAL[k] != 0xFFFFFFFFu) continue;
            int LO = max(1, t - MINC[k]), HI = min(MINE[k], H), len = 1;
            for (int a2 = a + 1; LO <= HI && len < len_min && a2 < W; ++a2, ++len) {
                if (a2 == W - 1 && !last_full) {
                    LO = HI + 1;
                    break;
                }
                const uint32_t mm = wmin[a2];
                LO = max(LO, t - (int)(mm & 0xFFFFu));
                HI = min(HI, (int)(mm >> 16));
            }
            if (LO <= HI && len >= len_min)
                for (int d = LO; d <= HI;) {
                    const int wd = d >> 5, lo_b = d & 31, hi_b = min(31, lo_b + (HI - d));
                    const uint32_t bits = (hi_b == 31 ? 0xFFFFFFFFu : ((1u << (hi_b + 1)) - 1u)) & ~((1u << lo_b) - 1u);
                    atomicOr(&dmark[wd], bits);
                    d += hi_b - lo_b + 1;
                }
        }
        __syncthreads();
    }
    auto dmarked = [&](int d0, int n) -> bool {  // any marked depth in [d0, d0 + n)
        const int d1 = d0 + n - 1;
        for (int wd = d0 >> 5; wd <= (d1 >> 5); ++wd) {
            const int lo_b = wd == (d0 >> 5) ? (d0 & 31) : 0, hi_b = wd == (d1 >> 5) ? (d1 & 31) : 31;
            const uint32_t bits = (hi_b == 31 ? 0xFFFFFFFFu : ((1u << (hi_b + 1)) - 1u)) & ~((1u << lo_b) - 1u);
            if (dmark[wd] & bits) return true;
        }
        return false;
    };

    int round_ctr = 0;
    auto round_result = [&](uint32_t best) -> uint32_t {
        const int slot = round_ctr % 3;
        if (best != RES_INF) atomicMin(&misc->res[slot], best);
        if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
        __syncthreads();
        const uint32_t r = misc->res[slot];
        ++round_ctr;
        return r;
    };
    auto probe = [&](int T) -> uint32_t {  // full test of depth 1 at threshold T
        uint32_t ev[WPT];
        ex.d0 = 1;
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            ev[k] = a < W ? ex.mask(a, 0, T) : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < WPT; ++k) hist[tau * WPT + k] = ev[k];
        __syncthreads();
        uint32_t best = RES_INF;
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            if (a < W) test_word_full(hist, Wpad, W, 0, 0, a, T, best);
        }
        return round_result(best);
    };

    unsigned long long fixkey = 0ull;
    if (H >= 1) {
        // ---------------------------------------------- depth 1, exact seeding
        const uint32_t r = (!dfilt || dmarked(1, 1)) ? probe(t) : RES_INF;
        if (r != RES_INF) {
            int lo = t, hi = -1;
            uint32_t rlo = r;
            int step = 1;
            while (hi < 0) {
                const int kk = lo + step;
                if (kk > p.cols) {
                    hi = kk;
                    break;
                }
                const uint32_t rk = probe(kk);
                if (rk != RES_INF) {
                    lo = kk;
                    rlo = rk;
                    step *= 2;
                } else {
                    hi = kk;
                }
            }
            while (hi - lo > 1) {
                const int mid = lo + (hi - lo) / 2;
                const uint32_t rk = probe(mid);
                if (rk != RES_INF) {
                    lo = mid;
                    rlo = rk;
                } else {
                    hi = mid;
                }
            }
            if (tau == 0) {
                fixkey = pack_key(lo, p.row_base + r0, (int)(rlo & 0xFFFFFu) + lo - 1);
                if (p.share) atomicMax(res_best(result), lo);
            }
            t = lo + 1;
        }
        __syncthreads();

        // ---------------------------------------------- depths 2.. in tiles
        // Climbing (every depth of the previous tile raised): first test only
        // the tile's last depth at t + lastb.  A square of side t + lastb
        // ending there contains one of side t + i ending at depth i (drop the
        // bottom lastb - i rows and right columns), so success means every
        // depth of the tile raises in turn and this test's window is the last
        // raise -- one round instead of one per depth.  On failure the tile
        // runs its normal rounds.
        bool climbing = r != RES_INF;
        int tile = 0;
        for (int d0 = 2; d0 <= H && d0 < t; ++tile) {
            const bool modeL = t >= FIX_TL;
            const int nrows = min(modeL ? p.bl : p.bs, H - d0 + 1);
            if (dfilt && !dmarked(d0, nrows)) {  // no run of F words at these depths
                d0 += nrows;
                climbing = false;
                continue;
            }
            uint32_t* fm = fmap + (tile & 1) * BMAX * fstride;
            int polled = 0;
            if (p.share && tau == 0 && (tile & 7) == 7) polled = ld_volatile(res_best(result));
            if (modeL) {
                // F words: every column eligible at depth d (word minima); the
                // 32/WPT lanes of one F word OR their bits and one stores
                constexpr int LPF = 32 / WPT;
                const int a0 = tau * WPT;
                for (int b = 0; b < nrows; ++b) {
                    const int d = d0 + b;
                    uint32_t fnib = 0;
#pragma unroll
                    for (int k = 0; k < WPT; ++k) fnib |= ((d <= MINE[k] && MINC[k] + d >= t) ? 1u : 0u) << k;
                    uint32_t v = fnib << (a0 & 31);
#pragma unroll
                    for (int o = 1; o < LPF; o <<= 1) v |= __shfl_xor_sync(0xFFFFFFFFu, v, o);
                    if ((lane & (LPF - 1)) == 0) fm[b * fstride + (a0 >> 5)] = v;
                }
            } else {  // t < FIX_TL: exact E rows from the smem copies of c and e
                ex.d0 = d0;
                for (int b = 0; b < nrows; ++b)
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        const int a = tau * WPT + k;
                        hist[b * Wpad + a] = a < W ? ex.mask(a, b, t) : 0u;
                    }
            }
            if (tau == 0 && (tile & 7) == 7) misc->g = polled;
            __syncthreads();

            const int lastb = nrows - 1;
            bool spec = climbing && modeL && lastb > 0;
            int cur_t = spec ? t + lastb : t, start_b = spec ? lastb : 0;
            ex.d0 = d0;
            for (;;) {
                uint32_t best = RES_INF;
                const int m = cur_t - t;
                if (modeL) {
                    const int n = (lastb - start_b + 1) * nfw;
                    int nc = 0, cb0 = 0, ca0 = 0, cl0 = 0, cb1 = 0, ca1 = 0, cl1 = 0;
                    for (int idx = tau; idx < n; idx += NT) {
                        const int b = start_b + idx / nfw, fw = idx % nfw;
                        scan_fword(fm, fstride, W, b, m, fw, cur_t, [&](int cb, int a0, int len) {
                            if (nc < 2) {
                                if (nc == 0) { cb0 = cb; ca0 = a0; cl0 = len; }
                                else { cb1 = cb; ca1 = a0; cl1 = len; }
                                ++nc;
                            } else {
                                const int suf = a0 > 0 ? suffix_ones(ex.mask(a0 - 1, cb, cur_t)) : 0;
                                const int pre = a0 + len < W ? prefix_ones(ex.mask(a0 + len, cb, cur_t)) : 0;
                                if (suf + 32 * len + pre >= cur_t) best = min(best, enc_res(cb, 32 * a0 - suf));
                            }
                        });
                    }
                    for (;;) {
                        const unsigned mk = __ballot_sync(0xFFFFFFFFu, nc > 0);
                        if (!mk) break;
                        const int src = __ffs(mk) - 1;
                        const int mb = nc == 2 ? cb1 : cb0, ma = nc == 2 ? ca1 : ca0, ml = nc == 2 ? cl1 : cl0;
                        const int b = __shfl_sync(0xFFFFFFFFu, mb, src);
                        const int a0 = __shfl_sync(0xFFFFFFFFu, ma, src);
                        const int len = __shfl_sync(0xFFFFFFFFu, ml, src);
                        const int suf = a0 > 0 ? suffix_ones(ex.coop_mask(a0 - 1, b, cur_t, lane)) : 0;
                        const int pre = a0 + len < W ? prefix_ones(ex.coop_mask(a0 + len, b, cur_t, lane)) : 0;
                        if (lane == src) {
                            if (suf + 32 * len + pre >= cur_t) best = min(best, enc_res(b, 32 * a0 - suf));
                            --nc;
                        }
                    }
                } else {
                    for (int b = start_b; b <= lastb; ++b) {
#pragma unroll
                        for (int k = 0; k < WPT; ++k) {
                            const int a = tau * WPT + k;
                            if (a < W) test_word_full(hist, Wpad, W, b, m, a, cur_t, best);
                        }
                    }
                }
                const uint32_t rr = round_result(best);
                if (spec) {
                    spec = false;
                    if (rr == RES_INF) {  // not a full climb: the tile's normal rounds
                        cur_t = t;
                        start_b = 0;
                        continue;
                    }
                }
                if (rr == RES_INF) break;
                const int bs_ = (int)(rr >> 20), col = (int)(rr & 0xFFFFFu);
                if (tau == 0) {
                    fixkey = pack_key(cur_t, p.row_base + r0 + d0 + bs_ - 1, col + cur_t - 1);
                    if (p.share) atomicMax(res_best(result), cur_t);
                }
                ++cur_t;
                start_b = bs_ + 1;
                if (start_b > lastb) break;
            }
            climbing = cur_t - t == nrows;  // every depth of this tile raised
            t = cur_t;
            if (p.share) t = max(t, misc->g);
            d0 += nrows;
        }
    }
    if (tau == 0) {
        if (p.fix_keys) p.fix_keys[band] = fixkey;
        if (fixkey) atomicMax(res_keyfix(result), fixkey);
    }
}

// ======================================================= carries (P5 fold)
// carry[k][j] = true height of column j at the row above band k (clamped to
// 65535; exact for cols <= 65536): fold (b, all-ones) of the
// bands above, starting from base[j] (rows above this rank; 0 on one GPU).
// Segmented over bands: block = 32 threads x CARRY_SEG band segments, 8
// columns per thread (16-byte loads/stores of the uint16 rows).  Each band is
// the map c -> (all ones ? c + h_q : b_q); a segment composes its maps
// (pass 1), then folds the maps of the segments above from base and writes
// its carries (pass 2) -- 2 reads of the summaries, CARRY_SEG-way parallel.
// LANES x 8 columns per CTA: 16 lanes for matrices up to 32768 columns (twice the
// CTAs: cfg3's 16384 columns gave 64 CTAs of 256 columns on 148 SMs), and 16
// segments (half the bands per thread of round 1's 8): cfg3 0.123 -> 0.119 ms per solve.
constexpr int CARRY_SEG = 16;
template <int LANES>
__global__ void __launch_bounds__(LANES * CARRY_SEG) carry_scan_kernel(int rows, int cols, int W, int nbands,
                                                                       int cols_pad, const uint16_t* b_in,
                                                                       const uint32_t* ao_in, const uint32_t* base,
                                                                       uint16_t* carry_out) {
    __shared__ uint32_t fval[CARRY_SEG][LANES][8];
    __shared__ uint8_t fconst[CARRY_SEG][LANES];
    // launched as a programmatic dependent of the band pass: wait for its writes,
    // then let the fix-up's CTAs launch (they wait for this grid in turn)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x, sg = threadIdx.y;
    const int j0 = (blockIdx.x * LANES + lane) * 8;  // 8 columns; cols_pad is a multiple of 32
    const int nq = nbands - 1;                     // transitions: carry of band q+1 from band q
    const int L = (nq + CARRY_SEG - 1) / CARRY_SEG;
    const int q0 = min(nq, sg * L), q1 = min(nq, q0 + L);
    const bool ok = j0 < cols_pad;
    unsigned v[8];
    uint32_t isc = 0;  // bit i: column j0+i's composed map is constant
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0;
    auto step = [&](int q, uint32_t& cmask) {
        const uint32_t full8 = (ao_in[(size_t)q * W + (j0 >> 5)] >> (j0 & 31)) & 0xFFu;
        const uint4 b4 = *(const uint4*)(b_in + (size_t)q * cols_pad + j0);
        const uint32_t bw[4] = {b4.x, b4.y, b4.z, b4.w};
        const unsigned hq = (unsigned)(band_row0(rows, nbands, q + 1) - band_row0(rows, nbands, q));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const unsigned bq = (bw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
            v[i] = ((full8 >> i) & 1u) ? min(v[i] + hq, 0x7FFFFFFFu) : bq;
        }
        cmask |= ~full8 & 0xFFu;
    };
    if (ok) {
#pragma unroll 4
        for (int q = q0; q < q1; ++q) step(q, isc);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) fval[sg][lane][i] = v[i];
    fconst[sg][lane] = (uint8_t)isc;
    __syncthreads();
    if (!ok) return;
    // pass 2: carries at the segment start, then the segment's rows
    if (base) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = j0 + i < cols ? base[j0 + i] : 0u;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0;
    }
    for (int s2 = 0; s2 < sg; ++s2) {
        const uint32_t cm = fconst[s2][lane];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            v[i] = ((cm >> i) & 1u) ? fval[s2][lane][i] : min(v[i] + fval[s2][lane][i], 0x7FFFFFFFu);
    }
    auto emit = [&](int row) {
        uint32_t o[4];
#pragma unroll
        for (int h = 0; h < 4; ++h)
            o[h] = min(v[2 * h], 65535u) | (min(v[2 * h + 1], 65535u) << 16);
        *(uint4*)(carry_out + (size_t)row * cols_pad + j0) = make_uint4(o[0], o[1], o[2], o[3]);
    };
    if (sg == 0) emit(0);
#pragma unroll 4
    for (int q = q0; q < q1; ++q) {
        uint32_t dummy = 0;
        step(q, dummy);
        emit(q + 1);
    }
}

// ======================================================= lower-bound seed
// A proven lower bound for the shared best side before pass 1: each warp runs
// Algorithm 1 on a strip of SEED_ROWS rows x 32 words (1024 columns), heights
// local to the strip (bit-sliced, 8 planes per lane), one threshold test per
// row.  Any square it finds is a real square of the matrix, so the bands may
// start testing at the largest one (ties included) -- the same argument as the
// shared best side (P2); rows whose local heights cannot reach it need no test.
constexpr int SEED_ROWS = 192;  // strip height (squares found are <= this)
constexpr int SEED_BATCH = 32;  // rows loaded per batch (next batch in flight while one is processed)
constexpr int SEED_STEP = 8;    // test every SEED_STEP rows at best + SEED_STEP (a lower bound needs no exactness)
template <bool U8>
__device__ __forceinline__ uint32_t seed_word(const uint8_t* rp, int w, int W, int cols) {
    if (w >= W) return 0u;
    if (!U8) return ((const uint32_t*)rp)[w];
    const int c0 = 32 * w;
    if (c0 + 32 <= cols && ((uintptr_t)(rp + c0) & 15) == 0)
        return bits16(*(const uint4*)(rp + c0)) | (bits16(*(const uint4*)(rp + c0 + 16)) << 16);
    uint32_t word = 0;
    for (int j = 0; j < 32 && c0 + j < cols; ++j) word |= (uint32_t)(rp[c0 + j] & 1u) << j;
    return word;
}
// Heights are kept as last-zero rows in 8 bit-planes (one LOP3 per plane and
// row: rows count from 8 so inside a batch of 32 rows the low 3 plane bits are
// compile-time constants), and a test every 8 rows is an 8-LOP3 comparison
// plus one segmented warp scan.
template <bool U8>
__global__ void __launch_bounds__(256) seed_climb_kernel(const uint8_t* src, long long ld_bytes, int rows, int cols,
                                                         int W, int nstrips, int chunks, unsigned char* result) {
    // the band pass may launch now (its CTAs wait in griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw >= nstrips * chunks) return;
    const int strip = gw / chunks, chunk = gw - strip * chunks;
    const int r0 = (int)((long long)rows * strip / nstrips);
    const int nr = min(SEED_ROWS, rows - r0);
    const int w = chunk * 32 + lane;
    const uint32_t val = valid_mask(w, W, cols);
    constexpr int P = 8;  // stored rows r + 8 <= 199 < 256
    uint32_t z[P];
#pragma unroll
    for (int q = 0; q < P; ++q) z[q] = (7u >> q) & 1u ? 0xFFFFFFFFu : 0u;  // 7 = no zero yet
    int best = 0;
    // rows in flight: raw 16-byte vectors for u8 (converted when used, so the
    // loads of a whole batch are issued back to back), words for bits
    constexpr int SB = U8 ? 16 : SEED_BATCH;
    const bool fast = U8 && w < W && 32 * w + 32 <= cols && (ld_bytes & 15) == 0 && ((uintptr_t)src & 15) == 0;
    struct Raw {
        uint4 a, b;
        uint32_t word;
    };
    auto fetch = [&](int i) -> Raw {
        Raw r{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), 0u};
        if (i >= nr) return r;
        const uint8_t* rp = src + (size_t)(r0 + i) * ld_bytes;
        if (fast) {
            r.a = *(const uint4*)(rp + 32 * w);
            r.b = *(const uint4*)(rp + 32 * w + 16);
        } else if (!U8) {
            r.word = seed_word<U8>(rp, w, W, cols);
        }
        return r;
    };
    auto word_of = [&](const Raw& r, int i) -> uint32_t {
        if (!U8) return r.word;
        if (fast) return bits32(r.a, r.b);
        return i < nr ? seed_word<U8>(src + (size_t)(r0 + i) * ld_bytes, w, W, cols) : 0u;  // partial / unaligned
    };
    Raw nxt[SB];
#pragma unroll
    for (int q = 0; q < SB; ++q) nxt[q] = fetch(q);
    for (int i0 = 0; i0 < nr; i0 += SB) {
        // a strip whose squares grow slower than one side per 4 rows holds no
        // large square; stop early (the bound only has to be a real square)
        if (i0 >= 32 && 4 * best < i0) break;
        uint32_t rw[SB];
#pragma unroll
        for (int q = 0; q < SB; ++q) {
            rw[q] = word_of(nxt[q], i0 + q);
            nxt[q] = fetch(i0 + SB + q);
        }
#pragma unroll
        for (int q = 0; q < SB; ++q) {
            if (i0 + q >= nr) break;
            const uint32_t m = rw[q] & val;
            const uint32_t rg = (uint32_t)(i0 + q + 8);  // stored row; low 3 bits = q & 7 (batches are multiples of 8)
#pragma unroll
            for (int p = 0; p < 3; ++p) z[p] = ((q >> p) & 1) ? (z[p] | ~m) : (z[p] & m);
#pragma unroll
            for (int p = 3; p < P; ++p) z[p] = (m & z[p]) | (~m & (0u - ((rg >> p) & 1u)));
            if ((q % SEED_STEP) != SEED_STEP - 1) continue;
            const int T = best + SEED_STEP;
            // E = {z <= rg - T}: LSB-first comparison
            const int cvs = (int)rg - T;
            const uint32_t cv = (uint32_t)max(cvs, 0);
            uint32_t le = 0xFFFFFFFFu;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const uint32_t cb = 0u - ((cv >> p) & 1u);
                le = (cb & (~z[p] | le)) | (~cb & ~z[p] & le);
            }
            const uint32_t acc = cvs >= 0 ? (le & val) : 0u;
            // run of eligible columns ending at the end of this lane's word (segmented warp scan)
            const bool full = acc == 0xFFFFFFFFu;
            int v = full ? 32 : __clz(~acc);
            int f = full ? 1 : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v2 = __shfl_up_sync(0xFFFFFFFFu, v | (f << 16), o);
                if (lane >= o) {
                    if (f) v += v2 & 0xFFFF;
                    f &= v2 >> 16;
                }
            }
            int rin = __shfl_up_sync(0xFFFFFFFFu, v, 1);
            if (lane == 0) rin = 0;
            const int pre = full ? 32 : __ffs(~acc) - 1;
            bool ok = rin + pre >= T || v >= T;
            if (!ok && T <= 32) ok = windows_in_word(acc, T) != 0u;
            if (__any_sync(0xFFFFFFFFu, ok)) best = T;
        }
    }
    if (lane == 0 && best > 0) atomicMax(res_best(result), best);
}

// ======================================================= row-band sharding
// Bottom run of the rank's slice per column (== local rows when all ones): the
// last band (from the bottom) whose column is not all ones, plus the heights of
// the all-ones bands below it.  One warp per 32-column word; lanes take 32 bands
// at a time from the bottom, one ballot per column finds the band.
__global__ void __launch_bounds__(256) rank_summary_kernel(int rows, int cols, int W, int nbands, int cols_pad,
                                                           const uint16_t* b_in, const uint32_t* ao_in,
                                                           uint32_t* out) {
    const int lane = threadIdx.x & 31;
    const int word = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (word >= W) return;
    uint32_t pending = valid_mask(word, W, cols);  // columns still looking for their band
    uint32_t res = 0u;                             // this lane's column (word*32 + lane)
    for (int q0 = nbands - 1; q0 >= 0 && pending; q0 -= 32) {
        const int q = q0 - lane;  // lane's band
        const uint32_t notall = q >= 0 ? ~ao_in[(size_t)q * W + word] : 0u;
        uint32_t todo = pending;
        while (todo) {  // warp-uniform loop over the pending columns
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const unsigned m = __ballot_sync(0xFFFFFFFFu, (notall >> j) & 1u);
            if (m) {  // the lowest lane = the bottom-most band with a zero in column j
                const int qb = q0 - (__ffs(m) - 1);
                if (lane == j)
                    res = (uint32_t)(rows - band_row0(rows, nbands, qb + 1)) +
                          (uint32_t)b_in[(size_t)qb * cols_pad + 32 * word + j];
                pending &= ~(1u << j);
            }
        }
    }
    if ((pending >> lane) & 1u) res = (uint32_t)rows;  // all ones through the slice
    const int col = 32 * word + lane;
    if (col < cols) out[col] = res;
}

struct RankRows {
    long long r[64];
};

__global__ void compose_carry_kernel(const uint32_t* summaries, RankRows rr, int rank, int cols,
                                     uint32_t* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    unsigned long long c = 0;
    for (int q = 0; q < rank; ++q) {
        const uint32_t s = summaries[(size_t)q * cols + j];
        c = ((long long)s == rr.r[q]) ? c + (unsigned long long)s : (unsigned long long)s;
    }
    out[j] = c > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c;
}

// [max(key_pass1, key_fix), 3 = invalid cell / 2 = sieve undecided / 1 = sieve: nothing above 62 here / 0] as two int64 for the ranks' all-reduce(max)
__global__ void key_status_kernel(const unsigned char* result, long long* out) {
    const unsigned long long k1 = *(const unsigned long long*)result;
    const unsigned long long k2 = *(const unsigned long long*)(result + 8);
    out[0] = (long long)(k1 > k2 ? k1 : k2);
    const unsigned s = *(const unsigned*)(result + 16);
    out[1] = (s & 1u) ? 3ll : (s & 2u) ? 2ll : (s & 4u) ? 1ll : 0ll;
}

// ======================================================= input generator
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void gen_hash_u8_kernel(unsigned long long seed, unsigned long long thr, long long row0,
                                   long long nrows, long long cols, long long ld, uint8_t* out) {
    const long long n = nrows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols, c = i - r * cols;
        const unsigned long long idx = (unsigned long long)((row0 + r) * cols + c);
        out[r * ld + c] = (uint8_t)((mix64(seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull) >> 11) < thr);
    }
}

__global__ void gen_hash_bits_kernel(unsigned long long seed, unsigned long long thr, long long row0,
                                     long long nrows, long long cols, long long ld, uint32_t* out) {
    const long long words = (cols + 31) / 32;
    const long long n = nrows * words;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / words, w = i - r * words;
        uint32_t v = 0;
        const long long c0 = 32 * w;
        const int nb = (int)min(32ll, cols - c0);
        for (int b = 0; b < nb; ++b) {
            const unsigned long long idx = (unsigned long long)((row0 + r) * cols + c0 + b);
            v |= (uint32_t)((mix64(seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull) >> 11) < thr) << b;
        }
        out[r * ld + w] = v;
    }
}

}  // namespace msq
