// msq_engine.cuh -- sm_100a kernels for the maximal-square hot path.
//
// Reference semantics: /root/reference/pkg/src/squarelab/squares.py:68-114
// (Algorithm 1 / _freq_core): per row, column one-run heights ("freq") are
// updated and ONE threshold test is made: do t consecutive columns have
// height >= t, t = best side so far + 1.  On success the side grows by one and
// the location is the cell where the t-run closes (squares.py:93-97).
//
// B200 design (DESIGN.md has the full argument):
//  * A matrix is cut into row bands, one CTA per band (<= one per SM).  Each
//    CTA streams its rows through a TMA bulk-copy ring in shared memory and
//    keeps, per 32-column word, the eligibility mask E = {j : h_j >= t} as a
//    bit-set in registers.  Heights are never stored: smem holds u_j, the row
//    of column j's last zero, and a column becomes eligible exactly when
//    rho - u_j >= t.  Per word we keep TRIG = min u over ineligible columns,
//    so a word is only revisited when a column can actually become eligible
//    (event-driven: ~3% of word-rows at p = 0.999).
//  * The threshold test runs on bit-sets with clz/ffs word walks; after the
//    first row only words that gained eligible bits can create a new run, so
//    the test is incremental.  B rows are tested per barrier ("tile"); a raise
//    inside a tile re-tests later rows at t+1 with E_b(t+1) = E_b(t) & E_{b-1}(t)
//    from the tile's E history.
//  * Bands run standalone (local heights); squares crossing a band's top are
//    recovered by a data-free fix-up on virtual heights c_j + d for columns
//    whose leading run from the band top is >= d.  The fix-up
//    reads no matrix data: only per-band (bottom run, leading depth, all-ones)
//    column summaries written by pass 1.
//  * Result: one 64-bit key per unit, (side, -bottom, -right), max-reduced.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace msq {

constexpr int KEY_DIM_BITS = 21;
constexpr unsigned long long KEY_DIM_MASK = (1ull << KEY_DIM_BITS) - 1ull;
constexpr int TRIG_INF = 1 << 29;
constexpr uint32_t RES_INF = 0xFFFFFFFFu;
constexpr int OFF_FIX = 65535;  // fix-up height offset: h = d + OFF - u, u = OFF - min(c, OFF)

__host__ __device__ __forceinline__ unsigned long long pack_key(long long side, long long bottom,
                                                                long long right) {
    if (side <= 0) return 0ull;
    return ((unsigned long long)side << (2 * KEY_DIM_BITS)) |
           ((KEY_DIM_MASK - (unsigned long long)bottom) << KEY_DIM_BITS) |
           (KEY_DIM_MASK - (unsigned long long)right);
}

__host__ __device__ __forceinline__ int band_row0(int rows, int nbands, int band) {
    return (int)(((long long)rows * band) / nbands);
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
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
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
__device__ __forceinline__ int ld_volatile(const int* p) { return *(const volatile int*)p; }

// 4 bytes in {0,1} -> 4 bits (byte i -> bit i).  Terms of the product land on
// distinct bit positions, so no carries ("u8 ingest").
__device__ __forceinline__ uint32_t nib4(uint32_t x) { return ((x * 0x01020408u) >> 24) & 0xFu; }
__device__ __forceinline__ uint32_t bits16(uint4 v) {
    return nib4(v.x) | (nib4(v.y) << 4) | (nib4(v.z) << 8) | (nib4(v.w) << 12);
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

// eligibility of word x at tile row b at threshold t + m (P7 AND-history)
__device__ __forceinline__ uint32_t e_at(const uint32_t* hist, int Wpad, int b, int m, int x) {
    uint32_t v = hist[b * Wpad + x];
    for (int q = 1; q <= m; ++q) v &= hist[(b - q) * Wpad + x];
    return v;
}

// length of the run continuing rightwards from word y (full words then a prefix)
__device__ __forceinline__ int run_right(const uint32_t* hist, int Wpad, int W, int b, int m, int y,
                                         int L, int t) {
    while (L < t && y < W) {
        uint32_t nx = e_at(hist, Wpad, b, m, y);
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

// FULL test: every run that STARTS in word a (each maximal run is walked once)
__device__ __forceinline__ void test_word_full(const uint32_t* hist, int Wpad, int W, int b, int m,
                                               int a, int t, uint32_t& best) {
    uint32_t x = e_at(hist, Wpad, b, m, a);
    if (x == 0) return;
    if (t <= 32) {
        uint32_t y = windows_in_word(x, t);
        if (y) best = min(best, enc_res(b, 32 * a + __ffs(y) - 1));
    }
    int s = __clz(~x);  // suffix run (from bit 31 down); 32 if full
    if (s == 0) return;
    if (s == 32 && a > 0 && (e_at(hist, Wpad, b, m, a - 1) >> 31)) return;  // continuation
    int L = run_right(hist, Wpad, W, b, m, a + 1, s, t);
    if (L >= t) best = min(best, enc_res(b, 32 * a + 32 - s));
}

// INCREMENTAL test: every run intersecting word a (a gained eligible bits)
__device__ __forceinline__ void test_word_incr(const uint32_t* hist, int Wpad, int W, int b, int m,
                                               int a, int t, uint32_t& best) {
    uint32_t x = e_at(hist, Wpad, b, m, a);
    if (x == 0) return;
    if (t <= 32) {
        uint32_t y = windows_in_word(x, t);
        if (y) best = min(best, enc_res(b, 32 * a + __ffs(y) - 1));
    }
    if (x & 1u) {  // run through bit 0: find its start on the left
        int start = 32 * a;
        for (int y = a - 1; y >= 0; --y) {
            uint32_t px = e_at(hist, Wpad, b, m, y);
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
        int s = __clz(~x);
        if (s > 0) {
            int L = run_right(hist, Wpad, W, b, m, a + 1, s, t);
            if (L >= t) best = min(best, enc_res(b, 32 * a + 32 - s));
        }
    }
}

// ------------------------------------------------------------------ params
struct Pass1Params {
    const uint8_t* src;         // matrix base (bytes)
    long long ld_bytes;         // row stride in bytes
    long long batch_stride;     // bytes between stacked matrices
    int rows, cols, W, nbands;  // per matrix
    int cols_pad;               // W * 32
    long long row_base;         // global row of row 0 (row-band sharding)
    int nstage;                 // TMA ring depth (tiles); 0 = direct loads
    int rs;                     // row stage bytes (16-B multiple)
    int row_bytes;              // bytes copied per row
    int share;                  // cross-band threshold sharing
    int write_summaries;        // e/b/allones outputs
    uint16_t* e_out;
    uint16_t* b_out;
    uint32_t* ao_out;
    unsigned long long* band_keys;  // [batch][nbands]
    unsigned char* results;         // msq_devresult blocks (32 B each)
};

struct FixParams {
    int rows, cols, W, nbands, cols_pad;
    long long row_base;
    int band_begin;             // first band fixed by this launch
    const uint16_t* e_in;
    const uint16_t* b_in;
    const uint32_t* ao_in;
    const uint32_t* base_carry;  // carry into band 0 (row-band sharding) or null
    int share;
    unsigned long long* fix_keys;  // [nbands]
    unsigned char* results;
};

// msq_devresult field access (layout fixed in msq.h)
__device__ __forceinline__ unsigned long long* res_key1(unsigned char* r) {
    return (unsigned long long*)(r + 0);
}
__device__ __forceinline__ unsigned long long* res_keyfix(unsigned char* r) {
    return (unsigned long long*)(r + 8);
}
__device__ __forceinline__ unsigned int* res_status(unsigned char* r) { return (unsigned int*)(r + 16); }
__device__ __forceinline__ int* res_best(unsigned char* r) { return (int*)(r + 20); }

struct Misc {
    uint32_t res[3];
    int g;      // polled shared best side
    int flag;
    int pad[3];
};

// ============================================================= pass 1 kernel
// One CTA = one band of one matrix.  Thread tau owns words [tau*WPT, tau*WPT+WPT).
template <int WPT, int B, bool U8, bool TMA>
__global__ void __launch_bounds__(512, 1) pass1_kernel(const Pass1Params p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int NT = blockDim.x;
    const int tau = threadIdx.x;
    const int band = (int)(blockIdx.x % (unsigned)p.nbands);
    const int mat = (int)(blockIdx.x / (unsigned)p.nbands);
    const int W = p.W;
    const int Wpad = NT * WPT;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    unsigned char* result = p.results + (size_t)mat * 32;

    // ---- shared memory carve-up (must match host plan)
    size_t off = 0;
    uint8_t* ring = smem + off;
    if (TMA) off += (size_t)p.nstage * B * p.rs;
    uint64_t* bars = (uint64_t*)(smem + off);
    if (TMA) off += ((size_t)p.nstage * 8 + 15) / 16 * 16;
    uint16_t* zs = (uint16_t*)(smem + off);
    off += (size_t)Wpad * 32 * 2;
    uint32_t* hist = (uint32_t*)(smem + off);
    off += (size_t)B * Wpad * 4;
    Misc* misc = (Misc*)(smem + off);

    const uint8_t* mbase = p.src + (size_t)mat * p.batch_stride;
    const size_t sum_base = (size_t)band * p.cols_pad;

    // ---- per-thread word state
    uint32_t E[WPT], NZ[WPT], VAL[WPT];
    int ZA[WPT], TRIG[WPT];
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
        const int a = tau * WPT + k;
        uint32_t v = 0;
        if (a < W) {
            const int rem = p.cols - 32 * a;
            v = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
        }
        VAL[k] = v;
        E[k] = 0;
        NZ[k] = v;
        ZA[k] = 0;
        TRIG[k] = v ? 0 : TRIG_INF;
    }
    for (int i = tau; i < Wpad * 16; i += NT) ((uint32_t*)zs)[i] = 0u;
    if (tau == 0) {
        misc->res[0] = misc->res[1] = misc->res[2] = RES_INF;
        misc->g = p.share ? ld_volatile(res_best(result)) : 0;
        if (TMA) {
            for (int s = 0; s < p.nstage; ++s) mbar_init(&bars[s], 1);
            fence_mbar_init();
        }
    }
    __syncthreads();

    const int ntiles = (H + B - 1) / B;
    if (TMA && tau == 0) {
        for (int tl = 0; tl < p.nstage && tl < ntiles; ++tl) {
            const int nr = min(B, H - tl * B);
            uint8_t* dst = ring + (size_t)(tl % p.nstage) * B * p.rs;
            mbar_expect_tx(&bars[tl % p.nstage], (uint32_t)(nr * p.row_bytes));
            for (int b = 0; b < nr; ++b)
                tma_row(dst + (size_t)b * p.rs, mbase + (size_t)(r0 + tl * B + b) * p.ld_bytes,
                        (uint32_t)p.row_bytes, &bars[tl % p.nstage]);
        }
    }

    int t = max(1, misc->g);
    bool full_next = false;
    unsigned long long bandkey = 0ull;
    int round_ctr = 0;
    uint32_t bad_or = 0;  // u8 validation accumulator

    for (int tile = 0; tile < ntiles; ++tile) {
        const int rho0 = tile * B + 1;
        const uint8_t* stage = nullptr;
        if (TMA) {
            const int s = tile % p.nstage;
            mbar_wait(&bars[s], (uint32_t)((tile / p.nstage) & 1));
            stage = ring + (size_t)s * B * p.rs;
        }
        int polled = 0;
        if (p.share && tau == 0 && (tile & 7) == 7) polled = ld_volatile(res_best(result));

        uint32_t dirty = 0;
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int rho = rho0 + b;
            uint32_t w[WPT];
            if (rho <= H) {
                // ------------------------------------------------ fetch row words
                if (U8) {
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        const int a = tau * WPT + k;
                        uint32_t word = 0;
                        if (a < W) {
                            if (TMA) {
                                const uint8_t* rp = stage + (size_t)b * p.rs + (size_t)a * 32;
                                uint4 v0 = *(const uint4*)rp;
                                uint4 v1 = make_uint4(0, 0, 0, 0);
                                if (a * 32 + 16 < p.rs) v1 = *(const uint4*)(rp + 16);
                                bad_or |= v0.x | v0.y | v0.z | v0.w | v1.x | v1.y | v1.z | v1.w;
                                word = bits16(v0) | (bits16(v1) << 16);
                            } else {
                                const uint8_t* rp = mbase + (size_t)(r0 + rho - 1) * p.ld_bytes;
                                const int c0 = 32 * a;
                                const int n = min(32, p.cols - c0);
                                for (int j = 0; j < n; ++j) {
                                    uint32_t cb = rp[c0 + j];
                                    bad_or |= cb;
                                    word |= (cb & 1u) << j;
                                }
                            }
                        }
                        w[k] = word & VAL[k];
                    }
                } else {
                    if (TMA) {
                        const uint32_t* rp = (const uint32_t*)(stage + (size_t)b * p.rs) + tau * WPT;
                        if (tau * WPT < W) {
                            if (WPT == 4) {
                                uint4 v = *(const uint4*)rp;
                                w[0] = v.x;
                                if (WPT > 1) w[1 % WPT] = v.y;
                                if (WPT > 2) w[2 % WPT] = v.z;
                                if (WPT > 3) w[3 % WPT] = v.w;
                            } else if (WPT == 2) {
                                uint2 v = *(const uint2*)rp;
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
                        const uint32_t* rp =
                            (const uint32_t*)(mbase + (size_t)(r0 + rho - 1) * p.ld_bytes);
#pragma unroll
                        for (int k = 0; k < WPT; ++k) {
                            const int a = tau * WPT + k;
                            w[k] = a < W ? rp[a] : 0u;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < WPT; ++k) w[k] &= VAL[k];
                }
                // ------------------------------------------------ update state
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    const uint32_t zeros = VAL[k] & ~w[k];
                    if (zeros) {
                        if (zeros == VAL[k]) {
                            ZA[k] = rho;  // whole word zero: lazy last-zero row
                        } else {
                            uint32_t zz = zeros;
                            while (zz) {
                                const int bit = __ffs(zz) - 1;
                                zz &= zz - 1;
                                zs[(k * 32 + bit) * NT + tau] = (uint16_t)rho;
                            }
                        }
                        uint32_t newly = NZ[k] & zeros;
                        if (newly && p.write_summaries) {
                            const size_t cb = sum_base + (size_t)(tau * WPT + k) * 32;
                            while (newly) {
                                const int bit = __ffs(newly) - 1;
                                newly &= newly - 1;
                                p.e_out[cb + bit] = (uint16_t)(rho - 1);
                            }
                        }
                        NZ[k] &= ~zeros;
                        E[k] &= ~zeros;
                        TRIG[k] = min(TRIG[k], rho);
                    }
                    if (rho >= TRIG[k] + t) {  // a column may have reached height t
                        uint32_t cand = VAL[k] & ~E[k] & w[k];
                        int nt = zeros ? rho : TRIG_INF;
                        uint32_t added = 0;
                        while (cand) {
                            const int bit = __ffs(cand) - 1;
                            cand &= cand - 1;
                            const int u = max((int)zs[(k * 32 + bit) * NT + tau], ZA[k]);
                            if (u + t <= rho)
                                added |= 1u << bit;
                            else
                                nt = min(nt, u);
                        }
                        E[k] |= added;
                        TRIG[k] = nt;
                        if (added) dirty |= 1u << (b * WPT + k);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < WPT; ++k) w[k] = 0;
            }
            // ------------------------------------------------ E history
            if (WPT == 4) {
                *(uint4*)(hist + b * Wpad + tau * 4) = rho <= H ? make_uint4(E[0], E[1 % WPT], E[2 % WPT], E[3 % WPT])
                                                                : make_uint4(0, 0, 0, 0);
            } else if (WPT == 2) {
                *(uint2*)(hist + b * Wpad + tau * 2) = rho <= H ? make_uint2(E[0], E[1 % WPT]) : make_uint2(0, 0);
            } else {
                hist[b * Wpad + tau] = rho <= H ? E[0] : 0u;
            }
        }
        if (tau == 0 && (tile & 7) == 7) misc->g = polled;
        __syncthreads();  // (A) E history complete; stage consumed

        if (TMA && tau == 0) {
            const int tl = tile + p.nstage;
            if (tl < ntiles) {
                const int s = tl % p.nstage;
                const int nr = min(B, H - tl * B);
                uint8_t* dst = ring + (size_t)s * B * p.rs;
                mbar_expect_tx(&bars[s], (uint32_t)(nr * p.row_bytes));
                for (int b = 0; b < nr; ++b)
                    tma_row(dst + (size_t)b * p.rs, mbase + (size_t)(r0 + tl * B + b) * p.ld_bytes,
                            (uint32_t)p.row_bytes, &bars[s]);
            }
        }

        // ---------------------------------------------------- test rounds
        const int lastb = min(B - 1, H - rho0);
        int cur_t = t, start_b = 0, full_from = full_next ? 0 : B, last_raise = -1;
        for (;;) {
            uint32_t best = RES_INF;
            const int m = cur_t - t;
            for (int b = start_b; b <= lastb; ++b) {
                const bool full = b >= full_from;
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    const int a = tau * WPT + k;
                    if (a < W) {
                        if (full)
                            test_word_full(hist, Wpad, W, b, m, a, cur_t, best);
                        else if ((dirty >> (b * WPT + k)) & 1u)
                            test_word_incr(hist, Wpad, W, b, m, a, cur_t, best);
                    }
                }
            }
            const int slot = round_ctr % 3;
            if (best != RES_INF) atomicMin(&misc->res[slot], best);
            if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
            __syncthreads();  // (B)
            const uint32_t r = misc->res[slot];
            ++round_ctr;
            if (r == RES_INF) break;
            const int bs = (int)(r >> 20), col = (int)(r & 0xFFFFFu);
            if (tau == 0) {
                bandkey = pack_key(cur_t, p.row_base + r0 + rho0 + bs - 1, col + cur_t - 1);
                if (p.share) atomicMax(res_best(result), cur_t);
            }
            last_raise = bs;
            ++cur_t;
            start_b = bs + 1;
            full_from = bs + 1;
            if (start_b > lastb) break;
        }
        // ---------------------------------------------------- state correction
        const int nraise = cur_t - t;
        const int meff = nraise - (last_raise == lastb ? 1 : 0);
        const int rho_last = rho0 + lastb;
        if (meff > 0) {
#pragma unroll
            for (int k = 0; k < WPT; ++k) {
                const int a = tau * WPT + k;
                if (a < W) {
                    const uint32_t en = e_at(hist, Wpad, lastb, meff, a);
                    const uint32_t removed = E[k] & ~en;
                    E[k] = en;
                    if (removed) TRIG[k] = min(TRIG[k], rho_last - t - meff + 1);
                }
            }
        }
        full_next = nraise > 0 && last_raise == lastb;
        t = cur_t;
        // ---------------------------------------------------- shared best jump
        if (p.share) {
            const int g = misc->g;
            if (g > t) {
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    uint32_t ee = E[k];
                    while (ee) {
                        const int bit = __ffs(ee) - 1;
                        ee &= ee - 1;
                        const int u = max((int)zs[(k * 32 + bit) * NT + tau], ZA[k]);
                        if (u + g > rho_last) {
                            E[k] &= ~(1u << bit);
                            TRIG[k] = min(TRIG[k], u);
                        }
                    }
                }
                t = g;
            }
        }
    }

    // ---------------------------------------------------------- band outputs
    if (p.write_summaries) {
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            if (a < W) {
                const size_t cb = sum_base + (size_t)a * 32;
                uint32_t nz = NZ[k];
                while (nz) {
                    const int bit = __ffs(nz) - 1;
                    nz &= nz - 1;
                    p.e_out[cb + bit] = (uint16_t)H;
                }
                uint16_t bb[32];
#pragma unroll
                for (int bit = 0; bit < 32; ++bit) {
                    const int u = max((int)zs[(k * 32 + bit) * NT + tau], ZA[k]);
                    bb[bit] = (uint16_t)(H - u);
                }
                uint4* dst = (uint4*)(p.b_out + cb);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 v;
                    v.x = (uint32_t)bb[8 * q + 0] | ((uint32_t)bb[8 * q + 1] << 16);
                    v.y = (uint32_t)bb[8 * q + 2] | ((uint32_t)bb[8 * q + 3] << 16);
                    v.z = (uint32_t)bb[8 * q + 4] | ((uint32_t)bb[8 * q + 5] << 16);
                    v.w = (uint32_t)bb[8 * q + 6] | ((uint32_t)bb[8 * q + 7] << 16);
                    dst[q] = v;
                }
                p.ao_out[(size_t)band * W + a] = NZ[k];
            }
        }
    }
    if (U8 && (bad_or & 0xFEFEFEFEu)) atomicOr(res_status(result), 1u);
    if (tau == 0) {
        if (p.band_keys) p.band_keys[(size_t)mat * p.nbands + band] = bandkey;
        if (bandkey) atomicMax(res_key1(result), bandkey);
    }
}

// ============================================================ fix-up kernel
// Data-free: virtual rows d = 1..min(H, t-1) of band `band`, height of column j
// at depth d is c_j + d while d <= e_j (leading ones of the band top), else 0.
template <int WPT, int B>
__global__ void __launch_bounds__(512, 1) fixup_kernel(const FixParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int NT = blockDim.x;
    const int tau = threadIdx.x;
    const int band = p.band_begin + blockIdx.x;
    const int W = p.W;
    const int Wpad = NT * WPT;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    unsigned char* result = p.results;

    size_t off = 0;
    uint16_t* us = (uint16_t*)(smem + off);
    off += (size_t)Wpad * 32 * 2;
    uint8_t* e8 = smem + off;
    off += (size_t)Wpad * 32;
    uint32_t* hist = (uint32_t*)(smem + off);
    off += (size_t)B * Wpad * 4;
    Misc* misc = (Misc*)(smem + off);

    // starting threshold: best side known after the band passes
    if (tau == 0) {
        misc->res[0] = misc->res[1] = misc->res[2] = RES_INF;
        int g = (int)(*(volatile unsigned long long*)res_key1(result) >> (2 * KEY_DIM_BITS));
        if (p.share) g = max(g, ld_volatile(res_best(result)));
        misc->g = g;
    }

    uint32_t E[WPT], ALIVE[WPT], VAL[WPT];
    int TRIG[WPT], ND[WPT];
    const size_t eb = (size_t)band * p.cols_pad;
#pragma unroll
    for (int k = 0; k < WPT; ++k) {
        const int a = tau * WPT + k;
        uint32_t v = 0;
        if (a < W) {
            const int rem = p.cols - 32 * a;
            v = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
        }
        VAL[k] = v;
        ALIVE[k] = 0;
        ND[k] = TRIG_INF;
        if (!v) continue;
        // ---- carry-in heights by look-back over the bands above (P5)
        uint32_t pending = v;
        long long acc = 0;
        for (int q = band - 1; q >= 0 && pending; --q) {
            const uint32_t m = p.ao_in[(size_t)q * W + a];
            uint32_t res = pending & ~m;
            while (res) {
                const int bit = __ffs(res) - 1;
                res &= res - 1;
                const long long c = acc + p.b_in[(size_t)q * p.cols_pad + 32 * a + bit];
                us[(k * 32 + bit) * NT + tau] = (uint16_t)(OFF_FIX - (int)min(c, (long long)OFF_FIX));
            }
            pending &= m;
            acc += band_row0(p.rows, p.nbands, q + 1) - band_row0(p.rows, p.nbands, q);
        }
        while (pending) {
            const int bit = __ffs(pending) - 1;
            pending &= pending - 1;
            const long long c = acc + (p.base_carry ? (long long)p.base_carry[32 * a + bit] : 0ll);
            us[(k * 32 + bit) * NT + tau] = (uint16_t)(OFF_FIX - (int)min(c, (long long)OFF_FIX));
        }
        // ---- leading-ones depth of the band top
        const uint4* ep = (const uint4*)(p.e_in + eb + (size_t)32 * a);
        uint32_t alive = 0;
        int nd = TRIG_INF;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v4 = ep[q];
            const uint32_t pr[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int bit = 8 * q + 2 * h + s;
                    const int e = (int)((pr[h] >> (16 * s)) & 0xFFFFu);
                    e8[(k * 32 + bit) * NT + tau] = (uint8_t)min(e, 255);
                    if (((v >> bit) & 1u) && e >= 1) {
                        alive |= 1u << bit;
                        nd = min(nd, e + 1);
                    }
                }
            }
        }
        ALIVE[k] = alive;
        ND[k] = nd;
    }
    __syncthreads();
    int t = max(1, misc->g);

    // eligibility of word k at depth d, threshold tt; also returns TRIG
    auto eval_word = [&](int k, int d, int tt, uint32_t& e_out, int& trig_out) {
        uint32_t al = ALIVE[k], e = 0;
        int tr = TRIG_INF;
        while (al) {
            const int bit = __ffs(al) - 1;
            al &= al - 1;
            const int u = us[(k * 32 + bit) * NT + tau];
            if (u + tt <= d + OFF_FIX)
                e |= 1u << bit;
            else
                tr = min(tr, u);
        }
        e_out = e;
        trig_out = tr;
    };
    auto store_hist0 = [&](const uint32_t* ev) {
#pragma unroll
        for (int k = 0; k < WPT; ++k) hist[tau * WPT + k] = ev[k];
    };
    int round_ctr = 0;
    // full test of tile row 0 at threshold tt; returns packed result or RES_INF
    auto full_test_row0 = [&](int tt) -> uint32_t {
        uint32_t best = RES_INF;
#pragma unroll
        for (int k = 0; k < WPT; ++k) {
            const int a = tau * WPT + k;
            if (a < W) test_word_full(hist, Wpad, W, 0, 0, a, tt, best);
        }
        const int slot = round_ctr % 3;
        if (best != RES_INF) atomicMin(&misc->res[slot], best);
        if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
        __syncthreads();
        const uint32_t r = misc->res[slot];
        ++round_ctr;
        return r;
    };

    unsigned long long fixkey = 0ull;
    if (H >= 1) {
        // ---------------------------------------------- depth 1, exact seeding
#pragma unroll
        for (int k = 0; k < WPT; ++k) eval_word(k, 1, t, E[k], TRIG[k]);
        store_hist0(E);
        __syncthreads();
        uint32_t r = full_test_row0(t);
        if (r != RES_INF) {
            // P3: the window test is monotone in k -> exponential + binary search
            int lo = t, hi = -1;
            uint32_t rlo = r;
            int step = 1;
            while (hi < 0) {
                const int kk = lo + step;
                if (kk > p.cols) {
                    hi = kk;
                    break;
                }
                uint32_t ev[WPT];
                int dummy;
#pragma unroll
                for (int k = 0; k < WPT; ++k) eval_word(k, 1, kk, ev[k], dummy);
                __syncthreads();
                store_hist0(ev);
                __syncthreads();
                const uint32_t rk = full_test_row0(kk);
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
                uint32_t ev[WPT];
                int dummy;
#pragma unroll
                for (int k = 0; k < WPT; ++k) eval_word(k, 1, mid, ev[k], dummy);
                __syncthreads();
                store_hist0(ev);
                __syncthreads();
                const uint32_t rk = full_test_row0(mid);
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
#pragma unroll
            for (int k = 0; k < WPT; ++k) eval_word(k, 1, t, E[k], TRIG[k]);
        }
        __syncthreads();

        // ---------------------------------------------- depths 2.. (tiles of B)
        bool full_next = false;
        int tile = 0;
        for (int d0 = 2; d0 <= H && d0 < t; d0 += B, ++tile) {
            int polled = 0;
            if (p.share && tau == 0 && (tile & 7) == 7) polled = ld_volatile(res_best(result));
            uint32_t dirty = 0;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const int d = d0 + b;
                if (d <= H) {
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        if (d >= ND[k]) {  // deaths: leading run of the band top ended
                            uint32_t al = ALIVE[k];
                            int nd = TRIG_INF;
                            while (al) {
                                const int bit = __ffs(al) - 1;
                                al &= al - 1;
                                int e = e8[(k * 32 + bit) * NT + tau];
                                if (e == 255 && d >= 256)
                                    e = p.e_in[eb + (size_t)32 * (tau * WPT + k) + bit];
                                if (e < d) {
                                    ALIVE[k] &= ~(1u << bit);
                                } else {
                                    nd = min(nd, e == 255 && d < 256 ? 256 : e + 1);
                                }
                            }
                            ND[k] = nd;
                            E[k] &= ALIVE[k];
                        }
                        if (d + OFF_FIX >= TRIG[k] + t) {  // entries: c_j + d reached t
                            uint32_t cand = ALIVE[k] & ~E[k];
                            int nt = TRIG_INF;
                            uint32_t added = 0;
                            while (cand) {
                                const int bit = __ffs(cand) - 1;
                                cand &= cand - 1;
                                const int u = us[(k * 32 + bit) * NT + tau];
                                if (u + t <= d + OFF_FIX)
                                    added |= 1u << bit;
                                else
                                    nt = min(nt, u);
                            }
                            E[k] |= added;
                            TRIG[k] = nt;
                            if (added) dirty |= 1u << (b * WPT + k);
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < WPT; ++k) hist[b * Wpad + tau * WPT + k] = d <= H ? E[k] : 0u;
            }
            if (tau == 0 && (tile & 7) == 7) misc->g = polled;
            __syncthreads();

            const int lastb = min(B - 1, H - d0);
            int cur_t = t, start_b = 0, full_from = full_next ? 0 : B, last_raise = -1;
            for (;;) {
                uint32_t best = RES_INF;
                const int m = cur_t - t;
                for (int b = start_b; b <= lastb; ++b) {
                    const bool full = b >= full_from;
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        const int a = tau * WPT + k;
                        if (a < W) {
                            if (full)
                                test_word_full(hist, Wpad, W, b, m, a, cur_t, best);
                            else if ((dirty >> (b * WPT + k)) & 1u)
                                test_word_incr(hist, Wpad, W, b, m, a, cur_t, best);
                        }
                    }
                }
                const int slot = round_ctr % 3;
                if (best != RES_INF) atomicMin(&misc->res[slot], best);
                if (tau == 0) misc->res[(round_ctr + 1) % 3] = RES_INF;
                __syncthreads();
                const uint32_t rr = misc->res[slot];
                ++round_ctr;
                if (rr == RES_INF) break;
                const int bs = (int)(rr >> 20), col = (int)(rr & 0xFFFFFu);
                if (tau == 0) {
                    fixkey = pack_key(cur_t, p.row_base + r0 + d0 + bs - 1, col + cur_t - 1);
                    if (p.share) atomicMax(res_best(result), cur_t);
                }
                last_raise = bs;
                ++cur_t;
                start_b = bs + 1;
                full_from = bs + 1;
                if (start_b > lastb) break;
            }
            const int nraise = cur_t - t;
            const int meff = nraise - (last_raise == lastb ? 1 : 0);
            const int d_last = d0 + lastb;
            if (meff > 0) {
#pragma unroll
                for (int k = 0; k < WPT; ++k) {
                    const int a = tau * WPT + k;
                    if (a < W) {
                        const uint32_t en = e_at(hist, Wpad, lastb, meff, a);
                        const uint32_t removed = E[k] & ~en;
                        E[k] = en;
                        if (removed) TRIG[k] = min(TRIG[k], d_last + OFF_FIX - t - meff + 1);
                    }
                }
            }
            full_next = nraise > 0 && last_raise == lastb;
            t = cur_t;
            if (p.share) {
                const int g = misc->g;
                if (g > t) {
#pragma unroll
                    for (int k = 0; k < WPT; ++k) {
                        uint32_t ee = E[k];
                        while (ee) {
                            const int bit = __ffs(ee) - 1;
                            ee &= ee - 1;
                            const int u = us[(k * 32 + bit) * NT + tau];
                            if (u + g > d_last + OFF_FIX) {
                                E[k] &= ~(1u << bit);
                                TRIG[k] = min(TRIG[k], u);
                            }
                        }
                    }
                    t = g;
                }
            }
        }
    }
    if (tau == 0) {
        if (p.fix_keys) p.fix_keys[band] = fixkey;
        if (fixkey) atomicMax(res_keyfix(result), fixkey);
    }
}

// ======================================================= row-band sharding
// per column: bottom run of the whole local slice (P5 fold of all bands)
__global__ void rank_summary_kernel(int rows, int cols, int W, int nbands, int cols_pad,
                                    const uint16_t* b_in, const uint32_t* ao_in, uint32_t* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    long long acc = 0;
    uint32_t s = 0;
    bool done = false;
    for (int q = nbands - 1; q >= 0; --q) {
        const bool full = (ao_in[(size_t)q * W + (j >> 5)] >> (j & 31)) & 1u;
        if (!full) {
            s = (uint32_t)(acc + b_in[(size_t)q * cols_pad + j]);
            done = true;
            break;
        }
        acc += band_row0(rows, nbands, q + 1) - band_row0(rows, nbands, q);
    }
    out[j] = done ? s : (uint32_t)acc;  // == rows: all ones
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
