// msq_sieve.cuh -- sieve engine for bit-packed matrices whose answer is a
// moderate square in a sea of sparse zeros (cfg4: 65536^2, Bernoulli 0.999).
//
// The band engines keep an exact per-column state for every row they stream
// (last-zero rows, first zeros, band summaries for the carry scan and the
// fix-up).  For sparse zeros that bookkeeping, not the 0.125 B/cell of input,
// is what bounds them.  The sieve streams the matrix once with no per-column
// state at all and runs the reference's Algorithm 1 (squares.py:84-103: column
// heights + one threshold test per row) on a coarse grid of 8x8-cell blocks
// instead:
//
//   G(R, C) = 1 iff the 8x8 block of cells (rows 8R.., columns 8C..) is all ones.
//
// A square of side s whose bottom-right cell is (i, j) contains every aligned
// block between its corners: at least floor((s-7)/8) block rows and columns,
// ending at the block (floor((i+1)/8)-1, floor((j+1)/8)-1) -- its anchor.  With
// D(R, C) = side of the largest all-ones square of G ending at block (R, C),
//
//   8 * max D  <=  answer  <=  8 * max D + 14,
//
// and every maximal square is anchored at a block with D >= max D - 1.  Its
// bottom-right cell lies 7..14 cells past the anchor's first cell and its side
// is <= 8D + 14, so it lies in the window of 8D + 21 cells that ends 14 cells
// past the anchor's first row and column.  So:
//
//   sieve_pass_kernel   streams the rows (TMA ring, one CTA per row band and
//                       column chunk), ANDs each 8-row tile into G bits, keeps
//                       the block heights of G as 5 saturating bit-planes per
//                       lane (one 32-block word per lane, the warp's lane 0 is
//                       the left halo) and tests one level per block row:
//                       "a run of >= l blocks of height >= l", l = best D - 1.
//                       Hits (rare) get their exact D and go to a candidate list.
//                       The first 31 block rows of a band have no carried-in
//                       heights: their G words are stored instead and
//   sieve_edge_kernel   redoes them from the bottom planes of the band above.
//   sieve_verify_kernel runs Algorithm 1 exactly (per-column heights, one test
//                       per row, leftmost window) on the <= 229 x 229 cell
//                       window of every candidate with D >= max D - 1 and keeps
//                       the best (side, first bottom row, leftmost column) key.
//
// The answer is exact whenever the sieve decides: max D in [7, 26] (answers
// 56..222) and the candidate list did not overflow.  Otherwise status bit 1
// asks the caller to run the band engine (MSQ_EAGAIN); nothing is guessed.
//
// Multi-GPU: a rank prepends the last SV_HALO_ROWS (256 >= 222) rows of the
// rank above (`halo`), so every square the sieve can report lies wholly inside
// the rows of the rank that holds its bottom row: no carry exchange, no fix-up.
#pragma once

namespace msq {

constexpr int SV_PL = 5;           // height planes: block heights saturate at 31
constexpr int SV_EDGE = 31;        // block rows at a band top that need carried-in heights
constexpr int SV_DMAX = 26;        // windows of 8 * 26 + 21 = 229 columns (from column 2 mod 8) fit 8 words
constexpr int SV_LMIN = 6;         // lowest level tested; the sieve decides for max D >= 7
constexpr int SV_CAP = 8192;       // candidate list entries
constexpr int SV_TR = 8;           // rows per tile = block height
constexpr int SV_MAXSLOTS = 16;    // TMA ring depth
constexpr int SV_HALO_ROWS = 256;  // rows a rank borrows from the rank above
constexpr int SV_VROWS = 8 * SV_DMAX + 21;
constexpr int SV_VWARPS = 4;       // verifier warps per CTA (one candidate each)
constexpr int SV_EWARPS = 4;       // edge-kernel warps per CTA

struct SieveCtl {
    int best;   // largest D found so far
    int count;  // candidates appended
    int abort;  // bit 0: D beyond SV_DMAX, bit 1: candidate list overflow
    int pad;
};

struct SieveParams {
    const uint8_t* src;   // local rows
    const uint8_t* halo;  // halo_rows rows above them (multi-GPU) or nullptr
    long long ld_bytes, halo_ld_bytes;
    int halo_rows;        // multiple of 8
    int rows;             // halo_rows + local rows
    int cols, W;
    long long row_base;   // global row index of row 0 of (halo, local rows)
    int CR, CC, CWn, WC;  // block rows, block columns, 32-block words per row, warp columns
    int nbands, nchunks, wmax, nslots, slot_row_bytes;
    uint32_t* gtop;       // [nbands][SV_EDGE][CWn] G words of each band's first block rows
    uint32_t* pbot;       // [nbands][SV_PL][CWn] height planes after each band's last block row
    unsigned long long* cand;  // [SV_CAP] D << 40 | block row << 16 | block column
    SieveCtl* ctl;
    unsigned char* result;
};

__device__ __forceinline__ const uint8_t* sv_row(const SieveParams& p, int r) {
    return r < p.halo_rows ? p.halo + (size_t)r * p.halo_ld_bytes
                           : p.src + (size_t)(r - p.halo_rows) * p.ld_bytes;
}
__device__ __forceinline__ int sv_band_cr0(const SieveParams& p, int band) {
    return (int)(((long long)p.CR * band) / p.nbands);
}

// bit c of the result: bits [c - m + 1, c] of the 64-bit (hi:lo) are all set (1 <= m <= 31)
__device__ __forceinline__ uint32_t sv_runs(uint32_t lo, uint32_t hi, int m) {
    int have = 1;
    while (2 * have <= m) {
        hi &= __funnelshift_l(lo, hi, have);
        lo &= lo << have;
        have *= 2;
    }
    if (have < m) hi &= __funnelshift_l(lo, hi, m - have);
    return hi;
}

// blocks of the lane's word where a run of m blocks of height >= m ends
__device__ __forceinline__ uint32_t sv_hits(const uint32_t (&h)[SV_PL], int m, int lane) {
    const uint32_t E = planes_ge<SV_PL>(h, m);
    uint32_t EL = __shfl_up_sync(0xFFFFFFFFu, E, 1);
    if (lane == 0) EL = 0u;
    return sv_runs(EL, E, m);
}

__device__ __forceinline__ void sv_emit(const SieveParams& p, uint32_t mask, int D, int R, int g) {
    while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const int idx = atomicAdd(&p.ctl->count, 1);
        if (idx < SV_CAP)
            p.cand[idx] = ((unsigned long long)D << 40) | ((unsigned long long)R << 16) |
                          (unsigned long long)(32 * g + j);
        else
            atomicOr(&p.ctl->abort, 2);
    }
}

// Rare path (warp-uniform entry): exact D of the blocks that passed level lvl,
// the shared best, and the candidates with D >= best - 1.
__device__ __noinline__ int sv_rare(const SieveParams& p, uint32_t h0, uint32_t h1, uint32_t h2, uint32_t h3,
                                    uint32_t h4, uint32_t hits, int lvl, bool record, int R, int g, int lane) {
    const uint32_t h[SV_PL] = {h0, h1, h2, h3, h4};
    uint32_t cur = hits, prev = 0u;
    int m = lvl;
    while (m < 31) {
        const uint32_t nxt = sv_hits(h, m + 1, lane) & cur;
        if (!__any_sync(0xFFFFFFFFu, nxt != 0u)) break;
        prev = cur & ~nxt;
        cur = nxt;
        ++m;
    }
    // cur: D == m (>= m at the planes' ceiling), prev: D == m - 1
    int best = 0;
    if (lane == 0) {
        best = atomicMax(&p.ctl->best, m);
        if (m > SV_DMAX) atomicOr(&p.ctl->abort, 1);
    }
    best = max(__shfl_sync(0xFFFFFFFFu, best, 0), m);
    if (record) {
        if (m >= best - 1) sv_emit(p, cur, m, R, g);
        if (m >= best) sv_emit(p, prev, m - 1, R, g);
    }
    return max(lvl, best - 1);
}

// One block row of the coarse Algorithm 1: heights, one test at the level.
__device__ __forceinline__ void sv_step(const SieveParams& p, uint32_t v, uint32_t (&h)[SV_PL], int& lvl,
                                        bool record, int R, int g, bool own, int lane) {
    planes_step<SV_PL>(h, v);
    uint32_t hits = sv_hits(h, lvl, lane);
    if (!own) hits = 0u;
    if (__any_sync(0xFFFFFFFFu, hits != 0u))
        lvl = sv_rare(p, h[0], h[1], h[2], h[3], h[4], hits, lvl, record, R, g, lane);
}

// 4 words -> 16 bits: bit 4k + b = byte b of word k is 0xFF
__device__ __forceinline__ uint32_t sv_flags16(const uint32_t (&a)[4]) {
    uint32_t out = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t y = ((a[k] & 0x7F7F7F7Fu) + 0x01010101u) & a[k] & 0x80808080u;
        out |= (((y >> 7) * 0x01020408u) >> 24) << (4 * k);
    }
    return out;
}

__global__ void __launch_bounds__(320, 1) sieve_pass_kernel(const SieveParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int band = blockIdx.x / p.nchunks, chunk = blockIdx.x - band * p.nchunks;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wc0 = p.WC * chunk / p.nchunks, wc1 = p.WC * (chunk + 1) / p.nchunks;
    const int ncw = wc1 - wc0;  // consumer warps of this chunk
    const int cr0 = sv_band_cr0(p, band);
    const int ntiles = sv_band_cr0(p, band + 1) - cr0;
    const int mw0 = max(0, 8 * (31 * wc0 - 1));  // matrix words [mw0, mw1) of each row
    const int mw1 = min(p.W, 8 * 31 * wc1);
    const uint32_t chunk_bytes = (uint32_t)(mw1 - mw0) * 4u;
    const uint32_t srb = (uint32_t)p.slot_row_bytes;
    const uint32_t slot_bytes = SV_TR * srb;
    uint8_t* ring = smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)p.nslots * slot_bytes);
    uint64_t* empty = full + SV_MAXSLOTS;
    volatile int* stop = (volatile int*)(empty + SV_MAXSLOTS);  // tile at which the producer gave up

    if (tid == 0) {
        for (int s = 0; s < p.nslots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (uint32_t)ncw);
        }
        *stop = -1;
        fence_mbar_init();
    }
    __syncthreads();

    // ------------------------------------------------------------ producer
    if (warp == p.wmax) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            for (int q = 0; q < ntiles; ++q) {
                const int s = q % p.nslots;
                if (q >= p.nslots) mbar_wait(&empty[s], (uint32_t)((q / p.nslots - 1) & 1));
                if ((q & 3) == 3 && ld_volatile(&p.ctl->abort)) {  // the sieve cannot decide: stop streaming
                    *stop = q;
                    mbar_arrive(&full[s]);
                    break;
                }
                mbar_expect_tx(&full[s], SV_TR * chunk_bytes);
                uint8_t* dst = ring + (size_t)s * slot_bytes;
                const int r = SV_TR * (cr0 + q);
#pragma unroll
                for (int b = 0; b < SV_TR; ++b)
                    tma_row(dst + (size_t)b * srb, sv_row(p, r + b) + (size_t)mw0 * 4, chunk_bytes, &full[s], pol);
            }
        }
        return;
    }
    if (warp >= ncw) return;

    // ------------------------------------------------------------ consumers
    const int g = 31 * (wc0 + warp) - 1 + lane;  // the lane's 32-block word (lane 0: left halo)
    const bool in = g >= 0 && g < p.CWn;
    const bool own = lane > 0 && in;
    uint32_t validc = 0u;
    if (in) {
        const int n = p.CC - 32 * g;
        validc = n >= 32 ? 0xFFFFFFFFu : (n > 0 ? (1u << n) - 1u : 0u);
    }
    // the lane's 8 matrix words = two 16-byte halves; lanes 4..7 (mod 8) read the
    // upper half first so a quarter-warp's 8 loads cover all 32 banks
    const int sw = (lane >> 2) & 1;
    const bool okA = in && 8 * g + 4 * sw < mw1;
    const bool okB = in && 8 * g + 4 * (1 - sw) < mw1;
    const uint32_t ring_s = smem_addr(ring);
    const uint32_t offA = okA ? (uint32_t)(8 * g + 4 * sw - mw0) * 4u : 0u;
    const uint32_t offB = okB ? (uint32_t)(8 * g + 4 * (1 - sw) - mw0) * 4u : 0u;
    uint32_t h[SV_PL] = {0u, 0u, 0u, 0u, 0u};
    int lvl = SV_LMIN;
    bool finished = true;

    for (int q = 0; q < ntiles; ++q) {
        const int s = q % p.nslots;
        const uint32_t par = (uint32_t)((q / p.nslots) & 1);
        const int gbest = (q & 3) == 0 ? ld_volatile(&p.ctl->best) : 0;  // used after the tile
        mbar_wait(&full[s], par);
        if (*stop == q) {
            finished = false;
            break;
        }
        const uint32_t slot_s = ring_s + (uint32_t)s * slot_bytes;
        uint32_t A[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
        uint32_t B[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
#pragma unroll
        for (int b = 0; b < SV_TR; ++b) {
            uint32_t wa[4], wb[4];
            lds_words<4>(slot_s + (uint32_t)b * srb + offA, wa);
            lds_words<4>(slot_s + (uint32_t)b * srb + offB, wb);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                A[k] &= wa[k];
                B[k] &= wb[k];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const uint32_t cA = okA ? sv_flags16(A) : 0u, cB = okB ? sv_flags16(B) : 0u;
        const uint32_t v = (sw ? (cB | (cA << 16)) : (cA | (cB << 16))) & validc;
        if (q < SV_EDGE && own) p.gtop[((size_t)band * SV_EDGE + q) * p.CWn + g] = v;
        sv_step(p, v, h, lvl, q >= SV_EDGE, cr0 + q, g, own, lane);
        if ((q & 3) == 0) lvl = max(lvl, gbest - 1);
    }
    if (own && finished) {
#pragma unroll
        for (int k = 0; k < SV_PL; ++k) p.pbot[((size_t)band * SV_PL + k) * p.CWn + g] = h[k];
    }
}

// The first block rows of every band again, now with the heights carried in
// from the band above (band 0: zeros).
__global__ void __launch_bounds__(32 * SV_EWARPS) sieve_edge_kernel(const SieveParams p) {
    __shared__ uint32_t vs[SV_EWARPS][SV_EDGE][32];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int unit = blockIdx.x * SV_EWARPS + warp;
    if (unit >= p.nbands * p.WC) return;
    if (ld_volatile(&p.ctl->abort)) return;
    const int band = unit / p.WC, wc = unit - band * p.WC;
    const int g = 31 * wc - 1 + lane;
    const bool in = g >= 0 && g < p.CWn;
    const bool own = lane > 0 && in;
    const int cr0 = sv_band_cr0(p, band);
    const int n = min(SV_EDGE, sv_band_cr0(p, band + 1) - cr0);
    for (int i = 0; i < n; ++i) vs[warp][i][lane] = in ? p.gtop[((size_t)band * SV_EDGE + i) * p.CWn + g] : 0u;
    uint32_t h[SV_PL];
#pragma unroll
    for (int k = 0; k < SV_PL; ++k)
        h[k] = (band > 0 && in) ? p.pbot[((size_t)(band - 1) * SV_PL + k) * p.CWn + g] : 0u;
    int lvl = max(SV_LMIN, ld_volatile(&p.ctl->best) - 1);
    __syncwarp();
    for (int i = 0; i < n; ++i) sv_step(p, vs[warp][i][lane], h, lvl, true, cr0 + i, g, own, lane);
}

// Algorithm 1 on the cell window of every candidate that can still hold the answer.
__global__ void __launch_bounds__(32 * SV_VWARPS) sieve_verify_kernel(const SieveParams p) {
    __shared__ __align__(16) uint32_t rowsm[SV_VWARPS][SV_VROWS][8];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * SV_VWARPS + warp, nw = gridDim.x * SV_VWARPS;
    const int best = ld_volatile(&p.ctl->best);
    if (ld_volatile(&p.ctl->abort) || best <= SV_LMIN) {  // undecided: the caller runs the band engine
        if (gw == 0 && lane == 0) atomicOr(res_status(p.result), 2u);
        return;
    }
    const int count = min(ld_volatile(&p.ctl->count), SV_CAP);
    const int T0 = 8 * best;
    for (int pass = 0; pass < 2; ++pass) {
        const int Dp = best - pass;
        for (int idx = gw; idx < count; idx += nw) {
            const unsigned long long c = p.cand[idx];
            const int D = (int)(c >> 40);
            if (D != Dp) continue;
            int t = max(T0, ld_volatile(res_best(p.result)));  // ties at the best side so far
            if (8 * D + 14 < t) continue;
            const int Rg = (int)((c >> 16) & 0xFFFFFFull), cg = (int)(c & 0xFFFFull);
            const int r_hi = min(p.rows - 1, 8 * Rg + 14), r_lo = max(0, 8 * (Rg - D) - 6);
            const int c_hi = min(p.cols - 1, 8 * cg + 14), c_lo = max(0, 8 * (cg - D) - 6);
            const int nr = r_hi - r_lo + 1, wa = c_lo >> 5, nwd = (c_hi >> 5) - wa + 1;
            uint32_t msk[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int lo = max(c_lo - 32 * (wa + k), 0), hi = min(c_hi - 32 * (wa + k), 31);
                msk[k] = (k < nwd && hi >= lo) ? ((hi == 31 ? 0xFFFFFFFFu : (1u << (hi + 1)) - 1u) & ~((1u << lo) - 1u))
                                               : 0u;
            }
            __syncwarp();
            // the window's words (lanes spread over rows and words, all loads in flight)
            for (int i = lane; i < nr * 8; i += 32) {
                const int rr = i >> 3, k = i & 7;
                uint32_t w = 0u;
                if (k < nwd) w = __ldg((const uint32_t*)(sv_row(p, r_lo + rr)) + wa + k);
                rowsm[warp][rr][k] = w;
            }
            __syncwarp();
            int lz[8];  // last zero row (window-relative) of column 32k + lane
#pragma unroll
            for (int k = 0; k < 8; ++k) lz[k] = -1;
            unsigned long long key = 0ull;
            int side = 0;
            for (int rr = 0; rr < nr && t <= nr; ++rr) {
                const uint4 a = *(const uint4*)&rowsm[warp][rr][0];
                const uint4 b = *(const uint4*)&rowsm[warp][rr][4];
                const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if ((w[k] & msk[k]) != msk[k] && !((w[k] >> lane) & 1u)) lz[k] = rr;
                if (rr + 1 < t) continue;
                // leftmost window of t columns of height >= t
                int run = 0, e = -1;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t x = __ballot_sync(0xFFFFFFFFu, rr - lz[k] >= t) & msk[k];
                    const int pre = x == 0xFFFFFFFFu ? 32 : __ffs(~x) - 1;
                    if (e < 0 && run + pre >= t) e = 32 * k + (t - run) - 1;
                    run = x == 0xFFFFFFFFu ? run + 32 : __clz(~x);
                }
                if (e >= 0) {
                    key = pack_key(t, p.row_base + r_lo + rr, (long long)32 * wa + e);
                    side = t;
                    ++t;
                }
            }
            if (key && lane == 0) {
                atomicMax(res_key1(p.result), key);
                atomicMax(res_best(p.result), side);
            }
        }
    }
}

}  // namespace msq
