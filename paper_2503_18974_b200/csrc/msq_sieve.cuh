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
//                       column chunk, a warp per 1024 columns), ANDs each
//                       8-row tile into G bits and stores G (1 bit per 64
//                       cells: 8 MB for 65536^2).  Stateless, so any split of
//                       the rows works and the kernel runs at the HBM rate; the
//                       CTAs cover the matrix a quarter at a time.
//   sieve_coarse_kernel (runs beside the streaming pass, one quarter behind it)
//                       Algorithm 1 on G (read from L2): block heights as 5
//                       saturating bit-planes per lane (one 32-block word per
//                       lane, lane 0 of a warp is the left halo), one level
//                       test per block row -- "a run of >= l blocks of height
//                       >= l", l = best D - 1 -- two rows per vote.  A unit
//                       owns 16 block rows and warms its heights up on the 31
//                       rows above.  Hits (rare) get their exact D and go to a
//                       candidate list.
//   sieve_verify_kernel (runs beside the coarse pass, taking candidates as they
//                       appear) runs Algorithm 1 exactly (per-column heights,
//                       one test per row, leftmost window) on the <= 229 x 229
//                       cell window of every candidate with D >= max D - 1 and
//                       keeps the best (side, first bottom row, leftmost column)
//                       key.
//
// The answer is exact whenever the sieve decides: max D in [7, 26] (answers
// 56..222) and the candidate list did not overflow.  Otherwise status bit 1
// (blocks too large, list overflow) or bit 2 (max D < 7: nothing above 62 in
// these rows) asks the caller to run the band engine (MSQ_EAGAIN); nothing is
// guessed.
//
// Multi-GPU: a rank prepends the last SV_HALO_ROWS (256 >= 222) rows of the
// rank above (`halo`), so every square the sieve can report lies wholly inside
// the rows of the rank that holds its bottom row: no carry exchange, no fix-up.
#pragma once

namespace msq {

constexpr int SV_PL = 5;           // height planes: block heights saturate at 31
constexpr int SV_EDGE = 31;        // block rows above a unit that warm its heights up (they saturate at 31)
constexpr int SV_OWN = 16;         // block rows a coarse unit owns
constexpr int SV_PHASES = 4;       // the streaming pass covers the matrix in up to this many sweeps (top quarter first, ...)
constexpr int SV_DMAX = 26;        // windows of 8 * 26 + 21 = 229 columns (from column 2 mod 8) fit 8 words
constexpr int SV_LMIN = 6;         // lowest level tested; the sieve decides for max D >= 7
constexpr int SV_CAP = 32768;      // candidate list entries
constexpr int SV_TR = 8;           // rows per tile = block height
constexpr int SV_MAXSLOTS = 16;    // TMA ring depth
constexpr int SV_HALO_ROWS = 256;  // rows a rank borrows from the rank above
constexpr int SV_VROWS = 8 * SV_DMAX + 21;
constexpr int SV_VWARPS = 8;       // verifier warps per CTA (one candidate per CTA; a power of two)
constexpr int SV_EWARPS = 4;       // coarse-kernel warps per CTA (one unit each)

struct SieveCtl {
    int best;   // largest D found so far
    int count;  // candidates appended
    int abort;  // bit 0: D beyond SV_DMAX, bit 1: candidate list overflow
    int done;   // coarse-pass warps that have finished (the verifier's cue that the list is final)
};

struct SieveParams {
    const uint8_t* src;   // local rows
    const uint8_t* halo;  // halo_rows rows above them (multi-GPU) or nullptr
    long long ld_bytes, halo_ld_bytes;
    int halo_rows;        // multiple of 8
    int rows;             // halo_rows + local rows
    int cols, W;
    long long row_base;   // global row index of row 0 of (halo, local rows)
    int CR, CC, CWn, WC;  // block rows, block columns, 32-block words per row, coarse warp columns (31 words each)
    int nbands, nchunks, wmax, nslots, slot_row_bytes;  // streaming pass: bands x chunks CTAs, wmax warps of 32 words
    int nunits;           // coarse pass: ceil(CR / SV_OWN) row units x WC warps
    uint32_t* G;          // [CR][CWn] block bitmap
    int coarse_warps;     // warps of sieve_coarse_kernel's grid: ctl->done ends there
    int nphases;          // sweeps of the streaming pass over the matrix (<= SV_PHASES; 1 for short slices)
    int prow[SV_PHASES + 1];  // their block-row borders: 0 = prow[0] < ... < prow[nphases] = CR
    int* pcnt;            // [SV_PHASES] streaming warps done with each phase (zeroed with ctl)
    int ptarget;          // = CTAs' consumer warps in total: a phase is complete at this count
    unsigned long long* cand;  // [SV_CAP] D << 40 | block row << 16 | block column
    SieveCtl* ctl;
    unsigned char* result;
};

__device__ __forceinline__ const uint8_t* sv_row(const SieveParams& p, int r) {
    return r < p.halo_rows ? p.halo + (size_t)r * p.halo_ld_bytes
                           : p.src + (size_t)(r - p.halo_rows) * p.ld_bytes;
}
// Phase (sweep) ph of the streaming pass covers block rows [prow[ph], prow[ph + 1]); CTA
// (band b) streams one contiguous piece of every phase.
__device__ __forceinline__ int sv_band_cr0(const SieveParams& p, int ph, int band) {
    return p.prow[ph] + (int)(((long long)(p.prow[ph + 1] - p.prow[ph]) * band) / p.nbands);
}
// the phase that produces block row R
__device__ __forceinline__ int sv_phase_of(const SieveParams& p, int R) {
    int ph = 0;
    while (ph + 1 < p.nphases && R >= p.prow[ph + 1]) ++ph;
    return ph;
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
        if (idx < SV_CAP)  // entries are nonzero; the verifier waits for a reserved slot to fill
            *(volatile unsigned long long*)(p.cand + idx) =
                ((unsigned long long)D << 40) | ((unsigned long long)R << 16) | (unsigned long long)(32 * g + j);
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

// One block row of the coarse Algorithm 1: heights, one test at the level (the
// replay path of SvBatch and its reference semantics).
__device__ __forceinline__ void sv_step(const SieveParams& p, uint32_t v, uint32_t (&h)[SV_PL], int& lvl,
                                        bool record, int R, int g, bool own, int lane) {
    planes_step<SV_PL>(h, v);
    uint32_t hits = sv_hits(h, lvl, lane);
    if (!own) hits = 0u;
    if (__any_sync(0xFFFFFFFFu, hits != 0u))
        lvl = sv_rare(p, h[0], h[1], h[2], h[3], h[4], hits, lvl, record, R, g, lane);
}

// The same, SV_BATCH block rows at a time.  A block with height >= l at one of
// the batch's rows had height >= l - SV_BATCH before the batch and a one in its
// first row, so a run of l such blocks is necessary for a hit anywhere in the
// batch: one compare, one shuffle, one run filter and one vote per batch; the
// rows in between only advance the heights.  A batch that passes the filter is
// replayed row by row (sv_step) from the heights it started with.  The level
// is the one the batch started with (levels only rise: a stale one adds hits).
#ifndef MSQ_SV_BATCH
#define MSQ_SV_BATCH 2
#endif
constexpr int SV_BATCH = MSQ_SV_BATCH;
struct SvBatch {
    uint32_t h0[SV_PL];    // heights before the batch
    uint32_t v[SV_BATCH];  // G words of its rows
    // branch-free forms of planes_ge (at lvl - SV_BATCH) / sv_runs (lvl) for the current level
    uint32_t nb[SV_PL];
    int sh[5];
    int lvl_of;

    __device__ __forceinline__ void set_level(int lvl) {
        lvl_of = lvl;
        const int lf = max(lvl - SV_BATCH, 0);
#pragma unroll
        for (int k = 0; k < SV_PL; ++k) nb[k] = ((lf >> k) & 1) ? 0u : 0xFFFFFFFFu;
        int have = 1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            sh[k] = 2 * have <= lvl ? have : 0;
            if (2 * have <= lvl) have *= 2;
        }
        sh[4] = lvl - have;
    }
    __device__ __forceinline__ void begin(const uint32_t (&h)[SV_PL]) {
#pragma unroll
        for (int k = 0; k < SV_PL; ++k) h0[k] = h[k];
#pragma unroll
        for (int j = 0; j < SV_BATCH; ++j) v[j] = 0u;
    }
    __device__ __forceinline__ void push(uint32_t (&h)[SV_PL], uint32_t vv, int j) {
        planes_step<SV_PL>(h, vv);
        v[j] = vv;
    }
    // can any row of the batch hold a hit (warp-uniform)
    __device__ __forceinline__ bool test(bool own, int lane) const {
        uint32_t ge = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
        for (int k = SV_PL - 1; k >= 0; --k) {
            ge |= eq & h0[k] & nb[k];
            eq &= h0[k] | nb[k];
        }
        uint32_t hi = (ge | eq) & v[0];
        uint32_t lo = __shfl_up_sync(0xFFFFFFFFu, hi, 1);
        if (lane == 0) lo = 0u;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            hi &= __funnelshift_l(lo, hi, sh[k]);
            lo &= lo << sh[k];
        }
        if (!own) hi = 0u;
        return __any_sync(0xFFFFFFFFu, hi != 0u);
    }
};

// finish a batch of cnt rows whose first block row is R0; h = heights after it
__device__ __forceinline__ void sv_batch_end(const SieveParams& p, SvBatch& bt, uint32_t (&h)[SV_PL], int cnt,
                                             int& lvl, int rec_from, int R0, int g, bool own, int lane) {
    if (bt.test(own, lane)) {
#pragma unroll
        for (int k = 0; k < SV_PL; ++k) h[k] = bt.h0[k];
        for (int j = 0; j < cnt; ++j) {
            uint32_t vj = bt.v[0];
#pragma unroll
            for (int u = 1; u < SV_BATCH; ++u) vj = j == u ? bt.v[u] : vj;
            sv_step(p, vj, h, lvl, R0 + j >= rec_from, R0 + j, g, own, lane);
        }
    }
    if (lvl != bt.lvl_of) bt.set_level(lvl);
    bt.begin(h);
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

__global__ void __launch_bounds__(288, 1) sieve_pass_kernel(const SieveParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int band = blockIdx.x / p.nchunks, chunk = blockIdx.x - band * p.nchunks;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Wp = (p.W + 3) & ~3;     // rows are copied in 16-byte units (the stride covers the pad words)
    const int WF = (Wp + 255) / 256;   // warp columns of 256 matrix words
    const int wc0 = WF * chunk / p.nchunks, wc1 = WF * (chunk + 1) / p.nchunks;
    const int ncw = wc1 - wc0;  // consumer warps of this chunk
    // nphases contiguous sub-bands per CTA, one per sweep (quarter) of the matrix, so the
    // bitmap of a quarter is complete while the next one streams and the coarse pass
    // (launched beside this kernel) works on it.  (Interleaving single tiles instead
    // cost 30% of the bandwidth: 89 -> 116 us on cfg4.)
    int tiles_of[SV_PHASES], first_of[SV_PHASES];
#pragma unroll
    for (int ph = 0; ph < SV_PHASES; ++ph) {
        first_of[ph] = ph < p.nphases ? sv_band_cr0(p, ph, band) : 0;
        tiles_of[ph] = ph < p.nphases ? sv_band_cr0(p, ph, band + 1) - first_of[ph] : 0;
    }
    const int mw0 = 256 * wc0;  // matrix words [mw0, mw1) of each row
    const int mw1 = min(Wp, 256 * wc1);
    const uint32_t chunk_bytes = (uint32_t)(mw1 - mw0) * 4u;
    const uint32_t srb = (uint32_t)p.slot_row_bytes;
    const uint32_t slot_bytes = SV_TR * srb;
    uint8_t* ring = smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)p.nslots * slot_bytes);
    uint64_t* empty = full + SV_MAXSLOTS;

    if (tid == 0) {
        for (int s = 0; s < p.nslots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (uint32_t)ncw);
        }
        fence_mbar_init();
    }
    if (blockIdx.x == 0 && tid < 8) {  // written again by the verifier only (tens of microseconds later)
        ((uint32_t*)p.result)[tid] = 0u;
        __threadfence();
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the coarse pass waits on the phase counters
    if (ncw <= 0) return;

    // ------------------------------------------------------------ producer
    if (warp == p.wmax) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int s = 0, lap = 0;
#pragma unroll 1
            for (int ph = 0; ph < p.nphases; ++ph) {
                for (int q = 0; q < tiles_of[ph]; ++q) {
                    if (lap > 0) mbar_wait(&empty[s], (uint32_t)((lap - 1) & 1));
                    mbar_expect_tx(&full[s], SV_TR * chunk_bytes);
                    uint8_t* dst = ring + (size_t)s * slot_bytes;
                    const int r = SV_TR * (first_of[ph] + q);
#pragma unroll
                    for (int b = 0; b < SV_TR; ++b)
                        tma_row(dst + (size_t)b * srb, sv_row(p, r + b) + (size_t)mw0 * 4, chunk_bytes, &full[s], pol);
                    if (++s == p.nslots) {
                        s = 0;
                        ++lap;
                    }
                }
            }
        }
        return;
    }
    if (warp >= ncw) return;

    // ------------------------------------------------------------ consumers
    const int g = 32 * (wc0 + warp) + lane;  // the lane's 32-block word of G
    const bool in = g < p.CWn;
    uint32_t validc = 0u;
    if (in) {
        const int n = p.CC - 32 * g;
        validc = n >= 32 ? 0xFFFFFFFFu : (n > 0 ? (1u << n) - 1u : 0u);
    }
    // the lane's 8 matrix words = two 16-byte halves; lanes 4..7 (mod 8) read the
    // upper half first so a quarter-warp's 8 loads cover all 32 banks
    const int sw = (lane >> 2) & 1;
    const bool okA = 8 * g + 4 * sw < mw1;
    const bool okB = 8 * g + 4 * (1 - sw) < mw1;
    const uint32_t ring_s = smem_addr(ring);
    const uint32_t offA = okA ? (uint32_t)(8 * g + 4 * sw - mw0) * 4u : 0u;
    const uint32_t offB = okB ? (uint32_t)(8 * g + 4 * (1 - sw) - mw0) * 4u : 0u;
    int s = 0;
    uint32_t par = 0u;
#pragma unroll 1
    for (int ph = 0; ph < p.nphases; ++ph) {
        uint32_t* grow = p.G + (size_t)first_of[ph] * p.CWn + (in ? g : 0);
        for (int q = 0; q < tiles_of[ph]; ++q) {
            mbar_wait(&full[s], par);
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
            if (in) grow[(size_t)q * p.CWn] = v;
            if (++s == p.nslots) {
                s = 0;
                par ^= 1u;
            }
        }
        // this warp's words of the phase are out: release the phase counter
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.pcnt + ph, 1);
    }
}

// Algorithm 1 on the block bitmap G.  Unit = (SV_OWN block rows, warp column of
// 31 words + the halo word on the left).  The 31 rows above the unit rebuild
// its carried-in heights (they saturate at 31); one climb at the last of them
// gives the unit a local lower bound for the shared best before it records
// anything.  The first unit has no rows above it and walks its own first rows
// for that bound, then starts again from zero heights.
__device__ __forceinline__ void sv_coarse_unit(const SieveParams& p, int unit, int lane) {
    if (unit >= p.nunits * p.WC) return;
    const int ru = unit / p.WC, wc = unit - ru * p.WC;
    const int g = 31 * wc - 1 + lane;
    const bool in = g >= 0 && g < p.CWn;
    const bool own = lane > 0 && in;
    const int R0 = ru * SV_OWN, R1 = min(p.CR, R0 + SV_OWN);
    const int Rw = ru > 0 ? R0 - SV_EDGE : 0;               // first warm-up row
    const int nwarm = ru > 0 ? SV_EDGE : min(SV_EDGE, R1);  // rows walked for heights only
    const uint32_t* gp = p.G + (in ? g : 0);
    // every word the unit needs in flight at once: the warm-up rows (last first), its
    // own rows, the control block
    uint32_t c[SV_EDGE + 2], vv[SV_OWN];
#pragma unroll
    for (int k = 1; k <= SV_EDGE; ++k)
        c[k] = (in && k <= nwarm) ? __ldcg(gp + (size_t)(Rw + nwarm - k) * p.CWn) : 0u;
#pragma unroll
    for (int j = 0; j < SV_OWN; ++j) vv[j] = (in && R0 + j < R1) ? __ldcg(gp + (size_t)(R0 + j) * p.CWn) : 0u;
    const int gbest = ld_volatile(&p.ctl->best);
    if (ld_volatile(&p.ctl->abort)) return;
    // ---- warm-up: heights only.  c[k] = "the last k rows are ones" is monotone in k,
    // so the height (how many k hold) has bit b set where c[m * 2^b] holds and
    // c[(m + 1) * 2^b] does not, m odd.
    uint32_t h[SV_PL];
    c[0] = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 1; k <= SV_EDGE; ++k) c[k] &= c[k - 1];
    c[SV_EDGE + 1] = 0u;
#pragma unroll
    for (int b = 0; b < SV_PL; ++b) {
        uint32_t acc = 0u;
#pragma unroll
        for (int m = 1; (m << b) <= SV_EDGE; m += 2) acc |= c[m << b] & ~c[min((m + 1) << b, SV_EDGE + 1)];
        h[b] = acc;
    }
    int lvl = max(SV_LMIN, gbest - 1);
    {   // one climb at the last warm-up row: a lower bound, nothing recorded
        uint32_t hits = sv_hits(h, lvl, lane);
        if (!own) hits = 0u;
        if (__any_sync(0xFFFFFFFFu, hits != 0u))
            lvl = sv_rare(p, h[0], h[1], h[2], h[3], h[4], hits, lvl, false, 0, g, lane);
    }
    if (ru == 0) {  // the first unit's own rows start from zero heights
#pragma unroll
        for (int k = 0; k < SV_PL; ++k) h[k] = 0u;
    }
    SvBatch bt;
    bt.set_level(lvl);
    bt.begin(h);
    // ---- own rows
#pragma unroll
    for (int part = 0; part < SV_OWN / SV_BATCH; ++part) {
        const int r0 = R0 + part * SV_BATCH;
        const int cnt = min(SV_BATCH, R1 - r0);
        if (cnt > 0) {
#pragma unroll
            for (int j = 0; j < SV_BATCH; ++j)
                if (j < cnt) bt.push(h, vv[part * SV_BATCH + j], j);
            sv_batch_end(p, bt, h, cnt, lvl, 0, r0, g, own, lane);
        }
    }
}

__global__ void __launch_bounds__(32 * SV_EWARPS) sieve_coarse_kernel(const SieveParams p) {
    // Launched beside sieve_pass_kernel (programmatic dependent launch without
    // griddepcontrol.wait): the CTA starts when the phases that produce its units'
    // block rows are complete (counters released by the streaming warps).
    __shared__ int go;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // the verifier's CTAs launch once every CTA of this grid has started and take the
    // candidates while the last units still run
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    {
        const int last_unit = min(blockIdx.x * SV_EWARPS + SV_EWARPS, p.nunits * p.WC) - 1;
        const int last_row = min(p.CR, (last_unit / p.WC + 1) * SV_OWN) - 1;
        if (threadIdx.x == 0) {
            const int ph1 = sv_phase_of(p, last_row);
            const volatile int* c = p.pcnt;
            int ok = 1;
            long long spins = 0;
            for (int ph = 0; ph <= ph1 && ok; ++ph)
                while (c[ph] < p.ptarget) {
                    __nanosleep(400);
                    if (++spins > (1ll << 23)) {  // never in practice: hand the input to the band engine
                        atomicOr(&p.ctl->abort, 2);
                        ok = 0;
                        break;
                    }
                }
            __threadfence();
            go = ok;
        }
        __syncthreads();
    }
    if (go) sv_coarse_unit(p, blockIdx.x * SV_EWARPS + warp, lane);
    __threadfence();  // this warp's candidates before its count in ctl->done
    __syncwarp();
    if (lane == 0) atomicAdd(&p.ctl->done, 1);
}

// Algorithm 1 on the cell window of every candidate that can still hold the
// answer; one CTA per candidate.  The grid is launched while the coarse pass
// still runs (programmatic dependent launch, no griddepcontrol.wait): CTA b takes
// list entries b, b + CTAs, ... as they appear and leaves when every coarse warp
// has finished (ctl->done) and its entries are used up.  A candidate is skipped
// when the shared best D or the best side so far already rule it out (both only
// grow).  All threads load the window (every load in flight at once) and fold
// the zeros of the rows before the first testable row into per-column last-zero
// rows.  Every warp then walks the remaining rows (heights from the last-zero
// rows) and tests every SV_VWARPS-th of them: at the best side so far (a tie),
// then upwards until the row's own largest square is known.  The largest key --
// side, then first bottom row, then leftmost column -- is Algorithm 1's answer
// for the window (squares.py:93-97).
__global__ void __launch_bounds__(32 * SV_VWARPS) sieve_verify_kernel(const SieveParams p) {
    __shared__ __align__(16) uint32_t rowsm[SV_VROWS][8];
    __shared__ int lzs[256];
    __shared__ int tsh;                   // best side so far (this window or any other)
    __shared__ unsigned long long keysh;  // best key of this window
    __shared__ unsigned long long csh;    // the candidate being worked on (0: none, 1: leave)
    __shared__ int bsh;                   // shared best D when it was taken
    constexpr int NT = 32 * SV_VWARPS;
    constexpr int LPT = (SV_VROWS * 8 + NT - 1) / NT;  // window words per thread
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int next = blockIdx.x;
    for (;;) {
        __syncthreads();  // the previous candidate's rows are done with
        if (tid == 0) {
            // wait for entry `next`, or for the end of the coarse pass
            unsigned long long c = 1ull;
            long long spins = 0;
            for (;;) {
                const int done = ld_volatile(&p.ctl->done) >= p.coarse_warps;  // read before the count
                __threadfence();
                const int count = min(ld_volatile(&p.ctl->count), SV_CAP);
                if (ld_volatile(&p.ctl->abort) && done) {  // undecided: nothing left to verify
                    c = 1ull;
                    break;
                }
                if (next < count) {
                    c = *(volatile unsigned long long*)(p.cand + next);
                    if (c) break;  // (a reserved slot whose entry has not landed yet reads 0)
                } else if (done) {
                    c = 1ull;
                    break;
                }
                __nanosleep(500);
                if (++spins > (1ll << 24)) {  // never in practice
                    atomicOr(&p.ctl->abort, 2);
                    c = 1ull;
                    break;
                }
            }
            csh = c;
            bsh = ld_volatile(&p.ctl->best);
            tsh = max(8 * bsh, ld_volatile(res_best(p.result)));  // ties at the best side so far
            keysh = 0ull;
        }
        for (int i = tid; i < 256; i += NT) lzs[i] = -1;
        __syncthreads();
        const unsigned long long c = csh;
        if (c == 1ull) break;
        next += gridDim.x;
        const int D = (int)(c >> 40), t0 = tsh;
        // CTA-uniform.  (D beyond SV_DMAX: the solve is already marked undecided and the
        // window would not fit.)
        if (D < bsh - 1 || D > SV_DMAX || 8 * D + 14 < t0) continue;
        const int Rg = (int)((c >> 16) & 0xFFFFFFull), cg = (int)(c & 0xFFFFull);
        const int r_hi = min(p.rows - 1, 8 * Rg + 14), r_lo = max(0, 8 * (Rg - D) - 6);
        const int c_hi = min(p.cols - 1, 8 * cg + 14), c_lo = max(0, 8 * (cg - D) - 6);
        const int nr = r_hi - r_lo + 1, wa = c_lo >> 5, nwd = (c_hi >> 5) - wa + 1;
        const int first = t0 - 1;  // first row (window-relative) whose heights can reach t0
        auto word_mask = [&](int k) -> uint32_t {
            const int lo = max(c_lo - 32 * (wa + k), 0), hi = min(c_hi - 32 * (wa + k), 31);
            return (k < nwd && hi >= lo) ? ((hi == 31 ? 0xFFFFFFFFu : (1u << (hi + 1)) - 1u) & ~((1u << lo) - 1u)) : 0u;
        };
        uint32_t wv[LPT];
#pragma unroll
        for (int u = 0; u < LPT; ++u) {
            const int i = tid + NT * u, rr = i >> 3, k = i & 7;
            wv[u] = (rr < nr && k < nwd) ? __ldg((const uint32_t*)(sv_row(p, r_lo + rr)) + wa + k) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < LPT; ++u) {
            const int i = tid + NT * u, rr = i >> 3, k = i & 7;
            if (rr < nr) {
                rowsm[rr][k] = wv[u];
                if (rr < first) {
                    uint32_t z = ~wv[u] & word_mask(k);
                    while (z) {
                        const int j = __ffs(z) - 1;
                        z &= z - 1;
                        atomicMax(&lzs[32 * k + j], rr);
                    }
                }
            }
        }
        __syncthreads();
        uint32_t msk[8];
        int lz[8];  // last zero row (window-relative) of column 32k + lane
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            msk[k] = word_mask(k);
            lz[k] = lzs[32 * k + lane];
        }
        // leftmost window end of t columns of height >= t at row rr, or -1
        auto window = [&](int rr, int t) -> int {
            int run = 0, e = -1;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t x = __ballot_sync(0xFFFFFFFFu, rr - lz[k] >= t) & msk[k];
                const int pre = x == 0xFFFFFFFFu ? 32 : __ffs(~x) - 1;
                if (e < 0 && run + pre >= t) e = 32 * k + (t - run) - 1;
                run = x == 0xFFFFFFFFu ? run + 32 : __clz(~x);
            }
            return e;
        };
        for (int rr = max(first, 0); rr < nr; ++rr) {
            const uint4 a = *(const uint4*)&rowsm[rr][0];
            const uint4 b = *(const uint4*)&rowsm[rr][4];
            const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if ((w[k] & msk[k]) != msk[k] && !((w[k] >> lane) & 1u)) lz[k] = rr;
            if (((rr - first) & (SV_VWARPS - 1)) != warp) continue;  // another warp's row
            int t = *(volatile int*)&tsh;
            if (rr + 1 < t || t > nr) continue;
            int e = window(rr, t);
            if (e < 0) continue;
            for (;;) {  // the row's own largest square
                const int e2 = rr + 1 > t ? window(rr, t + 1) : -1;
                if (e2 < 0) break;
                e = e2;
                ++t;
            }
            if (lane == 0) {
                atomicMax(&tsh, t);
                atomicMax(&keysh, pack_key(t, p.row_base + r_lo + rr, (long long)32 * wa + e));
            }
        }
        __syncthreads();
        if (tid == 0 && keysh) {
            atomicMax(res_key1(p.result), keysh);
            atomicMax(res_best(p.result), (int)(keysh >> (2 * KEY_DIM_BITS)));
        }
    }
    // the coarse pass is complete here: can the sieve answer at all?
    if (blockIdx.x == 0 && tid == 0) {
        const int aborted = ld_volatile(&p.ctl->abort), best = ld_volatile(&p.ctl->best);
        // undecided: blocks too large for the windows / too many candidates (bit 1), or
        // no block square of side 7 in these rows, i.e. nothing above 8 * 6 + 14 = 62
        // here (bit 2: still decided if another rank holds a larger square)
        if (aborted || best <= SV_LMIN) atomicOr(res_status(p.result), aborted ? 2u : 4u);
    }
}

}  // namespace msq
