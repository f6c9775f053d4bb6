// msq_strip.cuh -- barrier-free band pass for bit-packed matrices (sm_100a).
//
// Same band outputs as pass1_kernel (band key, first-zero depths e, bottom
// runs b, all-ones masks), for bit-packed bands whose threshold starts (from
// the lower-bound seed or the shared best side) in [STRIP_TMIN, STRIP_TMAX].
//
// Why it is exact without any CTA-wide synchronisation: let g_w(r) be the
// largest side of a square whose bottom-right cell lies in row r and in the
// column strip owned by warp w.  A k-square ending at (r, c) contains a
// (k-1)-square ending at (r-1, c), so g_w(r) <= g_w(r-1) + 1 (SURVEY P2 per
// strip) and Algorithm 1 (squares.py:84-103) run on the strip alone -- one
// test per row at t = best_w + 1 -- finds max_r g_w(r) and the first row and
// leftmost end where it occurs.  The band answer is the max of the strips'
// keys.  Thresholds may jump to a side M found elsewhere (tested as a tie, at
// t = M), exactly as the band engine shares its best side.
//
// Layout: warp w reads the window of 128 words [120w - 8, 120w + 120) of each
// row (4 words per lane, one 16-byte smem load), owns the 120 words from
// 120w on, and uses the 8 words to the left as a halo: every window of
// t <= STRIP_TMAX columns ending in its own words lies in the window.  Rows
// arrive through a TMA ring of 8-row slots (one bulk copy, one full and one
// empty mbarrier per slot); a producer warp refills a slot once every
// consumer warp released it.  No __syncthreads in the row loop.
//
// Per 8-row tile and word (threshold t >= 96, so any t-run of eligible
// columns contains >= Lmin = ceil((t-62)/32) whole "F" words, i.e. words with
// no zero in the last t rows -- the band engine's mode L):
//   zm  = rows of the tile with a zero in the word (8 flags)
//   F rows = [Z + t - rho0, first zero in the tile)   (Z = last zero row before)
//   a shuffle brings the left lane's 4 words; runs of Lmin F words are found
//   with byte-wise ANDs over the 8 row masks at once.
// Runs (rare) are checked exactly from per-column last-zero rows that each
// warp keeps for its own window in global scratch (written on zero events).
#pragma once

namespace msq {

constexpr int STRIP_WORDS = 128;  // words in a warp's window
constexpr int STRIP_HALO = 8;     // of which the first 8 are the halo
constexpr int STRIP_STRIDE = STRIP_WORDS - STRIP_HALO;
constexpr int STRIP_TR = 8;       // rows per tile (= per ring slot)
constexpr int STRIP_TMIN = 96;    // word-level filter valid (runs contain >= 2 whole words)
constexpr int STRIP_TMAX = 222;   // Lmin <= 5 (one neighbour lane) and t - 1 <= 32 * 7 (halo)
constexpr int STRIP_MAXSLOTS = 4;

struct StripParams {
    const uint8_t* src;
    long long ld_bytes;
    int rows, cols, W, nbands, cols_pad;
    long long row_base;
    int nslots, row_bytes, nwarps;
    uint16_t* zw;  // [nbands][nwarps][128*32] last-zero rows of each warp's window
    uint16_t* zb;  // [nbands][cols_pad] bottom runs (band output)
    uint16_t* e_out;
    uint32_t* ao_out;
    unsigned long long* band_keys;
    unsigned char* results;
    int* redo;  // [nbands]: 1 = band left to pass1_kernel (threshold outside the strip range)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ int strip_lmin(int t) { return (t - 62 + 31) / 32; }

__global__ void __launch_bounds__(640, 1) strip_kernel(const StripParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int band = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    const int ntiles = (H + STRIP_TR - 1) / STRIP_TR;
    const int slot_bytes = STRIP_TR * p.row_bytes;
    uint8_t* ring = smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)p.nslots * slot_bytes);
    uint64_t* empty = full + STRIP_MAXSLOTS;
    int* sh = (int*)(empty + STRIP_MAXSLOTS);  // [0] start threshold, [1] CTA best, [2] abort
    unsigned long long* skey = (unsigned long long*)(sh + 4);
    uint32_t* nz_sm = (uint32_t*)(sh + 8);  // [nwarps][128] never-zeroed masks of the warps' windows
    unsigned char* result = p.results;

    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the seed
    if (tid == 0) {
        const int t0 = max(1, ld_volatile(res_best(result)));
        sh[0] = t0;
        sh[1] = t0;
        sh[2] = 0;
        *skey = 0ull;
        const bool ok = t0 >= STRIP_TMIN && t0 <= STRIP_TMAX;
        p.redo[band] = ok ? 0 : 1;
        for (int s = 0; s < p.nslots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.nwarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int t0 = sh[0];
    if (t0 < STRIP_TMIN || t0 > STRIP_TMAX) return;  // pass1_kernel redoes this band

    // ------------------------------------------------------------ producer
    if (warp == p.nwarps) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            const uint8_t* bsrc = p.src + (size_t)r0 * p.ld_bytes;
            const bool contiguous = p.ld_bytes == (long long)p.row_bytes;
            for (int q = 0; q < ntiles; ++q) {
                const int s = q % p.nslots;
                if (q >= p.nslots) mbar_wait(&empty[s], (uint32_t)((q / p.nslots - 1) & 1));
                const int n = min(STRIP_TR, H - q * STRIP_TR);
                mbar_expect_tx(&full[s], (uint32_t)(n * p.row_bytes));
                uint8_t* dst = ring + (size_t)s * slot_bytes;
                const uint8_t* srow = bsrc + (size_t)q * STRIP_TR * p.ld_bytes;
                if (contiguous) {
                    tma_row(dst, srow, (uint32_t)(n * p.row_bytes), &full[s], pol);
                } else {
                    for (int b = 0; b < n; ++b)
                        tma_row(dst + (size_t)b * p.row_bytes, srow + (size_t)b * p.ld_bytes, (uint32_t)p.row_bytes,
                                &full[s], pol);
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int base_word = STRIP_STRIDE * warp - STRIP_HALO;
    const int i0 = 4 * lane;  // first window index of this lane
    uint32_t VAL[4];
    int ZW[4];
    uint32_t fullk = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int a = base_word + i0 + k;
        VAL[k] = (a >= 0 && a < p.W) ? valid_mask(a, p.W, p.cols) : 0u;
        ZW[k] = 0;
        fullk |= (VAL[k] == 0xFFFFFFFFu ? 1u : 0u) << k;
    }
    uint32_t own_mask = 0;  // words of this lane the warp owns (not halo, inside the matrix)
#pragma unroll
    for (int k = 0; k < 4; ++k) own_mask |= (i0 + k >= STRIP_HALO && VAL[k] != 0u ? 1u : 0u) << k;
    // smem byte offset of the lane's 4 words inside a row (clamped for words outside the row)
    const int a_ld = min(max(base_word + i0, 0), p.W - 4);
    const uint32_t ring_s = smem_addr(ring) + (uint32_t)(a_ld * 4);
    uint16_t* zwin = p.zw + ((size_t)band * p.nwarps + warp) * (STRIP_WORDS * 32);
    uint32_t* nzw = nz_sm + warp * STRIP_WORDS;
    *(uint4*)(nzw + i0) = make_uint4(VAL[0], VAL[1], VAL[2], VAL[3]);
    // the only word of the matrix that can be partial is W-1
    const int kpart = (p.cols & 31) ? (p.W - 1) - (base_word + i0) : -1;
    const uint32_t valpart = (kpart >= 0 && kpart < 4) ? valid_mask(p.W - 1, p.W, p.cols) : 0xFFFFFFFFu;
    __syncwarp();
    const size_t sum_base = (size_t)band * p.cols_pad;
    uint16_t* ebase = p.e_out + sum_base + (ptrdiff_t)(base_word + i0) * 32;  // e of the lane's first word

    int t = t0;
    int lmin = strip_lmin(t);
    unsigned long long key = 0ull;
    bool aborted = false;

    const uint32_t rb_bytes = (uint32_t)p.row_bytes;
    int s = 0;          // ring slot of tile q
    uint32_t par = 0u;  // its full-barrier phase parity
    for (int q = 0; q < ntiles; ++q, s = (s + 1 == p.nslots) ? 0 : s + 1, par ^= (s == 0) ? 1u : 0u) {
        const int row0 = q * STRIP_TR;
        const int nrows = min(STRIP_TR, H - row0);
        const int rho0 = row0 + 1;
        const uint32_t slot_s = ring_s + (uint32_t)(s * slot_bytes);
        // the grid's best side every 8 tiles, loaded here and used after the tile
        const int gglob = (q & 7) == 7 ? ld_volatile(res_best(result)) : 0;
        mbar_wait(&full[s], par);
        if (aborted) {  // keep the ring moving; pass1_kernel redoes the band
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            continue;
        }
        // ---- zero rows of each word over the tile
        // N: nibble b = which of the 4 words have a zero in tile row b
        // (all 8 rows of the slot are read; rows past the band end are masked off)
        uint32_t N = 0u;
#pragma unroll
        for (int b = 0; b < STRIP_TR; ++b) {
            uint32_t w[4];
            lds_words<4>(slot_s + (uint32_t)b * rb_bytes, w);
            uint32_t nb = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) nb |= ((~w[k] & VAL[k]) != 0u ? 1u : 0u) << k;
            N |= nb << (4 * b);
        }
        if (nrows < STRIP_TR) N &= (1u << (4 * nrows)) - 1u;
        // zm[k]: rows of word k with a zero, spread 4 bits apart (bit 4b)
        uint32_t zm[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) zm[k] = (N >> k) & 0x11111111u;
        // ---- F rows per word at t (before this tile's zeros move Z)
        uint32_t X = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int hi = zm[k] ? (__ffs(zm[k]) - 1) >> 2 : nrows;
            const int lo = max(0, ZW[k] + t - rho0);
            const uint32_t fr = ((fullk >> k) & 1u) && lo < hi ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
            X |= fr << (8 * k);
        }
        // runs of lmin F words ending in this lane's words: bytes = row masks of
        // the 8 words (left lane's 4, then ours); AND over lmin consecutive bytes
        const uint32_t PX = __shfl_up_sync(0xFFFFFFFFu, X, 1);
        // bytes of our 4 words ANDed with the lmin-1 bytes before each: funnel
        // shifts of (left lane's 4, ours); lmin <= 5, unused steps are all-ones
        const uint32_t PL = lane ? PX : 0u;
        uint32_t cm = X;
#pragma unroll
        for (int i = 1; i < 5; ++i) cm &= i < lmin ? __funnelshift_lc(PL, X, 8 * i) : 0xFFFFFFFFu;
        cm |= cm >> 16;
        cm |= cm >> 8;
        const uint32_t crows = __reduce_or_sync(0xFFFFFFFFu, cm & 0xFFu);

        if (crows) {
            // ---- rare path: rows with a candidate run, in order, at the running t.
            // Column state is the pre-tile state (zwin, NZ) plus the tile's own
            // rows up to the tested one, read back from the ring slot.
            for (int b = 0; b < nrows; ++b) {
                if (!((crows >> b) & 1u)) continue;  // warp-uniform
                const int rho = rho0 + b;
                uint32_t nib = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool f = ((fullk >> k) & 1u) && !(zm[k] & ((2u << (4 * b)) - 1u)) && ZW[k] + t <= rho;
                    nib |= (f ? 1u : 0u) << k;
                }
                // F words reaching the top of each lane's nibble (segmented scan)
                int R = __clz(~(nib << 28));
                bool allf = nib == 0xFu;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int o = __shfl_up_sync(0xFFFFFFFFu, R | (allf ? 0x10000 : 0), d);
                    if (lane >= d && allf) {
                        R += o & 0xFFFF;
                        allf = (o >> 16) & 1;
                    }
                }
                int cin = __shfl_up_sync(0xFFFFFFFFu, R, 1);
                if (lane == 0) cin = 0;
                const uint32_t nb0 = __shfl_down_sync(0xFFFFFFFFu, nib & 1u, 1);
                const uint32_t ends = nib & ~((nib >> 1) | ((lane < 31 ? nb0 : 0u) << 3));
                int cand0 = -1, cand1 = -1;  // at most two runs end in a nibble
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if ((ends >> k) & 1u) {
                        const int ones = __clz(~(nib << (31 - k)));
                        const int L = ones == k + 1 ? ones + cin : ones;
                        if (L >= lmin) {
                            const int c = ((i0 + k - L + 1) << 8) | L;
                            if (cand0 < 0) cand0 = c; else cand1 = c;
                        }
                    }
                }
                // column `lane` of window word i at row rho: (last-zero row before the
                // tile, never-zeroed, valid, zero in the tile up to this row)
                auto col_state = [&](int i, int& zr, uint32_t& nzv, uint32_t& vlw, uint32_t& tz) {
                    const int ic = min(max(i, 0), STRIP_WORDS - 1);
                    const int ag = base_word + ic;
                    nzv = nzw[ic];
                    vlw = (i == ic && ag >= 0 && ag < p.W) ? valid_mask(ag, p.W, p.cols) : 0u;
                    zr = zwin[ic * 32 + lane];
                    const int aw = min(max(base_word + ic, 0), p.W - 1);
                    const uint32_t wsl = smem_addr(ring) + (uint32_t)(s * slot_bytes + aw * 4);
                    tz = 0u;
                    for (int bb = 0; bb <= b; ++bb) {
                        uint32_t w1[1];
                        lds_words<1>(wsl + (uint32_t)bb * rb_bytes, w1);
                        tz |= ~w1[0];
                    }
                };
                auto elig = [&](int zr, uint32_t nzv, uint32_t vlw, uint32_t tz) -> uint32_t {
                    const bool e = !((tz >> lane) & 1u) && (((nzv >> lane) & 1u) ? rho >= t : zr + t <= rho);
                    return __ballot_sync(0xFFFFFFFFu, e) & vlw;
                };
                int beste = 0x7FFFFFFF;
#pragma unroll
                for (int ci = 0; ci < 2; ++ci) {
                    const int mine = ci ? cand1 : cand0;
                    unsigned bal = __ballot_sync(0xFFFFFFFFu, mine >= 0);
                    while (bal) {
                        const int l = __ffs(bal) - 1;
                        bal &= bal - 1;
                        const int c = __shfl_sync(0xFFFFFFFFu, mine, l);
                        const int a0 = c >> 8, L = c & 0xFF, a1 = a0 + L;
                        int zl, zrr;
                        uint32_t nl, nr_, vl, vr, tl, tr;
                        col_state(a0 - 1, zl, nl, vl, tl);  // both boundary words' loads in flight
                        col_state(a1, zrr, nr_, vr, tr);
                        const uint32_t el = elig(zl, nl, vl, tl), er = elig(zrr, nr_, vr, tr);
                        const int suf = __clz(~el);
                        const int pre = er == 0xFFFFFFFFu ? 32 : __ffs(~er) - 1;
                        if (suf + 32 * L + pre >= t) {
                            const int st = 32 * a0 - suf;
                            const int e = max(st + t - 1, 32 * STRIP_HALO);
                            if (e <= 32 * a1 + pre - 1) beste = min(beste, e);
                        }
                    }
                }
                if (beste != 0x7FFFFFFF) {  // warp-uniform: raise at this row
                    key = pack_key(t, p.row_base + r0 + rho - 1, (long long)32 * base_word + beste);
                    ++t;
                    if (t > STRIP_TMAX) aborted = true;
                    lmin = strip_lmin(t);
                    if (lane == 0) {
                        atomicMax(&sh[1], t - 1);
                        atomicMax(res_best(result), t - 1);
                    }
                }
            }
        }
        // ---- zero events, one (word, row) event or one zero bit per lane and
        // step, so the lanes' events share the steps: per-column last-zero rows
        // of the window, first zeros (e) of own columns, never-zeroed masks
        {
            uint32_t EV = N;  // bit 4b + k: word k, row b (rows in order per word)
            uint32_t cz = 0u, cn = 0u;
            int zoff = 0, eoff = 0;
            uint16_t crho = 0;
            while (EV | cz) {  // one zero bit per step (an event's first bit in the step that opens it)
                if (!cz) {
                    const int bit = __ffs(EV) - 1;
                    EV &= EV - 1;
                    const int k = bit & 3, b = bit >> 2;
                    uint32_t w1[1];
                    lds_words<1>(slot_s + (uint32_t)b * rb_bytes + 4u * (uint32_t)k, w1);
                    const int i = i0 + k;
                    cz = ~w1[0] & (k == kpart ? valpart : 0xFFFFFFFFu);
                    const uint32_t nk = nzw[i];
                    cn = ((own_mask >> k) & 1u) ? (nk & cz) : 0u;
                    nzw[i] = nk & ~cz;
                    zoff = i * 32;
                    eoff = k * 32;
                    crho = (uint16_t)(rho0 + b);
                }
                const int j = __ffs(cz) - 1;
                cz &= cz - 1;
                zwin[zoff + j] = crho;
                if ((cn >> j) & 1u) ebase[eoff + j] = (uint16_t)(crho - 1);
            }
        }
        // ---- last zero row per word, release the slot
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (zm[k]) ZW[k] = rho0 + ((31 - __clz(zm[k])) >> 2);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // shared best side (ties): the CTA's every tile, the grid's every 8 tiles
        const int g = max(ld_volatile(&sh[1]), gglob);
        if (g > t) {
            t = g;
            if (t > STRIP_TMAX) aborted = true;
            lmin = strip_lmin(t);
        }
    }
    if (aborted && lane == 0) {
        p.redo[band] = 1;
        atomicExch(&sh[2], 1);
    }

    // ------------------------------------------------------------ band outputs (own words)
    // word by word, lanes = columns: coalesced bottom runs, e = H for never-zeroed columns
    if (!aborted) {
        // 8 words per step: their last-zero rows are loaded (L2) before any is used
        for (int i8 = STRIP_HALO; i8 < STRIP_WORDS; i8 += 8) {
            int zr[8];
            uint32_t nzb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i8 + u;
                nzb[u] = nzw[i];
                zr[u] = (base_word + i < p.W && !((nzb[u] >> lane) & 1u)) ? (int)zwin[i * 32 + lane] : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int a = base_word + i8 + u;
                if (a < p.W) {
                    const size_t cb = sum_base + (size_t)a * 32;
                    p.zb[cb + lane] = (uint16_t)(H - zr[u]);
                    if ((nzb[u] >> lane) & 1u) p.e_out[cb + lane] = (uint16_t)H;
                    if (lane == 0) p.ao_out[(size_t)band * p.W + a] = nzb[u];
                }
            }
        }
    }
    if (lane == 0 && key && !aborted) atomicMax(skey, key);
    asm volatile("bar.sync 1, %0;" ::"r"(p.nwarps * 32) : "memory");  // consumers only
    if (tid == 0 && !ld_volatile(&sh[2])) {
        const unsigned long long k = *skey;
        p.band_keys[band] = k;
        if (k) atomicMax(res_key1(result), k);
    }
}

}  // namespace msq
