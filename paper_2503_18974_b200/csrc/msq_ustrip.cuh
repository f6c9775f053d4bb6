// msq_ustrip.cuh -- barrier-free band pass for u8 matrices (sm_100a).
//
// Same band outputs as pass1_kernel and strip_kernel (band key, leading-ones
// depths e, bottom runs b, all-ones masks) for u8 bands of <= USTRIP_MAXH rows,
// so the carry scan and the data-free fix-up are shared.
//
// Exactness is the strip argument of msq_strip.cuh: g_w(r), the largest side
// of a square whose bottom-right cell lies in row r and in the columns warp w
// owns, satisfies g_w(r) <= g_w(r-1) + 1, so Algorithm 1
// (/root/reference/pkg/src/squarelab/squares.py:84-103) run on the strip alone
// -- one test per row at t = best_w + 1, ties at a side found elsewhere --
// finds the strip's maximum with its first row and leftmost end.  Band-local
// heights never exceed the band height H, so every tested window has
// t <= H + 1 <= 8 * 32 + 1 columns and an 8-word halo on the left holds it.
//
// Layout: warp w owns the 56 words [56w, 56w + 56) and reads the window of 64
// words [56w - 8, 56w + 56): lane l holds window words l and l + 32 (so the
// ballots of the two halves are the window in word order).  Rows arrive through
// a TMA ring of R-row slots (one bulk copy, one full and one empty mbarrier per
// slot); a producer warp refills a slot once every consumer warp released it.
// No CTA-wide barrier in the row loop.
//
// Per row and word (u8 cells read from the slot, 2 x 16 bytes, halves in a
// lane-dependent order so a warp's loads are bank-conflict free):
//   * 32 cells -> 32 bits (four multiplies, three byte permutes); bytes outside
//     {0,1} are OR-accumulated and flag MSQ_EVALUE at the end;
//   * the last-zero row of each column as 8 bit-planes in registers, one LOP3 per
//     plane (rows are counted from R, so inside a slot the low log2(R) plane bits
//     are compile-time constants; a never-zeroed column reads as a zero in row -1);
//   * the first-zero row as 8 more planes while the warp has never-zeroed columns;
//   * from the row where the band-local height can reach t on: for t >= 63 a
//     filter first (a t-run holds ceil((t-62)/32) consecutive whole words with no
//     zero in their last t rows: the word's last zero row, two ballots, shifted
//     ANDs); then eligibility E = {z <= q - t} (8 LOP3), the run entering each
//     word (one shuffle for t <= 33, two for t <= 65, a segmented warp scan
//     above), and the
//     leftmost window end in the warp's own words -> raise.
#pragma once

namespace msq {

constexpr int USTRIP_WORDS = 64;  // window words per warp
constexpr int USTRIP_HALO = 8;
constexpr int USTRIP_STRIDE = USTRIP_WORDS - USTRIP_HALO;
constexpr int USTRIP_P = 8;       // planes: stored rows q = row + R <= 255
constexpr int USTRIP_MAXSLOTS = 8;
constexpr int USTRIP_MAXWARPS = 19;  // 1024 words (32768 columns) + producer <= 640 threads

struct UStripParams {
    const uint8_t* src;
    long long ld;  // bytes per row
    int rows, cols, W, nbands, cols_pad;
    long long row_base;
    int nslots, row_bytes, nwarps;  // row_bytes: ring row stride (the widest chunk + halo)
    int nchunks, cw;                // column chunks per band, own words per chunk
    int share;     // 0 (deterministic plans): every band from t = 1, no shared best side
    uint16_t* zb;  // [nbands][cols_pad] bottom runs (band output)
    uint16_t* e_out;
    uint32_t* ao_out;
    unsigned long long* band_keys;
    unsigned char* results;
    const int* redo;  // optional [nbands] (ubits_kernel): 0 = band done by strip_kernel
};

__host__ __device__ __forceinline__ int ustrip_maxh(int R) { return 256 - R; }

// 16 u8 cells -> 16 bits in the low half of the result (the product trick of bits16)
__device__ __forceinline__ uint32_t us_half(uint4 v) {
    const uint32_t p0 = (v.x + (v.y << 4)) * 0x01020408u;
    const uint32_t p1 = (v.z + (v.w << 4)) * 0x01020408u;
    return __byte_perm(p0, p1, 0x0073);
}

// bit-sliced z <= c for the 32 columns (c >= 0, c < 256), LSB-first
__device__ __forceinline__ uint32_t us_le(const uint32_t (&z)[USTRIP_P], uint32_t c) {
    uint32_t le = 0xFFFFFFFFu;
#pragma unroll
    for (int p = 0; p < USTRIP_P; ++p) {
        const uint32_t cb = 0u - ((c >> p) & 1u);
        le = (cb & (~z[p] | le)) | (~cb & ~z[p] & le);
    }
    return le;
}

template <int R>
__global__ void __launch_bounds__(640, 1) ustrip_kernel(const UStripParams p) {
    constexpr int LR = R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3;
    static_assert((1 << LR) == R, "R must be 1, 2, 4 or 8");
    extern __shared__ __align__(128) uint8_t smem[];
    // CTA = (band, column chunk): own words [chunk * cw, chunk * cw + cw); the
    // ring holds words [s0, s1) of each row (the chunk plus the halo on its left)
    const int band = blockIdx.x / p.nchunks, chunk = blockIdx.x % p.nchunks;
    const int cbeg = chunk * p.cw, cend = min(p.W, cbeg + p.cw);
    const int s0 = max(0, cbeg - USTRIP_HALO), s1 = cend;
    const int span_bytes = (s1 - s0) * 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    const int nslots_band = (H + R - 1) / R;
    const int slot_bytes = R * p.row_bytes;
    uint8_t* ring = smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)p.nslots * slot_bytes);
    uint64_t* empty = full + USTRIP_MAXSLOTS;
    int* sh = (int*)(empty + USTRIP_MAXSLOTS);  // [0] start threshold, [1] CTA best, [2] invalid cell
    unsigned long long* skey = (unsigned long long*)(sh + 4);
    unsigned char* result = p.results;

    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the seed
    if (tid == 0) {
        const int t0 = p.share ? max(1, ld_volatile(res_best(result))) : 1;
        sh[0] = t0;
        sh[1] = t0;
        sh[2] = 0;
        *skey = 0ull;
        for (int s = 0; s < p.nslots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], p.nwarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // ------------------------------------------------------------ producer
    if (warp == p.nwarps) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            const uint8_t* bsrc = p.src + (size_t)r0 * p.ld + (size_t)s0 * 32;
            const bool contiguous = p.ld == (long long)p.row_bytes && span_bytes == p.row_bytes;
            for (int q = 0; q < nslots_band; ++q) {
                const int s = q % p.nslots;
                if (q >= p.nslots) mbar_wait(&empty[s], (uint32_t)((q / p.nslots - 1) & 1));
                const int n = min(R, H - q * R);
                mbar_expect_tx(&full[s], (uint32_t)(n * span_bytes));
                uint8_t* dst = ring + (size_t)s * slot_bytes;
                const uint8_t* srow = bsrc + (size_t)q * R * p.ld;
                if (contiguous) {
                    tma_row(dst, srow, (uint32_t)(n * p.row_bytes), &full[s], pol);
                } else {
                    for (int b = 0; b < n; ++b)
                        tma_row(dst + (size_t)b * p.row_bytes, srow + (size_t)b * p.ld, (uint32_t)span_bytes,
                                &full[s], pol);
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int base_word = cbeg + USTRIP_STRIDE * warp - USTRIP_HALO;
    const int a0 = base_word + lane, a1 = base_word + 32 + lane;  // global words of window words lane, lane+32
    // words outside the ring span (left of the halo, right of the chunk) read as invalid
    const uint32_t VAL0 = (a0 >= s0 && a0 < s1) ? valid_mask(a0, p.W, p.cols) : 0u;
    const uint32_t VAL1 = (a1 >= s0 && a1 < s1) ? valid_mask(a1, p.W, p.cols) : 0u;
    const bool own0 = lane >= USTRIP_HALO && a0 < cend;
    const bool own1 = a1 < cend;
    // smem offsets of the two words' halves; half order swapped on lanes with bit 2
    // set, so 8 consecutive lanes cover all 32 banks
    const uint32_t swap = (lane >> 2) & 1u;
    const uint32_t sel = swap ? 0x1054u : 0x5410u;
    const int c0 = min(max(a0, s0), s1 - 1) - s0, c1 = min(max(a1, s0), s1 - 1) - s0;
    const uint32_t off0 = (uint32_t)(c0 * 32) + 16u * swap, off0b = (uint32_t)(c0 * 32) + 16u * (swap ^ 1u);
    const uint32_t off1 = (uint32_t)(c1 * 32) + 16u * swap, off1b = (uint32_t)(c1 * 32) + 16u * (swap ^ 1u);

    // last-zero rows (stored as row + R; never zeroed = R - 1) and first-zero rows (0 = none)
    uint32_t Z0[USTRIP_P], Z1[USTRIP_P], F0[USTRIP_P], F1[USTRIP_P];
#pragma unroll
    for (int q = 0; q < USTRIP_P; ++q) {
        Z0[q] = Z1[q] = (((uint32_t)(R - 1) >> q) & 1u) ? 0xFFFFFFFFu : 0u;
        F0[q] = F1[q] = 0u;
    }
    uint32_t NZ0 = VAL0, NZ1 = VAL1;  // never-zeroed columns
    int ZW0 = R - 1, ZW1 = R - 1;      // last row (stored form) with a zero in the word
    bool any_nz = true;
    uint32_t bad = 0u;

    // leftmost end (global column) of a window of t eligible columns ending in one of
    // the warp's own words, or -1; E0/E1 = eligibility of window words lane, lane+32
    auto exact_end = [&](const uint32_t E0, const uint32_t E1, const int t) -> int {
        const uint32_t full0 = E0 == 0xFFFFFFFFu, full1 = E1 == 0xFFFFFFFFu;
        const int suf0 = full0 ? 32 : __clz(~E0), suf1 = full1 ? 32 : __clz(~E1);
        const int pre0 = full0 ? 32 : __ffs(~E0) - 1, pre1 = full1 ? 32 : __ffs(~E1) - 1;
        int rin0, rin1;  // eligible run entering each word from the left (capped where exactness allows)
        if (t <= 33) {
            // windows span <= 2 words: min(run, 32) of the previous word suffices
            const int prev0 = __shfl_up_sync(0xFFFFFFFFu, suf0, 1);
            const int last0 = __shfl_sync(0xFFFFFFFFu, suf0, 31);
            const int prev1 = __shfl_up_sync(0xFFFFFFFFu, suf1, 1);
            rin0 = lane ? prev0 : 0;
            rin1 = lane ? prev1 : last0;
        } else if (t <= 65) {
            // windows span <= 3 words: min(run, 64) from the two previous words
            const int s01 = __shfl_up_sync(0xFFFFFFFFu, suf0, 1), s02 = __shfl_up_sync(0xFFFFFFFFu, suf0, 2);
            const int s11 = __shfl_up_sync(0xFFFFFFFFu, suf1, 1), s12 = __shfl_up_sync(0xFFFFFFFFu, suf1, 2);
            const int q31 = __shfl_sync(0xFFFFFFFFu, suf0, 31), q30 = __shfl_sync(0xFFFFFFFFu, suf0, 30);
            const int a0_ = lane >= 1 ? s01 : 0, b0_ = lane >= 2 ? s02 : 0;
            const int a1_ = lane >= 1 ? s11 : q31, b1_ = lane >= 2 ? s12 : (lane == 1 ? q31 : q30);
            rin0 = a0_ == 32 ? 32 + b0_ : a0_;
            rin1 = a1_ == 32 ? 32 + b1_ : a1_;
        } else {
            // segmented inclusive scans: run ending at bit 31 of each word
            int v0 = suf0 | ((int)full0 << 16), v1 = suf1 | ((int)full1 << 16);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u0 = __shfl_up_sync(0xFFFFFFFFu, v0, o);
                const int u1 = __shfl_up_sync(0xFFFFFFFFu, v1, o);
                if (lane >= o) {
                    if (v0 >> 16) v0 = ((v0 & 0xFFFF) + (u0 & 0xFFFF)) | (u0 & 0x10000);
                    if (v1 >> 16) v1 = ((v1 & 0xFFFF) + (u1 & 0xFFFF)) | (u1 & 0x10000);
                }
            }
            const int run31 = __shfl_sync(0xFFFFFFFFu, v0, 31) & 0xFFFF;  // run at the end of word 31
            // the second half's scan continues the first half's run where it is all-eligible
            const int tot1 = (v1 >> 16) ? (v1 & 0xFFFF) + run31 : (v1 & 0xFFFF);
            const int pv0 = __shfl_up_sync(0xFFFFFFFFu, v0 & 0xFFFF, 1);
            const int pt1 = __shfl_up_sync(0xFFFFFFFFu, tot1, 1);
            rin0 = lane ? pv0 : 0;
            rin1 = lane ? pt1 : run31;
        }
        // leftmost window end in each own word (bit index, or -1): the entering run
        // reaches a window end at bit max(0, t-1-rin) if it continues into the word
        // that far (pre > that bit); otherwise windows inside the word (t <= 32)
        int end0 = -1, end1 = -1;
        if (pre0 > 0 && rin0 + pre0 >= t) end0 = max(0, t - 1 - rin0);
        else if (t <= 32) {
            const uint32_t ww = windows_in_word(E0, t);
            if (ww) end0 = __ffs(ww) - 1 + t - 1;
        }
        if (pre1 > 0 && rin1 + pre1 >= t) end1 = max(0, t - 1 - rin1);
        else if (t <= 32) {
            const uint32_t ww = windows_in_word(E1, t);
            if (ww) end1 = __ffs(ww) - 1 + t - 1;
        }
        if (!own0) end0 = -1;
        if (!own1) end1 = -1;
        const unsigned b0 = __ballot_sync(0xFFFFFFFFu, end0 >= 0);
        const unsigned b1 = __ballot_sync(0xFFFFFFFFu, end1 >= 0);
        if (!(b0 | b1)) return -1;
        const int l = b0 ? __ffs(b0) - 1 : __ffs(b1) - 1;
        const int e = __shfl_sync(0xFFFFFFFFu, b0 ? end0 : end1, l);
        return 32 * (base_word + (b0 ? l : 32 + l)) + e;
    };

    int t = sh[0];
    bool climbing = false;  // every row of the previous slot raised
    unsigned long long key = 0ull;
    const uint32_t ring_s = smem_addr(ring);
    int s = 0;
    uint32_t par = 0u;
    for (int q = 0; q < nslots_band; ++q, s = (s + 1 == p.nslots) ? 0 : s + 1, par ^= (s == 0) ? 1u : 0u) {
        const int row0 = q * R;
        const int nrows = min(R, H - row0);
        const uint32_t slot_s = ring_s + (uint32_t)(s * slot_bytes);
        const int gglob = (p.share && (q & 3) == 3) ? ld_volatile(res_best(result)) : 0;
        // high plane masks of this slot's stored rows (row0 + R is a multiple of R)
        const uint32_t qbase = (uint32_t)(row0 + R);
        uint32_t hm[USTRIP_P];
#pragma unroll
        for (int pl = 0; pl < USTRIP_P; ++pl) hm[pl] = 0u - ((qbase >> pl) & 1u);
        mbar_wait(&full[s], par);
        // ---- the slot's rows as bits (bytes validated on the way)
        uint32_t pw0[R], pw1[R];
#pragma unroll
        for (int b = 0; b < R; ++b) {
            pw0[b] = pw1[b] = 0xFFFFFFFFu;
            if (b >= nrows) continue;
            const uint32_t rs = slot_s + (uint32_t)(b * p.row_bytes);
            uint4 v0a, v0b, v1a, v1b;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v0a.x), "=r"(v0a.y), "=r"(v0a.z), "=r"(v0a.w) : "r"(rs + off0));
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v1a.x), "=r"(v1a.y), "=r"(v1a.z), "=r"(v1a.w) : "r"(rs + off1));
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v0b.x), "=r"(v0b.y), "=r"(v0b.z), "=r"(v0b.w) : "r"(rs + off0b));
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v1b.x), "=r"(v1b.y), "=r"(v1b.z), "=r"(v1b.w) : "r"(rs + off1b));
            bad |= v0a.x | v0a.y | v0a.z | v0a.w | v0b.x | v0b.y | v0b.z | v0b.w;
            bad |= v1a.x | v1a.y | v1a.z | v1a.w | v1b.x | v1b.y | v1b.z | v1b.w;
            pw0[b] = __byte_perm(us_half(v0a), us_half(v0b), sel);
            pw1[b] = __byte_perm(us_half(v1a), us_half(v1b), sel);
        }
        // ---- climbing: every row of the last slot raised.  Test the slot's last row
        // first at t + R - 1 from the state before the slot (a column zeroed in the
        // slot is lower than R there): a square of side t + R - 1 ending there
        // contains one of side t + i ending at row i of the slot, so on success
        // every row raises in turn and this window is the last raise.
        bool spec = false;
        if (climbing && nrows == R && R > 1 && row0 + 1 >= t) {
            uint32_t cz0 = 0u, cz1 = 0u;
#pragma unroll
            for (int b = 0; b < R; ++b) {
                cz0 |= ~pw0[b];
                cz1 |= ~pw1[b];
            }
            const int ts = t + R - 1;
            const uint32_t c = (uint32_t)(row0 + R - t);  // q of the last row - ts
            const int col = exact_end(us_le(Z0, c) & VAL0 & ~cz0, us_le(Z1, c) & VAL1 & ~cz1, ts);
            if (col >= 0) {
                key = pack_key(ts, p.row_base + r0 + row0 + R - 1, col);
                if (lane == 0 && p.share) {
                    atomicMax(&sh[1], ts);
                    atomicMax(res_best(result), ts);
                }
                t = ts + 1;
                spec = true;
            }
        }
        int raises = spec ? R : 0;
#pragma unroll
        for (int b = 0; b < R; ++b) {
            if (b >= nrows) break;
            const uint32_t zm0 = ~pw0[b] & VAL0, zm1 = ~pw1[b] & VAL1;
            const int qrow = row0 + R + b;
            ZW0 = zm0 ? qrow : ZW0;
            ZW1 = zm1 ? qrow : ZW1;
            // last zero := this row (q = qbase + b: low LR bits are b)
#pragma unroll
            for (int pl = 0; pl < USTRIP_P; ++pl) {
                const uint32_t m = pl < LR ? (((b >> pl) & 1) ? 0xFFFFFFFFu : 0u) : hm[pl];
                Z0[pl] = (Z0[pl] & ~zm0) | (zm0 & m);
                Z1[pl] = (Z1[pl] & ~zm1) | (zm1 & m);
            }
            if (any_nz) {  // first zeros (warp-uniform)
                const uint32_t n0 = zm0 & NZ0, n1 = zm1 & NZ1;
#pragma unroll
                for (int pl = 0; pl < USTRIP_P; ++pl) {
                    const uint32_t m = pl < LR ? (((b >> pl) & 1) ? 0xFFFFFFFFu : 0u) : hm[pl];
                    F0[pl] |= n0 & m;
                    F1[pl] |= n1 & m;
                }
                NZ0 &= ~zm0;
                NZ1 &= ~zm1;
                any_nz = __any_sync(0xFFFFFFFFu, (NZ0 | NZ1) != 0u);
            }
            if (spec) continue;
            const int row = row0 + b;  // band-local row (0-based)
            bool test = row + 1 >= t;  // warp-uniform: band-local heights can reach t
            if (test && t >= 63) {
                // mode L: a t-run of eligible columns holds Lmin = ceil((t - 62) / 32) >= 1
                // consecutive whole "F" words (no zero in their last t rows); the exact
                // test runs only on rows whose window map has such a run
                const int cq = row + R - t;
                const unsigned f0 = __ballot_sync(0xFFFFFFFFu, VAL0 == 0xFFFFFFFFu && ZW0 <= cq);
                const unsigned f1 = __ballot_sync(0xFFFFFFFFu, VAL1 == 0xFFFFFFFFu && ZW1 <= cq);
                const unsigned long long M = (unsigned long long)f0 | ((unsigned long long)f1 << 32);
                unsigned long long X = M;
                const int lmin = (t - 62 + 31) / 32;
                for (int i = 1; i < lmin && X; ++i) X &= M >> i;
                test = X != 0ull;
            }
            if (test) {
                const uint32_t c = (uint32_t)(row + R - t);  // eligible: z <= q - t
                const int col = exact_end(us_le(Z0, c) & VAL0, us_le(Z1, c) & VAL1, t);
                if (col >= 0) {  // warp-uniform: raise at this row
                    key = pack_key(t, p.row_base + r0 + row, col);
                    if (lane == 0 && p.share) {
                        atomicMax(&sh[1], t);
                        atomicMax(res_best(result), t);
                    }
                    ++t;
                    ++raises;
                }
            }
        }
        climbing = raises == nrows && nrows == R;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // shared best side (ties): the CTA's every slot, the grid's every 8 slots
        const int g = max(ld_volatile(&sh[1]), gglob);
        if (g > t) t = g;
    }

    // ------------------------------------------------------------ band outputs (own words)
    // word by word, lanes = columns: planes of window word i come from lane i & 31
    const int Hs = H;
    const size_t sum_base = (size_t)band * p.cols_pad;
#pragma unroll 1
    for (int i = USTRIP_HALO; i < USTRIP_WORDS; ++i) {
        const int a = base_word + i;
        if (a >= cend) break;  // warp-uniform
        const int src_lane = i & 31;
        const bool second = i >= 32;
        uint32_t zv = 0u, fv = 0u;
#pragma unroll
        for (int pl = 0; pl < USTRIP_P; ++pl) {
            const uint32_t zp = __shfl_sync(0xFFFFFFFFu, second ? Z1[pl] : Z0[pl], src_lane);
            const uint32_t fp = __shfl_sync(0xFFFFFFFFu, second ? F1[pl] : F0[pl], src_lane);
            zv |= ((zp >> lane) & 1u) << pl;
            fv |= ((fp >> lane) & 1u) << pl;
        }
        const uint32_t nz = __shfl_sync(0xFFFFFFFFu, second ? NZ1 : NZ0, src_lane);
        const size_t cb = sum_base + (size_t)a * 32;
        // bottom run = (last row + R) - z; first-zero depth = f - R (never zeroed: H)
        p.zb[cb + lane] = (uint16_t)(Hs - 1 + R - (int)zv);
        p.e_out[cb + lane] = (uint16_t)(((nz >> lane) & 1u) ? Hs : (int)fv - R);
        if (lane == 0) p.ao_out[(size_t)band * p.W + a] = nz;
    }
    if ((bad & 0xFEFEFEFEu) != 0u) atomicOr((unsigned*)&sh[2], 1u);
    if (lane == 0 && key) atomicMax(skey, key);
    asm volatile("bar.sync 1, %0;" ::"r"(p.nwarps * 32) : "memory");  // consumers only
    if (tid == 0) {
        const unsigned long long k = *skey;
        if (p.nchunks == 1) p.band_keys[band] = k;
        else if (k) atomicMax(p.band_keys + band, k);  // chunked: zeroed by the launch
        if (k) atomicMax(res_key1(result), k);
        if (ld_volatile(&sh[2])) atomicOr(res_status(result), 1u);
    }
}

}  // namespace msq
