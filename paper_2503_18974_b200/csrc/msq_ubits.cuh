// msq_ubits.cuh -- barrier-free band pass for bit-packed matrices, any threshold (sm_100a).
//
// The bit-packed twin of ustrip_kernel (msq_ustrip.cuh): the same strip argument
// (Algorithm 1, /root/reference/pkg/src/squarelab/squares.py:84-103, run per
// warp column strip, one test per row, ties at sides found elsewhere), the same
// band outputs, but
//   * rows are 32-column words already (LSB = lowest column), 4 per lane: lane l
//     holds window words l, l+32, l+64, l+96 of a 128-word window whose first 16
//     words are the halo -- every window of t <= 16*32 + 1 columns ending in one
//     of the warp's 112 own words lies inside it, and band-local squares are
//     <= H <= USTRIP_BITS_MAXH;
//   * the last-zero row of each column as 9 bit-planes in registers (bands of
//     up to 504 rows): the low log2(R) planes (the row inside an R-row slot)
//     every row, the high planes once per slot for the columns zeroed in it;
//   * first zeros are rare single events in bit-packed data: a column's first
//     zero stores its depth e directly (the columns never zeroed get e = H at
//     the end), instead of a second set of planes.
// Tests: from the row where band-local heights can reach t, a word-level filter
// for t >= 63 (a t-run holds ceil((t-62)/32) consecutive whole words with no
// zero in their last t rows: four ballots make the window's 128-bit map), then
// the exact test (E = {z <= q - t}, runs entering each word, leftmost window
// end in an own word).  No CTA-wide barrier in the row loop; rows arrive
// through the TMA ring of ustrip_kernel.
#pragma once

namespace msq {

constexpr int UB_WORDS = 128;  // window words per warp (4 per lane)
constexpr int UB_HALO = 16;
constexpr int UB_STRIDE = UB_WORDS - UB_HALO;
constexpr int UB_P = 9;        // planes: stored rows q = row + R <= 511
constexpr int UB_MAXWARPS = 19;
__host__ __device__ __forceinline__ int ubits_maxh(int R) { return 512 - R; }

template <int P>
__device__ __forceinline__ uint32_t ub_le(const uint32_t (&z)[P], uint32_t c) {
    uint32_t le = 0xFFFFFFFFu;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const uint32_t cb = 0u - ((c >> p) & 1u);
        le = (cb & (~z[p] | le)) | (~cb & ~z[p] & le);
    }
    return le;
}

template <int R>
__global__ void __launch_bounds__(640, 1) ubits_kernel(const UStripParams p) {
    constexpr int LR = R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3;
    static_assert((1 << LR) == R, "R must be 1, 2, 4 or 8");
    extern __shared__ __align__(128) uint8_t smem[];
    // CTA = (band, column chunk): own words [chunk * cw, chunk * cw + cw); the
    // ring holds words [s0, s1) of each row (the chunk plus the halo on its left)
    const int band = blockIdx.x / p.nchunks, chunk = blockIdx.x % p.nchunks;
    const int cbeg = chunk * p.cw, cend = min(p.W, cbeg + p.cw);
    const int s0 = max(0, cbeg - UB_HALO), s1 = cend;
    const int span_bytes = (s1 - s0) * 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = band_row0(p.rows, p.nbands, band);
    const int H = band_row0(p.rows, p.nbands, band + 1) - r0;
    const int nslots_band = (H + R - 1) / R;
    const int slot_bytes = R * p.row_bytes;
    uint8_t* ring = smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)p.nslots * slot_bytes);
    uint64_t* empty = full + USTRIP_MAXSLOTS;
    int* sh = (int*)(empty + USTRIP_MAXSLOTS);  // [0] start threshold, [1] CTA best
    unsigned long long* skey = (unsigned long long*)(sh + 4);
    unsigned char* result = p.results;

    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the seed / strip pass
    if (p.redo && ld_volatile(p.redo + band) == 0) return;  // done by strip_kernel (unchunked plans)
    if (tid == 0) {
        const int t0 = p.share ? max(1, ld_volatile(res_best(result))) : 1;
        sh[0] = t0;
        sh[1] = t0;
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
            const uint8_t* bsrc = p.src + (size_t)r0 * p.ld + (size_t)s0 * 4;
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
    const int base_word = cbeg + UB_STRIDE * warp - UB_HALO;
    uint32_t VAL[4], off[4];
    bool own[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int a = base_word + 32 * i + lane;
        VAL[i] = (a >= s0 && a < s1) ? valid_mask(a, p.W, p.cols) : 0u;  // ring span only
        own[i] = (32 * i + lane) >= UB_HALO && a < cend;
        off[i] = (uint32_t)((min(max(a, s0), s1 - 1) - s0) * 4);
    }
    uint32_t Z[4][UB_P];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int pl = 0; pl < UB_P; ++pl) Z[i][pl] = (((uint32_t)(R - 1) >> pl) & 1u) ? 0xFFFFFFFFu : 0u;
    uint32_t NZ[4];
    int ZW[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        NZ[i] = own[i] ? VAL[i] : 0u;  // never-zeroed own columns (first zeros are stored)
        ZW[i] = R - 1;
    }
    const size_t sum_base = (size_t)band * p.cols_pad;

    // leftmost end (global column) of a window of t eligible columns ending in one of
    // the warp's own words at the row whose stored form minus t is c, or -1;
    // cz = columns known ineligible (zeroed since the planes were last exact)
    auto exact_end = [&](const uint32_t c, const int t, const uint32_t (&cz)[4]) -> int {
        uint32_t E[4];
        int suf[4], pre[4];
        bool fl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            E[i] = ub_le<UB_P>(Z[i], c) & VAL[i] & ~cz[i];
            fl[i] = E[i] == 0xFFFFFFFFu;
            suf[i] = fl[i] ? 32 : __clz(~E[i]);
            pre[i] = fl[i] ? 32 : __ffs(~E[i]) - 1;
        }
        int rin[4];
        if (t <= 33) {
            int last_prev = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int pv = __shfl_up_sync(0xFFFFFFFFu, suf[i], 1);
                rin[i] = lane ? pv : last_prev;
                last_prev = __shfl_sync(0xFFFFFFFFu, suf[i], 31);
            }
        } else if (t <= 65) {
            // windows span <= 3 words: min(run, 64) from the two previous words
            int p31 = 0, p30 = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int s1 = __shfl_up_sync(0xFFFFFFFFu, suf[i], 1);
                const int s2 = __shfl_up_sync(0xFFFFFFFFu, suf[i], 2);
                const int a = lane >= 1 ? s1 : p31;
                const int bb = lane >= 2 ? s2 : (lane == 1 ? p31 : p30);
                rin[i] = a == 32 ? 32 + bb : a;
                p31 = __shfl_sync(0xFFFFFFFFu, suf[i], 31);
                p30 = __shfl_sync(0xFFFFFFFFu, suf[i], 30);
            }
        } else {
            int carry = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                int v = suf[i] | ((int)fl[i] << 16);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                    if (lane >= o && (v >> 16)) v = ((v & 0xFFFF) + (u & 0xFFFF)) | (u & 0x10000);
                }
                const int tot = (v >> 16) ? (v & 0xFFFF) + carry : (v & 0xFFFF);
                const int pt = __shfl_up_sync(0xFFFFFFFFu, tot, 1);
                rin[i] = lane ? pt : carry;
                carry = __shfl_sync(0xFFFFFFFFu, tot, 31);
            }
        }
        int endb[4];
        unsigned bal[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int e = -1;
            if (pre[i] > 0 && rin[i] + pre[i] >= t) e = max(0, t - 1 - rin[i]);
            else if (t <= 32) {
                const uint32_t ww = windows_in_word(E[i], t);
                if (ww) e = __ffs(ww) - 1 + t - 1;
            }
            endb[i] = own[i] ? e : -1;
            bal[i] = __ballot_sync(0xFFFFFFFFu, endb[i] >= 0);
        }
        if (!(bal[0] | bal[1] | bal[2] | bal[3])) return -1;
        const int i = bal[0] ? 0 : bal[1] ? 1 : bal[2] ? 2 : 3;
        const int l = __ffs(bal[i]) - 1;
        const int ev = __shfl_sync(0xFFFFFFFFu, i == 0 ? endb[0] : i == 1 ? endb[1] : i == 2 ? endb[2] : endb[3], l);
        return 32 * (base_word + 32 * i + l) + ev;
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
        const uint32_t qbase = (uint32_t)(row0 + R);
        uint32_t hm[UB_P];
#pragma unroll
        for (int pl = 0; pl < UB_P; ++pl) hm[pl] = 0u - ((qbase >> pl) & 1u);
        mbar_wait(&full[s], par);
        uint32_t anyz[4] = {0u, 0u, 0u, 0u};  // columns zeroed in this slot so far
        int lastb[4] = {-1, -1, -1, -1};       // last row of this slot with a zero in the word
        auto flush = [&]() {                   // high planes / ZW of the columns zeroed in the slot
#pragma unroll
            for (int i = 0; i < 4; ++i) {
#pragma unroll
                for (int pl = LR; pl < UB_P; ++pl) Z[i][pl] = (Z[i][pl] & ~anyz[i]) | (anyz[i] & hm[pl]);
                if (lastb[i] >= 0) ZW[i] = (int)qbase + lastb[i];
                anyz[i] = 0u;
                lastb[i] = -1;
            }
        };
        // climbing (every row of the last slot raised): test the slot's last row first
        // at t + R - 1 from the state before the slot (see ustrip_kernel)
        bool spec = false;
        if (climbing && nrows == R && R > 1 && row0 + 1 >= t) {
            uint32_t cz[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int b = 0; b < R; ++b) {
                const uint32_t rs = slot_s + (uint32_t)(b * p.row_bytes);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint32_t w;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(rs + off[i]));
                    cz[i] |= ~w & VAL[i];
                }
            }
            const int ts = t + R - 1;
            const int col = exact_end((uint32_t)(row0 + R - t), ts, cz);
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
            const uint32_t rs = slot_s + (uint32_t)(b * p.row_bytes);
            uint32_t zm[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint32_t w;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(rs + off[i]));
                zm[i] = ~w & VAL[i];
            }
            // low planes (the row inside the slot) every row; the high planes and
            // the word's last zero row once per slot for the columns zeroed in it
            // (tests before that mask those columns out: their height is <= R < t,
            // and a test with t <= R flushes first)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
#pragma unroll
                for (int pl = 0; pl < LR; ++pl)
                    Z[i][pl] = ((b >> pl) & 1) ? (Z[i][pl] | zm[i]) : (Z[i][pl] & ~zm[i]);
                anyz[i] |= zm[i];
                lastb[i] = zm[i] ? b : lastb[i];
            }
            // first zeros: e = depth of the row (rare single events)
            const uint32_t n0 = zm[0] & NZ[0], n1 = zm[1] & NZ[1], n2 = zm[2] & NZ[2], n3 = zm[3] & NZ[3];
            if (__any_sync(0xFFFFFFFFu, (n0 | n1 | n2 | n3) != 0u)) {
                const uint32_t nn[4] = {n0, n1, n2, n3};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint32_t x = nn[i];
                    uint16_t* eb = p.e_out + sum_base + (size_t)(base_word + 32 * i + lane) * 32;
                    while (x) {
                        const int j = __ffs(x) - 1;
                        x &= x - 1;
                        eb[j] = (uint16_t)(row0 + b);
                    }
                    NZ[i] &= ~zm[i];
                }
            }
            if (spec) continue;
            const int row = row0 + b;
            bool test = row + 1 >= t;
            if (test && t <= R) flush();  // exact state for the small thresholds
            if (test && t >= 63) {  // word-level filter (warp-uniform)
                const int cq = row + R - t;
                unsigned f[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    f[i] = __ballot_sync(0xFFFFFFFFu, VAL[i] == 0xFFFFFFFFu && anyz[i] == 0u && ZW[i] <= cq);
                const int lmin = (t - 62 + 31) / 32;
                // runs of lmin F words in the 128-bit map f[0..3] (word order)
                unsigned X[4] = {f[0], f[1], f[2], f[3]};
                for (int k = 1; k < lmin; ++k) {  // X &= map >> k (lmin <= 15 < 32)
#pragma unroll
                    for (int i = 0; i < 4; ++i) X[i] &= (f[i] >> k) | (i < 3 ? f[i + 1] << (32 - k) : 0u);
                }
                test = (X[0] | X[1] | X[2] | X[3]) != 0u;
            }
            if (test) {
                const int col = exact_end((uint32_t)(row + R - t), t, anyz);
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
        flush();
        climbing = raises == nrows && nrows == R;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const int g = max(ld_volatile(&sh[1]), gglob);
        if (g > t) t = g;
    }

    // ------------------------------------------------------------ band outputs (own words)
#pragma unroll 1
    for (int wi = UB_HALO; wi < UB_WORDS; ++wi) {
        const int a = base_word + wi;
        if (a >= cend) break;  // warp-uniform
        const int src_lane = wi & 31, qi = wi >> 5;
        uint32_t zv = 0u;
#pragma unroll
        for (int pl = 0; pl < UB_P; ++pl) {
            const uint32_t zsel = qi == 0 ? Z[0][pl] : qi == 1 ? Z[1][pl] : qi == 2 ? Z[2][pl] : Z[3][pl];
            const uint32_t zp = __shfl_sync(0xFFFFFFFFu, zsel, src_lane);
            zv |= ((zp >> lane) & 1u) << pl;
        }
        const uint32_t nsel = qi == 0 ? NZ[0] : qi == 1 ? NZ[1] : qi == 2 ? NZ[2] : NZ[3];
        const uint32_t nz = __shfl_sync(0xFFFFFFFFu, nsel, src_lane);
        const size_t cb = sum_base + (size_t)a * 32;
        p.zb[cb + lane] = (uint16_t)(H - 1 + R - (int)zv);
        if ((nz >> lane) & 1u) p.e_out[cb + lane] = (uint16_t)H;
        if (lane == 0) p.ao_out[(size_t)band * p.W + a] = nz;
    }
    if (lane == 0 && key) atomicMax(skey, key);
    asm volatile("bar.sync 1, %0;" ::"r"(p.nwarps * 32) : "memory");  // consumers only
    if (tid == 0) {
        const unsigned long long k = *skey;
        if (p.nchunks == 1) p.band_keys[band] = k;
        else if (k) atomicMax(p.band_keys + band, k);  // chunked: zeroed by the launch
        if (k) atomicMax(res_key1(result), k);
    }
}

}  // namespace msq
