// msq_team.cuh -- register-resident team engine for small matrices (sm_100a).
//
// One team of TEAM lanes solves one whole matrix (cols <= 1024, rows < 2^PB):
// lane tau owns the 32-column word tau.  32/TEAM matrices share a warp, so the
// batch of cfg2 (4096 x 256^2) runs 4 matrices per warp with no shared memory
// and no barrier -- only warp shuffles and ballots.  Per row and lane:
//
//   m  = the word's 32 cells as bits (u8: 8 multiplies + 3 byte permutes)
//   z  = last-zero row per column, bit-sliced over PB registers:
//        z_p = m ? z_p : bit p of rho           (one LOP3 per plane)
//   E  = { z <= rho - t }  = { height >= t }    (one LOP3 per plane, LSB first)
//   one threshold test at t = best + 1 (P2: one raise per row at most):
//        a segmented warp scan of "ones reaching the word's top" gives the run
//        entering each word; the leftmost window end is the first lane of the
//        team (ballot) with a run >= t ending inside its word.
//
// This is Algorithm 1 (squares.py:84-103, the thresholds coupled as in
// verify.py:115-128) with the location of the final raise (squares.py:93-97):
// the first row whose test succeeds at t, and in it the leftmost window.
// Rows stream straight from HBM with 16-byte loads, D rows in flight per lane
// (register ring), so the kernel is a pure stream: no TMA, no smem.
#pragma once

namespace msq {

// bits of 32 u8 cells (bytes 0/1) given as two 16-byte vectors; any byte
// outside {0,1} sets bits of *bad (the caller reports MSQ_EVALUE)
__device__ __forceinline__ uint32_t team_bits_u8(const uint4 a, const uint4 b, uint32_t& bad) {
    bad |= (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w) & 0xFEFEFEFEu;
    // (x0 + 16 x1) * 0x01020408: byte 3 = the 8 cells of x0,x1 in column order
    const uint32_t p0 = (a.x + (a.y << 4)) * 0x01020408u;
    const uint32_t p1 = (a.z + (a.w << 4)) * 0x01020408u;
    const uint32_t p2 = (b.x + (b.y << 4)) * 0x01020408u;
    const uint32_t p3 = (b.z + (b.w << 4)) * 0x01020408u;
    return __byte_perm(__byte_perm(p0, p1, 0x0073), __byte_perm(p2, p3, 0x0073), 0x5410);
}

// shift schedule of the in-word window test at threshold t: bit j of
// A = E & (E << s0) & ... (6 doubling / closing steps, 0 = no-op) is set iff
// columns j-t+1..j of the word are all eligible; inner = 0 when t > 32
__device__ __forceinline__ void window_schedule(int t, int (&sh)[6], uint32_t& inner) {
    int len = 1;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        sh[k] = 2 * len <= t ? len : 0;
        len = 2 * len <= t ? 2 * len : len;
    }
    sh[5] = t > len && t <= 32 ? t - len : 0;
    inner = t <= 32 ? 0xFFFFFFFFu : 0u;
}

template <bool U8, bool VEC>
struct TeamRow;

// u8, 16-byte aligned rows, cols % 32 == 0: two vector loads per lane
template <>
struct TeamRow<true, true> {
    uint4 a, b;
    __device__ __forceinline__ void load(const uint8_t* row, int tau, bool on, int) {
        if (on) {
            const uint4* q = reinterpret_cast<const uint4*>(row + 32 * tau);
            a = __ldcs(q);
            b = __ldcs(q + 1);
        } else {
            a = b = make_uint4(0, 0, 0, 0);
        }
    }
    __device__ __forceinline__ uint32_t bits(uint32_t& bad) const { return team_bits_u8(a, b, bad); }
};

// u8, any shape: byte loads of the valid columns
template <>
struct TeamRow<true, false> {
    uint32_t w, bad_bytes;
    __device__ __forceinline__ void load(const uint8_t* row, int tau, bool on, int cols) {
        w = 0u;
        bad_bytes = 0u;
        if (on) {
            const int c0 = 32 * tau;
            const int n = min(32, cols - c0);
            for (int j = 0; j < n; ++j) {
                const uint32_t v = row[c0 + j];
                bad_bytes |= v & 0xFEu;
                w |= (v & 1u) << j;
            }
        }
    }
    __device__ __forceinline__ uint32_t bits(uint32_t& bad) const {
        bad |= bad_bytes;
        return w;
    }
};

// bit-packed rows: one word per lane
template <bool VEC>
struct TeamRow<false, VEC> {
    uint32_t w;
    __device__ __forceinline__ void load(const uint8_t* row, int tau, bool on, int) {
        w = on ? __ldcs(reinterpret_cast<const uint32_t*>(row) + tau) : 0u;
    }
    __device__ __forceinline__ uint32_t bits(uint32_t&) const { return w; }
};

template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}
constexpr int LUT_SEL = 0xE2;  // (a=z, b=m, c=r): m ? z : r
constexpr int LUT_LE = 0x8E;   // (a=z, b=le, c=cb): cb ? (~z | le) : (~z & le)

// Row-band mode (one matrix, short but wide enough to want several teams):
// team k runs Algorithm 1 on band k alone and writes the band outputs of
// pass1_kernel (first-zero depth e, bottom run b, never-zeroed masks, band
// key) for the carry scan and the data-free fix-up.
struct TeamBands {
    int nbands, cols_pad;
    long long row_base;
    uint16_t* e_out;
    uint16_t* zb;
    uint32_t* ao_out;
    unsigned long long* band_keys;
};

// TEAM lanes per matrix (power of two >= words), PB bit planes, D rows in
// flight per lane (a multiple of 8).  Rows are counted from 8 (z = r + 8 for
// a zero in 0-based row r, 7 = no zero yet), so within a group of 8 rows the
// low 3 bits of the row number are compile-time constants and the upper ones
// are uniform: the last-zero update is one LOP3 per plane.  rows <= 2^PB - 8.
template <int TEAM, int PB, bool U8, bool VEC, int D, bool BANDS>
__global__ void __launch_bounds__(128) team_kernel(const uint8_t* __restrict__ src, long long mat_stride,
                                                   long long ld_bytes, int rows, int cols, int W, int batch,
                                                   unsigned char* __restrict__ results, const TeamBands tb) {
    static_assert(D % 8 == 0, "groups of 8 rows");
    constexpr int MPW = 32 / TEAM;  // matrices per warp
    constexpr unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const int gwarp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (gwarp * MPW >= batch) return;  // whole warps only: the rest take part in every vote
    const int tau = lane & (TEAM - 1);
    const int tbase = lane & ~(TEAM - 1);
    const unsigned tmask = (TEAM == 32 ? FULL : ((1u << TEAM) - 1u)) << tbase;
    const unsigned below = (1u << lane) - 1u;  // lanes under this one
    const int mat = gwarp * MPW + lane / TEAM;
    const bool mat_ok = mat < batch;
    const bool on = mat_ok && tau < W;
    const uint32_t val = on ? valid_mask(tau, W, cols) : 0u;
    // band mode: "matrix" = band of the one matrix; rows = the largest band height
    // (band mode passes the matrix's row count in mat_stride)
    const int band_r0 = BANDS ? band_row0((int)mat_stride, tb.nbands, mat_ok ? mat : 0) : 0;
    const int my_rows = BANDS ? (mat_ok ? band_row0((int)mat_stride, tb.nbands, mat + 1) - band_r0 : 0) : rows;
    const uint8_t* base = BANDS ? src + (size_t)band_r0 * (size_t)ld_bytes
                                : src + (size_t)(mat_ok ? mat : 0) * (size_t)mat_stride;
    uint32_t fz[PB], nz = val;  // band mode: first-zero rows (bit-planes), never-zeroed columns
#pragma unroll
    for (int q = 0; q < PB; ++q) fz[q] = (7u >> q) & 1u ? FULL : 0u;

    uint32_t z[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) z[q] = (7u >> q) & 1u ? FULL : 0u;  // 7 = no zero yet
    int t = 1;
    int sh[6];
    uint32_t inner;
    window_schedule(t, sh, inner);
    unsigned long long key = 0ull;
    uint32_t bad = 0u;

    TeamRow<U8, VEC> ring[D];
#pragma unroll
    for (int d = 0; d < D; ++d)
        if (d < rows) ring[d].load(base + (size_t)d * ld_bytes, tau, on && d < my_rows, cols);

    for (int r0 = 0; r0 < rows; r0 += D) {
#pragma unroll
        for (int g = 0; g < D / 8; ++g) {
            const uint32_t rg = (uint32_t)(r0 + 8 * g + 8);  // row number of the group (multiple of 8)
            uint32_t rb[PB];
#pragma unroll
            for (int q = 3; q < PB; ++q) rb[q] = 0u - ((rg >> q) & 1u);
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                const int r = r0 + 8 * g + d;
                if (r >= rows) break;  // warp-uniform
                const TeamRow<U8, VEC> cur = ring[8 * g + d];
                if (r + D < rows) ring[8 * g + d].load(base + (size_t)(r + D) * ld_bytes, tau, on && r + D < my_rows, cols);
                const bool live = !BANDS || r < my_rows;  // band mode: rows past this band's end
                const uint32_t m = live ? (cur.bits(bad) & val) : FULL;
                if (BANDS) {  // first zeros: fz = newly ? r + 8 : fz
                    const uint32_t newly = nz & ~m;
#pragma unroll
                    for (int q = 0; q < 3 && q < PB; ++q) fz[q] = (d >> q) & 1 ? (fz[q] | newly) : (fz[q] & ~newly);
#pragma unroll
                    for (int q = 3; q < PB; ++q) fz[q] = lop3<LUT_SEL>(fz[q], ~newly, rb[q]);
                    nz &= m;
                }
                // last-zero rows: z = m ? z : r + 8
#pragma unroll
                for (int q = 0; q < 3 && q < PB; ++q) z[q] = (d >> q) & 1 ? (z[q] | ~m) : (z[q] & m);
#pragma unroll
                for (int q = 3; q < PB; ++q) z[q] = lop3<LUT_SEL>(z[q], m, rb[q]);
                // E = {z <= r + 8 - t} = {height >= t}: LSB-first comparison
                const uint32_t cv = (uint32_t)max(r + 8 - t, 0);
                uint32_t le = FULL;
#pragma unroll
                for (int q = 0; q < PB; ++q) le = lop3<LUT_LE>(z[q], le, 0u - ((cv >> q) & 1u));
                const uint32_t E = live ? (le & val) : 0u;

                // ---- threshold test at t: leftmost window of t eligible columns
                const uint32_t nE = ~E;
                const int pre = nE ? __ffs(nE) - 1 : 32;  // ones from bit 0
                const int suf = __clz(nE);                // ones below the top (32 if full)
                // run entering the word: the suffix of the last non-full word
                // below this one plus 32 per full word in between
                const unsigned nfb = ~__ballot_sync(FULL, nE == 0u) & tmask & below;
                const int h = nfb ? 31 - __clz(nfb) : lane;  // nearest non-full word below
                const int sufb = __shfl_sync(FULL, suf, h);
                const int cin = nfb ? sufb + 32 * (lane - 1 - h) : 32 * tau;
                int endpos = 32;
                if (pre > 0 && t - cin - 1 < pre) endpos = max(t - cin - 1, 0);
                {  // windows inside the word (t <= 32): fixed shift schedule, no branches
                    uint32_t A = E & inner;
#pragma unroll
                    for (int k = 0; k < 6; ++k) A &= A << sh[k];
                    if (A) endpos = min(endpos, __ffs(A) - 1);
                }
                const unsigned bal = __ballot_sync(FULL, endpos < 32) & tmask;
                if (bal) {  // team-uniform: only the team's lanes take part
                    const int endcol = __shfl_sync(tmask, 32 * tau + endpos, __ffs(bal) - 1);
                    key = pack_key(t, BANDS ? tb.row_base + band_r0 + r : r, endcol);
                    ++t;
                    window_schedule(t, sh, inner);
                }
            }
        }
    }
    const unsigned badbal = __ballot_sync(FULL, bad != 0u) & tmask;
    if (BANDS) {
        if (mat_ok && on) {  // this word's 32 columns: bottom runs and leading-ones depths
            const int H = my_rows;
            const size_t cb = (size_t)mat * tb.cols_pad + (size_t)tau * 32;
            uint32_t bw[16], ew[16];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                int zl = 0, fl = 0;
#pragma unroll
                for (int q = 0; q < PB; ++q) {
                    zl |= (int)((z[q] >> j) & 1u) << q;
                    fl |= (int)((fz[q] >> j) & 1u) << q;
                }
                const uint32_t bj = (uint32_t)(H + 7 - zl);               // z = 7: never zeroed -> H
                const uint32_t ej = ((nz >> j) & 1u) ? (uint32_t)H : (uint32_t)(fl - 8);
                if (j & 1) {
                    bw[j >> 1] |= bj << 16;
                    ew[j >> 1] |= ej << 16;
                } else {
                    bw[j >> 1] = bj;
                    ew[j >> 1] = ej;
                }
            }
            uint4* bq = (uint4*)(tb.zb + cb);
            uint4* eq = (uint4*)(tb.e_out + cb);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bq[q] = make_uint4(bw[4 * q], bw[4 * q + 1], bw[4 * q + 2], bw[4 * q + 3]);
                eq[q] = make_uint4(ew[4 * q], ew[4 * q + 1], ew[4 * q + 2], ew[4 * q + 3]);
            }
            tb.ao_out[(size_t)mat * W + tau] = nz;
        }
        if (mat_ok && tau == 0) {
            tb.band_keys[mat] = key;
            if (key) atomicMax(res_key1(results), key);
            if (badbal) atomicOr(res_status(results), 1u);
        }
        return;
    }
    if (mat_ok && tau == 0) {
        unsigned char* res = results + (size_t)mat * 32;
        if (key) *res_key1(res) = key;
        if (badbal) atomicOr(res_status(res), 1u);
    }
}

}  // namespace msq
