// msq_rowdp.cuh -- the DP baselines and the traced mode on the GPU (sm_100a).
//
// Reference: dp_full / dp_rows (/root/reference/pkg/src/squarelab/squares.py
// :142-171, :174-200) -- dp = min(up, left, diag) + 1 on ones, out-of-range
// neighbours 0, best on a strict improvement (so the reported cell is the first
// maximal bottom-right in row-major order) -- and the per-row snapshots of
// freq_square_traced (squares.py:33-45, :104-113, :129-139): after row i the
// heights ("freq") and found_max_width.
//
// Row-parallel form of the recurrence.  A k-square ends at (i, j) iff column j
// has a one-run of height >= k ending in row i, row i has a one-run of length
// >= k ending in column j, and a (k-1)-square ends at (i-1, j-1).  So
//     dp[i][j] = cell ? min(h[i][j], w[i][j], dp[i-1][j-1] + 1) : 0
// with h the column heights (the reference's freq) and w the row runs: the only
// dependence inside a row is the row run, a prefix scan.  found_max_width after
// row i is max(dp[0..i][*]) (Algorithm 1 finds every new maximum in the row
// where it first occurs).
//
// Layout: one warp per column strip of 32*CPT columns (u8: 16 columns per lane,
// one 16-byte load; bits: one 32-column word per lane).  A warp walks all rows
// of its strip; lane state = the CPT heights and the previous row's dp values.
// The row run entering a lane is a warp scan of (all-ones, trailing run); the
// run and dp value at the strip's last column are published per row to the
// next strip through global memory (strip s waits for strip s-1: a wavefront,
// strips taken in order through an atomic ticket so a waited-on strip is always
// resident).  Not a throughput path: the baselines and the traced mode only.
#pragma once

namespace msq {

constexpr int ROWDP_WARPS = 4;  // warps (independent strips) per CTA

// 64-bit result key of the DP kernels: side << 40 | (2^40 - 1 - linear index
// of the bottom-right cell) -- max = largest side, then first in row-major order.
// rows * cols < 2^40 (any matrix that fits in device memory).
constexpr int ROWDP_LIN_BITS = 40;
__host__ __device__ __forceinline__ unsigned long long rowdp_key(long long side, long long lin) {
    return side <= 0 ? 0ull
                     : ((unsigned long long)side << ROWDP_LIN_BITS) |
                           (((1ull << ROWDP_LIN_BITS) - 1ull) - (unsigned long long)lin);
}

struct RowDpParams {
    const uint8_t* src;     // u8 cells (ld bytes per row) or packed words (ld words per row)
    long long ld;
    long long rows, cols;
    int nstrips;
    int vec;                       // u8: rows are 16-byte aligned and cols % 16 == 0
    unsigned long long* bnd;       // [nstrips][rows] (w_last + 1) << 32 | (dp_last + 1); zeroed
    unsigned int* ticket;          // strip ticket counter; zeroed
    unsigned long long* key;       // result key (atomicMax)
    unsigned int* status;          // bit 0: invalid u8 cell
    uint32_t* heights;             // optional [rows][cols] heights after each row (traced)
    int* rowmax;                   // optional [rows] max dp per row (traced); zeroed
};

template <int CPT>
__device__ __forceinline__ void rowdp_load_u8(const RowDpParams& p, long long i, long long c0, uint32_t (&c)[CPT],
                                              uint32_t& bad) {
    const uint8_t* row = p.src + i * p.ld;
    if (p.vec && c0 + CPT <= p.cols) {
        const uint4 v = __ldcs((const uint4*)(row + c0));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < CPT; ++k) c[k] = (w[k >> 2] >> (8 * (k & 3))) & 0xFFu;
    } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) c[k] = (c0 + k < p.cols) ? (uint32_t)row[c0 + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        bad |= c[k] & 0xFEu;
        c[k] &= 1u;
    }
}

template <int CPT>
__device__ __forceinline__ void rowdp_load_bits(const RowDpParams& p, long long i, long long c0, uint32_t (&c)[CPT],
                                                uint32_t&) {
    const uint32_t* row = (const uint32_t*)p.src + i * p.ld;
    const uint32_t w = c0 < p.cols ? row[c0 >> 5] : 0u;
#pragma unroll
    for (int k = 0; k < CPT; ++k) c[k] = (c0 + k < p.cols) ? (w >> k) & 1u : 0u;
}

template <bool BITS>
__global__ void __launch_bounds__(32 * ROWDP_WARPS) rowdp_kernel(const RowDpParams p) {
    constexpr int CPT = BITS ? 32 : 16;
    const int lane = threadIdx.x & 31;
    int s = 0;
    if (lane == 0) s = (int)atomicAdd(p.ticket, 1u);
    s = __shfl_sync(0xFFFFFFFFu, s, 0);
    if (s >= p.nstrips) return;
    const long long c0 = (long long)s * 32 * CPT + (long long)lane * CPT;
    uint32_t h[CPT], dpp[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) h[k] = dpp[k] = 0u;
    uint32_t bad = 0u;
    unsigned long long best = 0ull;
    int bestv = 0;
    const unsigned long long* in_bnd = s ? p.bnd + (size_t)(s - 1) * p.rows : nullptr;
    unsigned long long* out_bnd = (s + 1 < p.nstrips) ? p.bnd + (size_t)s * p.rows : nullptr;
    unsigned long long cache = 0ull;  // lane k < 8 holds the boundary entry of row base + k
    long long cache_base = -8;
    uint32_t dp_left_prev = 0u;  // dp of the column left of the strip, previous row

    for (long long i = 0; i < p.rows; ++i) {
        uint32_t c[CPT];
        if constexpr (BITS) rowdp_load_bits<CPT>(p, i, c0, c, bad);
        else rowdp_load_u8<CPT>(p, i, c0, c, bad);
        // boundary from the strip on the left (row run at its last column in this
        // row, its dp there in this row): 8 rows per poll
        uint32_t w_in = 0u, dp_in = 0u;
        if (in_bnd) {
            if (i >= cache_base + 8) {
                cache_base = i;
                const long long n = min(8ll, p.rows - i);
                for (;;) {
                    if (lane < n) cache = *(volatile const unsigned long long*)(in_bnd + i + lane);
                    if (__all_sync(0xFFFFFFFFu, lane >= n || cache != 0ull)) break;
                    __nanosleep(64);
                }
            }
            const unsigned long long e = __shfl_sync(0xFFFFFFFFu, cache, (int)(i - cache_base));
            w_in = (uint32_t)(e >> 32) - 1u;
            dp_in = (uint32_t)e - 1u;
        }
        // lane summary: trailing run, all ones
        uint32_t suf = 0u;
#pragma unroll
        for (int k = 0; k < CPT; ++k) suf = c[k] ? suf + 1u : 0u;
        uint32_t all = suf == (uint32_t)CPT ? 1u : 0u;
        // inclusive warp scan of (all, run): left (aL, sL) then right (aR, sR) ->
        // (aL & aR, aR ? sL + sR : sR)
        uint32_t a = all, r = suf;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t ao = __shfl_up_sync(0xFFFFFFFFu, a, d);
            const uint32_t ro = __shfl_up_sync(0xFFFFFFFFu, r, d);
            if (lane >= d) {
                if (a) r += ro;
                a &= ao;
            }
        }
        uint32_t ae = __shfl_up_sync(0xFFFFFFFFu, a, 1), re = __shfl_up_sync(0xFFFFFFFFu, r, 1);
        if (lane == 0) {
            ae = 1u;
            re = 0u;
        }
        uint32_t w = ae ? w_in + re : re;  // run entering the lane's first column
        // dp of the column left of the lane's first one, previous row
        uint32_t diag = __shfl_up_sync(0xFFFFFFFFu, dpp[CPT - 1], 1);
        if (lane == 0) diag = dp_left_prev;
        uint32_t rm = 0u;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            w = c[k] ? w + 1u : 0u;
            h[k] = c[k] ? h[k] + 1u : 0u;
            const uint32_t up_left = dpp[k];
            const uint32_t v = c[k] ? min(min(h[k], w), diag + 1u) : 0u;
            diag = up_left;
            dpp[k] = v;
            rm = max(rm, v);
            if ((int)v > bestv) {
                bestv = (int)v;
                best = rowdp_key(v, i * p.cols + c0 + k);
            }
        }
        dp_left_prev = dp_in;
        if (out_bnd && lane == 31)
            *(volatile unsigned long long*)(out_bnd + i) =
                ((unsigned long long)(w + 1u) << 32) | (unsigned long long)(dpp[CPT - 1] + 1u);
        if (p.heights) {
            uint32_t* hr = p.heights + i * p.cols + c0;
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                if (c0 + k < p.cols) hr[k] = h[k];
        }
        if (p.rowmax) {
            const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, rm);
            if (lane == 0 && m) atomicMax(p.rowmax + i, (int)m);
        }
    }
    // warp max of the keys, one atomic per strip
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, best, d);
        best = o > best ? o : best;
    }
    const uint32_t anybad = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (lane == 0) {
        if (best) atomicMax(p.key, best);
        if (anybad) atomicOr(p.status, 1u);
    }
}

// brute_force_square (squares.py:203-249) restated per anchor: grow the square
// at (top, left) while the new bottom row and the new right column are ones,
// counting raw cell reads exactly as the reference does (its cells_visited).
// One thread per anchor; small inputs only (the reference caps rows*cols at
// ORACLE_CELL_CAP = 10^4, squares.py:17).
__global__ void __launch_bounds__(256) brute_kernel(const uint8_t* __restrict__ src, long long ld, int rows, int cols,
                                                    unsigned long long* key, unsigned long long* visited,
                                                    unsigned int* status) {
    const long long a = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= (long long)rows * cols) return;
    const int top = (int)(a / cols), left = (int)(a % cols);
    const int limit = min(rows - top, cols - left);
    unsigned long long v = 0ull;
    int k = 0;
    uint32_t bad = 0u;
    while (k < limit) {
        bool ok = true;
        for (int j = left; j <= left + k; ++j) {  // new bottom row
            ++v;
            const uint32_t c = src[(long long)(top + k) * ld + j];
            bad |= c & 0xFEu;
            if (!(c & 1u)) {
                ok = false;
                break;
            }
        }
        if (ok) {
            for (int i = top; i < top + k; ++i) {  // new right column
                ++v;
                const uint32_t c = src[(long long)i * ld + left + k];
                bad |= c & 0xFEu;
                if (!(c & 1u)) {
                    ok = false;
                    break;
                }
            }
        }
        if (!ok) break;
        ++k;
    }
    // anchors in row-major order: the first anchor of the largest k wins (the
    // reference's strict `k > best`), i.e. the smallest linear index
    atomicAdd(visited, v);
    if (k) atomicMax(key, rowdp_key(k, a));
    if (bad) atomicOr(status, 1u);
}

}  // namespace msq
