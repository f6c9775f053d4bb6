// msq_hist.cuh -- histogram maximal rectangle, the reference's
// histogram.py baseline: per-row column heights (build_histograms, :26-35)
// and one monotonic-stack sweep per row (largest_rect_in_histogram, :38-57),
// best over rows (maximal_rectangle, :60-70).
//   hist_heights_kernel: one thread per column walks down the rows (coalesced
//     across threads) and writes the uint16 height of every cell, transposed;
//   hist_rows_kernel: one thread per row runs the stack sweep over its
//     histogram (stack of column indices in global scratch, L1/L2-resident);
//     the first strictly larger rectangle is kept, and rows combine through a
//     64-bit atomicMax of (area, first row) so the earliest row with the
//     largest area wins, exactly as the reference's strict comparisons.
#pragma once

namespace msq {

// heights column-major (h[j * rows + i]) so that the row threads of the sweep
// read neighbouring rows from neighbouring addresses; a 32-row x 256-column
// shared tile turns the column walk's writes into row-contiguous runs
__global__ void __launch_bounds__(256) hist_heights_kernel(const uint8_t* __restrict__ cells, long long ld, int rows,
                                                           int cols, uint16_t* __restrict__ h,
                                                           unsigned* __restrict__ bad) {
    __shared__ uint16_t tile[32][257];
    const int j0 = blockIdx.x * 256;
    const int j = j0 + threadIdx.x;
    uint32_t run = 0, b = 0;
    for (int i0 = 0; i0 < rows; i0 += 32) {
        for (int q = 0; q < 32; ++q) {
            const int i = i0 + q;
            if (j < cols && i < rows) {
                const uint32_t v = cells[(long long)i * ld + j];
                b |= v & 0xFEu;
                run = (v & 1u) ? run + 1 : 0;
            }
            tile[q][threadIdx.x] = (uint16_t)run;
        }
        __syncthreads();
        // thread t writes rows i0 + (t & 31) of columns j0 + (t >> 5) + 8k
        for (int k = 0; k < 32; ++k) {
            const int c = (threadIdx.x >> 5) + 8 * k, i = i0 + (threadIdx.x & 31);
            if (j0 + c < cols && i < rows) h[(long long)(j0 + c) * rows + i] = tile[threadIdx.x & 31][c];
        }
        __syncthreads();
    }
    if (b) atomicOr(bad, 1u);
}

// stacks are column-major too (st[pos * rows + i])
__global__ void __launch_bounds__(128) hist_rows_kernel(const uint16_t* __restrict__ h, int rows, int cols,
                                                        uint16_t* __restrict__ stacks,
                                                        unsigned long long* __restrict__ best_key,
                                                        unsigned long long* __restrict__ row_hw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    auto H = [&](int idx) -> int { return h[(long long)idx * rows + i]; };
    auto ST = [&](int pos) -> uint16_t& { return stacks[(long long)pos * rows + i]; };
    int top = 0;  // stack size
    long long barea = 0;
    int bh = 0, bw = 0;
    int toph = -1;  // height of the bar on top of the stack (cached)
    for (int idx = 0; idx <= cols; ++idx) {
        const int bar = idx < cols ? H(idx) : 0;
        while (top > 0 && toph >= bar) {
            const int hh = toph;
            --top;
            const int left = top > 0 ? ST(top - 1) + 1 : 0;
            toph = top > 0 ? H(ST(top - 1)) : -1;
            const int width = idx - left;
            const long long area = (long long)hh * width;
            if (area > barea) {
                barea = area;
                bh = hh;
                bw = width;
            }
        }
        if (idx < cols) {
            ST(top++) = (uint16_t)idx;
            toph = bar;
        }
    }
    row_hw[i] = ((unsigned long long)bh << 32) | (unsigned)bw;
    if (barea > 0) atomicMax(best_key, ((unsigned long long)barea << 24) | (unsigned long long)(0xFFFFFF - i));
}

}  // namespace msq
