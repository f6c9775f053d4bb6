// msq_hist.cuh -- histogram maximal rectangle, the reference's
// histogram.py baseline: per-row column heights (build_histograms, :26-35)
// and one monotonic-stack sweep per row (largest_rect_in_histogram, :38-57),
// best over rows (maximal_rectangle, :60-70).
//   hist_heights_kernel: one thread per column walks down the rows (coalesced
//     across threads) and writes the uint16 height of every cell;
//   hist_rows_kernel: one thread per row runs the stack sweep over its
//     histogram (stack of column indices in global scratch, L1/L2-resident);
//     the first strictly larger rectangle is kept, and rows combine through a
//     64-bit atomicMax of (area, first row) so the earliest row with the
//     largest area wins, exactly as the reference's strict comparisons.
#pragma once

namespace msq {

__global__ void __launch_bounds__(256) hist_heights_kernel(const uint8_t* __restrict__ cells, long long ld, int rows,
                                                           int cols, uint16_t* __restrict__ h,
                                                           unsigned* __restrict__ bad) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    uint32_t run = 0, b = 0;
    for (int i = 0; i < rows; ++i) {
        const uint32_t v = cells[(long long)i * ld + j];
        b |= v & 0xFEu;
        run = (v & 1u) ? run + 1 : 0;
        h[(long long)i * cols + j] = (uint16_t)run;
    }
    if (b) atomicOr(bad, 1u);
}

__global__ void __launch_bounds__(128) hist_rows_kernel(const uint16_t* __restrict__ h, int rows, int cols,
                                                        uint16_t* __restrict__ stacks,
                                                        unsigned long long* __restrict__ best_key,
                                                        unsigned long long* __restrict__ row_hw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const uint16_t* hr = h + (long long)i * cols;
    uint16_t* st = stacks + (long long)i * cols;
    int top = 0;  // stack size
    long long barea = 0;
    int bh = 0, bw = 0;
    for (int idx = 0; idx <= cols; ++idx) {
        const int bar = idx < cols ? hr[idx] : 0;
        while (top > 0 && hr[st[top - 1]] >= bar) {
            const int hh = hr[st[--top]];
            const int left = top > 0 ? st[top - 1] + 1 : 0;
            const int width = idx - left;
            const long long area = (long long)hh * width;
            if (area > barea) {
                barea = area;
                bh = hh;
                bw = width;
            }
        }
        if (idx < cols) st[top++] = (uint16_t)idx;
    }
    row_hw[i] = ((unsigned long long)bh << 32) | (unsigned)bw;
    if (barea > 0) atomicMax(best_key, ((unsigned long long)barea << 24) | (unsigned long long)(0xFFFFFF - i));
}

}  // namespace msq
