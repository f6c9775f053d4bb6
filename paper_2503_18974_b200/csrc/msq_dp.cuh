// msq_dp.cuh -- the three-way-min DP (Eq. 1 of the paper) on the GPU, batched:
// the independent second solver of the GPU verification campaigns
// (verify.py here; the reference runs dp_full beside freq_square in
// verify.py:32-37).  Restates dp_full (squares.py:142-171): dp = min(up, left,
// diag) + 1 on ones, border cells 1, best updated on a strict improvement, so
// the reported cell is the first maximal bottom-right in row-major order.
// One thread per matrix, one row of dp values in local memory (cols <= 256):
// meant for the campaign sizes (<= 64 x 64), not for throughput.
#pragma once

namespace msq {

constexpr int DP_MAXCOLS = 256;

__global__ void __launch_bounds__(128) dp_batch_kernel(const uint8_t* __restrict__ src, int batch, int rows,
                                                       int cols, unsigned char* __restrict__ results) {
    const int mat = blockIdx.x * blockDim.x + threadIdx.x;
    if (mat >= batch) return;
    const uint8_t* m = src + (size_t)mat * rows * cols;
    uint16_t prev[DP_MAXCOLS];
    int best = 0, bi = -1, bj = -1;
    uint32_t bad = 0;
    for (int i = 0; i < rows; ++i) {
        int diag = 0, left = 0;
        for (int j = 0; j < cols; ++j) {
            const uint32_t c = m[(size_t)i * cols + j];
            bad |= c & 0xFEu;
            const int up = i ? prev[j] : 0;
            int v = 0;
            if (c & 1u) v = (i == 0 || j == 0) ? 1 : min(min(up, left), diag) + 1;
            diag = up;
            left = v;
            prev[j] = (uint16_t)v;
            if (v > best) {
                best = v;
                bi = i;
                bj = j;
            }
        }
    }
    unsigned char* res = results + (size_t)mat * 32;
    *res_key1(res) = best ? pack_key(best, bi, bj) : 0ull;
    if (bad) *res_status(res) = 1u;
}

}  // namespace msq
