// msq_cube.cuh -- cube extension: one probe of max_cube's
// binary search (cubes.py:92-125) in two launches.  The depth-frequency
// matrix (depth_freq_update, cubes.py:58-72) of every depth is thresholded at
// k by one pass along depth per (row, col) (a thread walks its column of
// voxels, coalesced across threads); exists_cube_at_depth (cubes.py:75-89) for
// all depths is then one batched maximal-square solve of the [depth, rows,
// cols] stack of thresholded layers (register team engine or band engine).
#pragma once

namespace msq {

__global__ void __launch_bounds__(256) cube_threshold_kernel(const uint8_t* __restrict__ vol, int depth,
                                                             long long layer, int k, uint8_t* __restrict__ out,
                                                             unsigned* __restrict__ bad) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= layer) return;
    int f = 0;
    uint32_t b = 0;
    for (int d = 0; d < depth; ++d) {
        const uint32_t v = vol[(long long)d * layer + c];
        b |= v & 0xFEu;
        f = (v & 1u) ? f + 1 : 0;
        out[(long long)d * layer + c] = f >= k ? 1 : 0;
    }
    if (b) atomicOr(bad, 1u);
}

}  // namespace msq
