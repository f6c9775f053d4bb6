// msq_ingest.cuh -- text ingest on the GPU: the reference's
// '0'/'1' line format (grid.py:172-206 parse_matrix, frozen by SPEC.md) read
// straight into solver input, u8 cells or LSB-first bit-packed words.
//
// A valid text has every line of the same length, so line i occupies bytes
// [i*(cols+1), i*(cols+1)+cols) followed by '\n' (optional after the last
// line).  Each CTA takes 8192 characters of one line: 16-byte loads of the
// covering aligned span into shared memory, then 32 characters per thread ->
// one output word (bits) or 32 bytes (u8).  Any character outside {'0','1'}
// or a terminator out of place marks the line; the first marked line
// (atomicMin) is where the reference's sequential parse raises, and the host
// re-derives the exact error type and message from that line alone.
#pragma once

namespace msq {

constexpr int INGEST_CHARS = 8192;  // characters of one line per CTA (256 threads x 32)

template <bool BITS>
__global__ void __launch_bounds__(256) ingest_text_kernel(const uint8_t* __restrict__ text, long long nbytes,
                                                          int rows, int cols, uint8_t* __restrict__ out,
                                                          long long ld_bytes, unsigned long long* bad_line) {
    __shared__ __align__(16) uint8_t tile[INGEST_CHARS + 48];
    const int row = blockIdx.y;
    const int c0 = blockIdx.x * INGEST_CHARS;
    const int n = min(INGEST_CHARS, cols - c0);
    if (n <= 0) return;
    const long long start = (long long)row * (cols + 1) + c0;  // first character of this chunk
    const bool last_chunk = c0 + n == cols;
    // span [start, start + n (+1 terminator when it must exist)) clipped to the text
    const long long want = start + n + (last_chunk ? 1 : 0);
    const long long stop = min(want, nbytes);
    const long long a0 = start & ~15ll;
    const int span = (int)(stop > a0 ? stop - a0 : 0);
    for (int o = threadIdx.x * 16; o < span; o += blockDim.x * 16) {
        if (a0 + o + 16 <= nbytes) {
            *(uint4*)(tile + o) = *(const uint4*)(text + a0 + o);
        } else {
            for (int q = 0; q < 16 && a0 + o + q < nbytes; ++q) tile[o + q] = text[a0 + o + q];
        }
    }
    __syncthreads();
    const int off = (int)(start - a0);
    bool bad = stop < start + n;  // text ends inside the line
    const int j0 = threadIdx.x * 32;
    uint32_t word = 0;
    if (j0 < n && !bad) {
        const int m = min(32, n - j0);
        if (m == 32) {
            // 32 characters as 8 words: aligned shared loads funnel-shifted to
            // the line's byte offset; 4 characters validated and packed at once
            const int o = off + j0;
            const uint32_t* tw = (const uint32_t*)(tile + (o & ~3));
            const uint32_t sh = 8u * (uint32_t)(o & 3);
            uint32_t prev = tw[0];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t next = tw[q + 1];
                const uint32_t c4 = __funnelshift_r(prev, next, sh);
                prev = next;
                bad |= ((c4 ^ 0x30303030u) & 0xFEFEFEFEu) != 0u;
                word |= ((((c4 & 0x01010101u) * 0x01020408u) >> 24) & 0xFu) << (4 * q);
            }
        } else {
            for (int q = 0; q < m; ++q) {
                const uint32_t ch = tile[off + j0 + q];
                bad |= (ch & 0xFEu) != 0x30u;
                word |= (ch & 1u) << q;
            }
        }
        if (BITS) {
            ((uint32_t*)(out + (long long)row * ld_bytes))[(c0 + j0) >> 5] = word;
        } else {
            uint8_t* o = out + (long long)row * ld_bytes + c0 + j0;
            for (int q = 0; q < m; ++q) o[q] = (uint8_t)((word >> q) & 1u);
        }
    }
    if (threadIdx.x == 0 && last_chunk && !bad) {
        // terminator: '\n', or the end of the text after the last line
        const long long tpos = start + n;
        if (tpos < nbytes) bad = tile[off + n] != '\n';
        else bad = row != rows - 1;
        if (row == rows - 1 && tpos + 1 < nbytes) bad = true;  // bytes after the last line
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(bad_line, (unsigned long long)row + 1);
}

}  // namespace msq
