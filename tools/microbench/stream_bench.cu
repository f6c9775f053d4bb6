// Pipeline-skeleton calibration for the band kernels (not product code):
// how fast can 148 CTAs x 512 threads stream 512 MiB of rows (8 KiB each)
// through (a) a TMA ring with tile barriers, (b) a TMA ring with per-stage
// empty barriers, (c) plain LDG.128 with register prefetch.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) { while (!mbar_try_wait(bar, parity)) {} }

// (a) tile barriers: rows in tiles of B, refill after the tile's barrier by the last warp
template <int B>
__global__ void __launch_bounds__(512, 1) k_tile(const uint32_t* src, int rows_per_cta, int words, int nstage, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = (uint64_t*)smem;
    uint32_t* ring = (uint32_t*)(smem + 256);
    const int rb = words * 4;
    const uint32_t* base = src + (size_t)blockIdx.x * rows_per_cta * words;
    if (threadIdx.x == 0) { for (int s = 0; s < nstage; ++s) mbar_init(&bars[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    int issued = 0;
    const int issuer = blockDim.x - 32;
    if (threadIdx.x == issuer)
        for (; issued < nstage && issued < rows_per_cta; ++issued) {
            mbar_expect_tx(&bars[issued], rb);
            tma_row(ring + (size_t)issued * words, base + (size_t)issued * words, rb, &bars[issued]);
        }
    uint32_t acc = 0, zw[4] = {0, 0, 0, 0};
    for (int row0 = 0; row0 < rows_per_cta; row0 += B) {
        for (int b = 0; b < B; ++b) {
            const int r = row0 + b, s = r % nstage;
            mbar_wait(&bars[s], (r / nstage) & 1);
            const uint4 v = ((const uint4*)(ring + (size_t)s * words))[threadIdx.x];
            zw[0] = v.x != ~0u ? r : zw[0]; zw[1] = v.y != ~0u ? r : zw[1];
            zw[2] = v.z != ~0u ? r : zw[2]; zw[3] = v.w != ~0u ? r : zw[3];
            acc |= (zw[0] + zw[1] + zw[2] + zw[3] > (unsigned)r) ? 1u : 0u;
        }
        __syncthreads();
        if (threadIdx.x == issuer) {
            const int upto = min(row0 + nstage, rows_per_cta);
            for (; issued < upto; ++issued) {
                const int s = issued % nstage;
                mbar_expect_tx(&bars[s], rb);
                tma_row(ring + (size_t)s * words, base + (size_t)issued * words, rb, &bars[s]);
            }
        }
        __syncthreads();
    }
    if (acc == 12345) out[0] = acc;
}

// (b) producer warp + per-stage empty barriers, no CTA-wide barriers
__global__ void __launch_bounds__(544, 1) k_prod(const uint32_t* src, int rows_per_cta, int words, int nstage, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = (uint64_t*)(smem + 128);
    uint32_t* ring = (uint32_t*)(smem + 256);
    const int rb = words * 4;
    const uint32_t* base = src + (size_t)blockIdx.x * rows_per_cta * words;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstage; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x >= 512) {
        if (threadIdx.x == 512)
            for (int r = 0; r < rows_per_cta; ++r) {
                const int s = r % nstage;
                if (r >= nstage) mbar_wait(&empty[s], ((r / nstage) - 1) & 1);
                mbar_expect_tx(&full[s], rb);
                tma_row(ring + (size_t)s * words, base + (size_t)r * words, rb, &full[s]);
            }
        return;
    }
    uint32_t acc = 0, zw[4] = {0, 0, 0, 0};
    for (int r = 0; r < rows_per_cta; ++r) {
        const int s = r % nstage;
        mbar_wait(&full[s], (r / nstage) & 1);
        const uint4 v = ((const uint4*)(ring + (size_t)s * words))[threadIdx.x];
        zw[0] = v.x != ~0u ? r : zw[0]; zw[1] = v.y != ~0u ? r : zw[1];
        zw[2] = v.z != ~0u ? r : zw[2]; zw[3] = v.w != ~0u ? r : zw[3];
        acc |= (zw[0] + zw[1] + zw[2] + zw[3] > (unsigned)r) ? 1u : 0u;
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345) out[0] = acc;
}

// (c) plain LDG.128, 8 rows in flight per thread
__global__ void __launch_bounds__(512, 1) k_ldg(const uint32_t* src, int rows_per_cta, int words, uint32_t* out) {
    const uint4* base = (const uint4*)(src + (size_t)blockIdx.x * rows_per_cta * words);
    const int w4 = words / 4;
    uint32_t acc = 0, zw[4] = {0, 0, 0, 0};
    for (int r0 = 0; r0 < rows_per_cta; r0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) v[b] = __ldg(base + (size_t)(r0 + b) * w4 + threadIdx.x);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int r = r0 + b;
            zw[0] = v[b].x != ~0u ? r : zw[0]; zw[1] = v[b].y != ~0u ? r : zw[1];
            zw[2] = v[b].z != ~0u ? r : zw[2]; zw[3] = v[b].w != ~0u ? r : zw[3];
            acc |= (zw[0] + zw[1] + zw[2] + zw[3] > (unsigned)r) ? 1u : 0u;
        }
    }
    if (acc == 12345) out[0] = acc;
}

int main() {
    const int words = 2048, rows = 65536, ctas = 148;
    const int rpc = 440;  // rows per CTA (148*440 = 65120)
    const size_t bytes = (size_t)rows * words * 4;
    uint32_t *src, *out;
    cudaMalloc(&src, bytes);
    cudaMalloc(&out, 64);
    cudaMemset(src, 0xFF, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        const double gbs = (double)ctas * rpc * words * 4 / (ms * 1e-3) / 1e9;
        printf("%-28s %8.3f ms  %7.1f GB/s  err=%s\n", name, ms, gbs, cudaGetErrorString(cudaGetLastError()));
    };
    for (int ns : {8, 16, 24}) {
        const int smem = 256 + ns * words * 4;
        cudaFuncSetAttribute(k_tile<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_prod, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        char nm[64];
        snprintf(nm, 64, "tile B=4 nstage=%d", ns);
        run(nm, [&] { k_tile<4><<<ctas, 512, smem>>>(src, rpc, words, ns, out); });
        snprintf(nm, 64, "tile B=1 nstage=%d", ns);
        run(nm, [&] { k_tile<1><<<ctas, 512, smem>>>(src, rpc, words, ns, out); });
        snprintf(nm, 64, "producer nstage=%d", ns);
        run(nm, [&] { k_prod<<<ctas, 544, smem>>>(src, rpc, words, ns, out); });
    }
    run("ldg 8 rows in flight", [&] { k_ldg<<<ctas, 512>>>(src, rpc, words, out); });
    return 0;
}
