// msq_fixup2.cuh -- band-boundary fix-up as a window search (sm_100a).
//
// Squares crossing the top of band k: column j has a virtual
// height c_j + d at depth d while d <= e_j (c = carry-in height above the band
// top, e = leading ones of the band).  A square of side k with its bottom at
// depth d over the columns W = [s, s + k) exists iff d <= e_j and c_j + d >= k
// for every j in W, i.e. iff max(1, k - min_W c) <= d <= min_W e.  So side k
// occurs somewhere in the band iff some window of k columns has
//     min_W e >= 1  and  min_W c + min_W e >= k,
// a property monotone in k (a sub-window of a feasible window is feasible).
// The band's largest crossing side K is found by an exponential + binary
// search on k (no per-depth climb), and its first occurrence in row-major
// order of the bottom-right cell -- what Algorithm 1 reports
// (/root/reference/pkg/src/squarelab/squares.py:93-97) -- is the smallest
// depth d* = min_W max(1, K - min_W c), then the smallest window end among the
// windows feasible at d*.  (A square wholly inside the band can show up here
// too; the band pass reports it with the same key, so the max is unchanged.)
//
// Only columns with e_j >= 1 and c_j + e_j >= T (T = the best side known when
// the CTA starts, ties included) can lie in a window of side >= T, so the CTA
// first collects the maximal runs of such columns of length >= T ("ranges";
// they are rare: none on most bands) and searches only windows starting there.
// Window minima: a warp takes 32 consecutive window starts inside one
// 32-column block; the partial blocks at both ends are warp suffix / prefix
// scans (c and e packed in one word, two 16-bit mins per step) and the whole
// blocks between come from a sparse table of block minima in shared memory.
#pragma once

namespace msq {

constexpr int FIX2_THREADS = 512;
constexpr int FIX2_RMAX = 512;  // ranges kept per band (more: one range over the whole row)

constexpr int FIX2_SMEM_WORDS = 1024;  // bands of <= 32768 columns keep c|e in shared memory

struct Fix2Layout {
    int table, pm, ranges, misc, ce, total, levels;
};
__host__ __device__ inline Fix2Layout fix2_layout(int W) {
    Fix2Layout L{};
    int lv = 1;
    while ((1 << lv) <= W) ++lv;
    L.levels = lv;
    int off = 0;
    L.table = off;
    off += (lv * W * 4 + 15) & ~15;
    L.pm = off;
    off += (W * 4 + 15) & ~15;
    L.ranges = off;
    off += FIX2_RMAX * 8;
    L.misc = off;
    off += 64;
    L.ce = off;
    if (W <= FIX2_SMEM_WORDS) off += W * 32 * 4;
    L.total = off;
    return L;
}

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vminu2(a, b); }

template <bool SMALL>
__device__ __forceinline__ bool fix2_chunk(const uint16_t* __restrict__ cg, const uint16_t* __restrict__ eg,
                                           const uint32_t* ce, const uint32_t* __restrict__ table, int W, int cols,
                                           int B, int k, int x, int y, int lane, uint32_t& mins_out, int& s_out) {
    // window starts s = 32B + lane within [x, y - k]; c/e packed (c | e << 16),
    // from the shared copy `ce` when the band has one
    auto packed = [&](int blk) -> uint32_t {
        const int j = 32 * blk + lane;
        if (blk >= W || j >= cols) return 0u;
        if (ce) return ce[j];
        return (uint32_t)__ldg(cg + j) | ((uint32_t)__ldg(eg + j) << 16);
    };
    const int s = 32 * B + lane;
    const uint32_t v0 = packed(B);
    uint32_t m;
    if (SMALL) {  // k <= 32: the window lies in blocks B, B + 1
        uint32_t lo = v0, hi = packed(B + 1);
        // sliding minimum over k consecutive elements of the 64-element pair (lo, hi)
        uint32_t acc_lo = lo, acc_hi = hi;  // min over [i, i + len)
        int len = 1;
        while (len < k) {
            const int st = min(len, k - len);
            const uint32_t nlo = __shfl_down_sync(0xFFFFFFFFu, acc_lo, st);
            const uint32_t nhi = __shfl_down_sync(0xFFFFFFFFu, acc_hi, st);
            const uint32_t flo = __shfl_sync(0xFFFFFFFFu, acc_hi, (lane + st) & 31);
            acc_lo = vmin2(acc_lo, lane + st < 32 ? nlo : flo);
            acc_hi = vmin2(acc_hi, lane + st < 32 ? nhi : 0u);
            len += st;
        }
        m = acc_lo;
    } else {
        // suffix minimum of block B from s
        uint32_t suf = v0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_down_sync(0xFFFFFFFFu, suf, o);
            if (lane + o < 32) suf = vmin2(suf, u);
        }
        const int B1 = (32 * B + k - 1) >> 5;  // end block of lane 0
        uint32_t p1 = packed(B1), p2 = packed(B1 + 1);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u1 = __shfl_up_sync(0xFFFFFFFFu, p1, o);
            const uint32_t u2 = __shfl_up_sync(0xFFFFFFFFu, p2, o);
            if (lane >= o) {
                p1 = vmin2(p1, u1);
                p2 = vmin2(p2, u2);
            }
        }
        const int off = (k - 1) & 31;
        const int o = (lane + off) & 31;
        const bool second = lane + off >= 32;
        const uint32_t q1 = __shfl_sync(0xFFFFFFFFu, p1, o), q2 = __shfl_sync(0xFFFFFFFFu, p2, o);
        uint32_t pre = second ? q2 : q1;
        // whole blocks between: [B + 1, B1 - 1] (end in B1) or [B + 1, B1] (end in B1 + 1)
        auto query = [&](int a, int b) -> uint32_t {
            if (a > b) return 0xFFFFFFFFu;
            const int n = b - a + 1;
            const int l = 31 - __clz(n);
            return vmin2(table[l * W + a], table[l * W + b - (1 << l) + 1]);
        };
        const uint32_t mid1 = query(B + 1, B1 - 1), mid2 = query(B + 1, min(B1, W - 1));
        m = vmin2(vmin2(suf, pre), second ? mid2 : mid1);
    }
    const int minc = (int)(m & 0xFFFFu), mine = (int)(m >> 16);
    const bool ok = s >= x && s <= y - k && mine >= 1 && minc + mine >= k;
    mins_out = m;
    s_out = s;
    return ok;
}

__global__ void __launch_bounds__(FIX2_THREADS, 1) fixup2_kernel(const FixParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent of the carry scan
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = FIX2_THREADS / 32;
    const int band = p.band_begin + blockIdx.x;
    const int W = p.W, cols = p.cols;
    const int r0 = band_row0(p.rows, p.nbands, band);
    unsigned char* result = p.results;
    const Fix2Layout Lo = fix2_layout(W);
    uint32_t* table = (uint32_t*)(smem + Lo.table);
    uint32_t* pm = (uint32_t*)(smem + Lo.pm);
    int2* ranges = (int2*)(smem + Lo.ranges);
    int* misc = (int*)(smem + Lo.misc);  // [0] T, [1] nranges, [2] overflow, [3] flag, [4] maxlen
    unsigned long long* mkey = (unsigned long long*)(misc + 8);
    const uint16_t* cg = p.carry_in + (size_t)band * p.cols_pad;
    const uint16_t* eg = p.e_in + (size_t)band * p.cols_pad;

    if (tid == 0) {
        int g = (int)(*(volatile unsigned long long*)res_key1(result) >> (2 * KEY_DIM_BITS));
        if (p.share) g = max(g, ld_volatile(res_best(result)));
        misc[0] = max(1, g);
        misc[1] = 0;
        misc[2] = 0;
        misc[4] = 0;
    }
    __syncthreads();
    const int T = misc[0];

    // ---- potential columns (e >= 1, c + e >= T) per 32-column block; block minima.
    // A lane loads 8 columns of c and of e (16 bytes each); 4 lanes make a block;
    // a warp covers 8 blocks per step, 4 steps of loads in flight.
    uint32_t* ce = W <= FIX2_SMEM_WORDS ? (uint32_t*)(smem + Lo.ce) : nullptr;
    {
        const uint4* c4 = (const uint4*)cg;
        const uint4* e4 = (const uint4*)eg;
        const int ngroups = (W + 7) / 8;  // 8 blocks per warp step
        constexpr int U = 4;
        for (int g0 = warp; g0 < ngroups; g0 += U * nwarps) {
            uint4 cv[U], ev[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int g = g0 + u * nwarps;
                const int i = g * 32 + lane;  // uint4 index: columns 8i .. 8i + 7
                cv[u] = ev[u] = make_uint4(0, 0, 0, 0);
                if (g < ngroups && 8 * i < 32 * W) {
                    cv[u] = __ldg(c4 + i);
                    ev[u] = __ldg(e4 + i);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int g = g0 + u * nwarps;
                if (g >= ngroups) break;  // warp-uniform
                const int i = g * 32 + lane;
                const uint32_t cw[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
                const uint32_t ew[4] = {ev[u].x, ev[u].y, ev[u].z, ev[u].w};
                uint32_t bits = 0u, mins = 0xFFFFFFFFu;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int j = 8 * i + q;
                    const uint32_t c = (cw[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
                    const uint32_t e = (ew[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
                    const bool v = j < cols;
                    const uint32_t pk = v ? (c | (e << 16)) : 0u;
                    if (ce && 8 * i < 32 * W) ce[j] = pk;
                    bits |= (v && e >= 1 && (int)(c + e) >= T ? 1u : 0u) << q;
                    mins = vmin2(mins, pk);
                }
                // 4 lanes per block: OR the bytes into a word, min the minima
                uint32_t word = bits << (8 * (lane & 3));
                word |= __shfl_xor_sync(0xFFFFFFFFu, word, 1);
                word |= __shfl_xor_sync(0xFFFFFFFFu, word, 2);
                mins = vmin2(mins, __shfl_xor_sync(0xFFFFFFFFu, mins, 1));
                mins = vmin2(mins, __shfl_xor_sync(0xFFFFFFFFu, mins, 2));
                const int B = i >> 2;
                if ((lane & 3) == 0 && B < W) {
                    pm[B] = word;
                    table[B] = mins;
                }
            }
        }
    }
    __syncthreads();
    // ---- sparse table of block minima (level 0 written above)
    for (int l = 1; l < Lo.levels; ++l) {
        const int h = 1 << (l - 1);
        for (int B = tid; B + 2 * h <= W; B += FIX2_THREADS)
            table[l * W + B] = vmin2(table[(l - 1) * W + B], table[(l - 1) * W + B + h]);
        __syncthreads();
    }
    auto query = [&](int a, int b) -> uint32_t {  // packed minima over blocks [a, b]
        const int l = 31 - __clz(b - a + 1);
        return vmin2(table[l * W + a], table[l * W + b - (1 << l) + 1]);
    };
    // ---- block-level lower bound (shared-threshold mode): whole blocks [a, a + L)
    // with min c + min e = V >= 1 hold a square of side min(32 L, V); the largest
    // L with 32 L <= V (V falls as L grows) by binary lifting, then L and L + 1.
    // Published at once so every band's exact search starts from it.
    if (p.share) {
        if (tid == 0) misc[6] = 0;
        __syncthreads();
        int lb = 0;
        auto val = [&](int a, int L) -> int {
            const uint32_t m = query(a, a + L - 1);
            const int me = (int)(m >> 16);
            return me >= 1 ? (int)(m & 0xFFFFu) + me : -1;
        };
        for (int a = tid; a < W; a += FIX2_THREADS) {
            int L = 0;
            for (int st = 1 << (Lo.levels - 1); st; st >>= 1)
                if (a + L + st <= W && 32 * (L + st) <= val(a, L + st)) L += st;
            if (L) lb = max(lb, 32 * L);
            if (a + L + 1 <= W) lb = max(lb, min(32 * (L + 1), val(a, L + 1)));
        }
        lb = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)max(lb, 0));
        if (lane == 0 && lb > 0) atomicMax(&misc[6], lb);
        __syncthreads();
        if (tid == 0) {
            if (misc[6] > 0) atomicMax(res_best(result), misc[6]);
            misc[0] = max(misc[0], max(misc[6], ld_volatile(res_best(result))));
        }
        __syncthreads();
    }
    const int T2 = misc[0];  // >= T: the threshold the ranges and the search use
    // ---- ranges: column intervals holding every window of side >= T2
    // T2 >= 63: such a window contains Lmin = ceil((T2 - 62) / 32) whole blocks, and
    // every Lmin consecutive whole blocks of it have min c + min e >= T2 ("cores");
    // merged runs of core starts a0..a1 give the range [32 a0 - 31, 32 (a1 + Lmin) + 31).
    // T2 < 63: maximal runs of potential columns (e >= 1, c + e >= T) of length >= T2.
    const bool cores = T2 >= 63;
    const int Lmin = cores ? (T2 - 62 + 31) / 32 : 0;
    if (cores) {  // core starts -> pm (reused as a bitmap over blocks)
        __syncthreads();
        for (int a0 = 32 * warp; a0 < W; a0 += 32 * nwarps) {
            const int a = a0 + lane;
            bool q = false;
            if (a + Lmin <= W) {
                const uint32_t m = query(a, a + Lmin - 1);
                const int mc = (int)(m & 0xFFFFu), me = (int)(m >> 16);
                q = me >= 1 && mc + me >= T2;
            }
            const unsigned bq = __ballot_sync(0xFFFFFFFFu, q);
            if (lane == 0) pm[a0 >> 5] = bq;
        }
        __syncthreads();
    }
    if (warp == 0) {
        const int nbits = cores ? W : 32 * W;  // bitmap length (core starts / columns)
        const int nwords = (nbits + 31) >> 5;
        const int minlen = cores ? 1 : T2;
        auto emit = [&](int st, int en) {  // a run [st, en) of the bitmap
            int x = st, y = en;
            if (cores) {
                x = max(0, 32 * st - 31);
                y = min(cols, 32 * (en - 1 + Lmin) + 31);
            }
            const int slot = atomicAdd(&misc[1], 1);
            if (slot < FIX2_RMAX) ranges[slot] = make_int2(x, y);
            atomicMax(&misc[4], y - x);
        };
        int carry = 0;  // run length at the end of the previous 32 words
        for (int B0 = 0; B0 < nwords; B0 += 32) {
            const int B = B0 + lane;
            const uint32_t m = B < nwords ? pm[B] : 0u;
            const bool full = m == 0xFFFFFFFFu;
            const int pre = full ? 32 : __ffs(~m) - 1, suf = full ? 32 : __clz(~m);
            int v = suf | ((int)full << 16);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xFFFFFFFFu, v, o);
                if (lane >= o && (v >> 16)) v = ((v & 0xFFFF) + (u & 0xFFFF)) | (u & 0x10000);
            }
            const int incl = (v & 0xFFFF) + ((v >> 16) ? carry : 0);  // run at the end of word B
            int rin = __shfl_up_sync(0xFFFFFFFFu, incl, 1);
            if (lane == 0) rin = carry;
            if (B <= nwords && !full) {  // (word nwords, past the end, ends a run reaching the last bit)
                const int R = rin + pre;  // the run entering word B ends at bit pre
                if (R >= minlen && R > 0) emit(32 * B + pre - R, 32 * B + pre);
                if (B < nwords) {  // runs inside the word
                    uint32_t inner = m & ~((pre == 32 ? 0xFFFFFFFFu : ((1u << pre) - 1u)));
                    inner &= suf ? ~(0xFFFFFFFFu << (32 - suf)) : 0xFFFFFFFFu;
                    while (inner) {
                        const int st = __ffs(inner) - 1;
                        const uint32_t rest = ~inner & (0xFFFFFFFFu << st);
                        const int en = rest ? __ffs(rest) - 1 : 32;
                        if (en - st >= minlen) emit(32 * B + st, 32 * B + en);
                        inner &= en == 32 ? 0u : (0xFFFFFFFFu << en);
                    }
                }
            }
            carry = __shfl_sync(0xFFFFFFFFu, incl, 31);  // 0 when the chunk passed the end
        }
        if (lane == 0 && carry >= minlen && carry > 0) emit(32 * nwords - carry, 32 * nwords);
        if (lane == 0 && misc[1] > FIX2_RMAX) {  // too many: one range over the whole row
            ranges[0] = make_int2(0, cols);
            misc[1] = 1;
            misc[4] = cols;
        }
    }
    __syncthreads();
    const int nr = misc[1];
    unsigned long long fixkey = 0ull;
    if (nr > 0) {
        // ---- feasibility of side k over every range (one CTA pass)
        // (also refreshes misc[5] = the grid's best side; stops once a warp found a window)
        volatile int* vflag = misc + 3;
        auto feasible = [&](int k) -> bool {
            if (tid == 0) {
                misc[3] = 0;
                misc[5] = p.share ? max(misc[5], ld_volatile(res_best(result))) : 0;
            }
            __syncthreads();
            bool any = false;
            for (int r = 0; r < nr && !any; ++r) {
                const int2 rg = ranges[r];
                if (rg.y - rg.x < k) continue;
                const int Bs = rg.x >> 5, Be = (rg.y - k) >> 5;
                for (int B = Bs + warp; B <= Be; B += nwarps) {
                    if (*vflag) {
                        any = true;
                        break;
                    }
                    uint32_t mm;
                    int s;
                    const bool ok = k <= 32 ? fix2_chunk<true>(cg, eg, ce, table, W, cols, B, k, rg.x, rg.y, lane, mm, s)
                                            : fix2_chunk<false>(cg, eg, ce, table, W, cols, B, k, rg.x, rg.y, lane, mm, s);
                    if (__any_sync(0xFFFFFFFFu, ok)) {
                        any = true;
                        break;
                    }
                }
            }
            if (any && lane == 0) *vflag = 1;
            __syncthreads();
            return misc[3] != 0;
        };
        if (tid == 0) misc[5] = 0;
        int lo = T2;
        const int U = misc[4];
        bool ok = lo <= U && feasible(lo);
        int hi = -1, step = 1;
        while (ok && hi < 0) {  // exponential search, jumping to a larger side found elsewhere
            const int G = misc[5];
            if (G > lo) {
                if (G > U || !feasible(G)) {  // this band cannot reach the grid's best side
                    ok = false;
                    break;
                }
                lo = G;
                step = 1;
                continue;
            }
            const int kk = lo + step;
            if (kk > U) {
                hi = U + 1;
                break;
            }
            if (feasible(kk)) {
                lo = kk;
                step *= 2;
            } else {
                hi = kk;
            }
        }
        while (ok && hi - lo > 1) {
            const int mid = lo + (hi - lo) / 2;
            if (feasible(mid)) lo = mid;
            else hi = mid;
        }
        if (ok) {
            // ---- first occurrence of side K = lo: smallest depth, then smallest end
            const int K = lo;
            if (tid == 0) *mkey = ~0ull;
            __syncthreads();
            for (int r = 0; r < nr; ++r) {
                const int2 rg = ranges[r];
                if (rg.y - rg.x < K) continue;
                const int Bs = rg.x >> 5, Be = (rg.y - K) >> 5;
                for (int B = Bs + warp; B <= Be; B += nwarps) {
                    uint32_t mm;
                    int s;
                    const bool okw = K <= 32 ? fix2_chunk<true>(cg, eg, ce, table, W, cols, B, K, rg.x, rg.y, lane, mm, s)
                                            : fix2_chunk<false>(cg, eg, ce, table, W, cols, B, K, rg.x, rg.y, lane, mm, s);
                    if (okw) {
                        const int d = max(1, K - (int)(mm & 0xFFFFu));
                        atomicMin(mkey, ((unsigned long long)d << 32) | (unsigned long long)(s + K - 1));
                    }
                }
            }
            __syncthreads();
            if (tid == 0) {
                const unsigned long long mk = *mkey;
                const int d = (int)(mk >> 32), end = (int)(mk & 0xFFFFFFFFu);
                fixkey = pack_key(K, p.row_base + r0 + d - 1, end);
                if (p.share) atomicMax(res_best(result), K);
            }
        }
    }
    if (tid == 0) {
        if (p.fix_keys) p.fix_keys[band] = fixkey;
        if (fixkey) atomicMax(res_keyfix(result), fixkey);
    }
}

}  // namespace msq
