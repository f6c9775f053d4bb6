// msq.cu -- C ABI (include/msq.h) over the sm_100a kernels in msq_engine.cuh.
//
// Replaces the reference's Python hot loop, squares.py:68-114 (_freq_core),
// behind the same call shape freq_square(m, audit=None) -> SquareResult
// (squares.py:117-126); the Python mirror lives in ../squares.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "msq.h"
#include "msq_engine.cuh"
#include "msq_team.cuh"
#include "msq_strip.cuh"
#include "msq_ustrip.cuh"
#include "msq_ubits.cuh"
#include "msq_fixup2.cuh"
#include "msq_dp.cuh"
#include "msq_ingest.cuh"
#include "msq_cube.cuh"
#include "msq_hist.cuh"
#include "msq_rowdp.cuh"
#include "msq_sieve.cuh"

namespace {

constexpr int kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA (sm_100)
constexpr int kModeLThreshold = 96;  // >= 63 (see msq_engine.cuh)
constexpr int kMaxWords = 2048;   // 65536 columns

thread_local int32_t g_last_launches = 0;
thread_local char g_last_err[256] = "";
unsigned long long* g_prof = nullptr;  // debug: per-unit phase counters

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }
inline long long round_up(long long a, long long b) { return ceil_div(a, b) * b; }

int num_sms() {
    static int sms[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev < 64 && sms[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        sms[dev] = v;
    }
    return dev < 64 ? sms[dev] : 148;
}

struct WsLayout {
    size_t band_keys, fix_keys, zb, e, ao, carry, zw, redo, total;
};

// ---- strip pass (msq_strip.cuh): bit-packed single matrices, several bands
int strip_warps(const msq_plan* p) { return (int)ceil_div(p->words, msq::STRIP_STRIDE); }
int strip_fixed_smem(const msq_plan* p) {  // barriers, flags, never-zeroed masks
    return 2 * msq::STRIP_MAXSLOTS * 8 + 32 + strip_warps(p) * msq::STRIP_WORDS * 4;
}
int strip_slots(const msq_plan* p) {
    const long long slot = (long long)msq::STRIP_TR * p->row_stage_bytes;
    return (int)std::min<long long>(msq::STRIP_MAXSLOTS, (kSmemMax - 256 - strip_fixed_smem(p)) / slot);
}
int strip_smem(const msq_plan* p) {
    return strip_slots(p) * msq::STRIP_TR * p->row_stage_bytes + strip_fixed_smem(p);
}
bool strip_applies(const msq_plan* p) {
    if (p->flags & MSQ_PLAN_NO_STRIP) return false;  // experiments
    if (p->col_chunks > 1) return false;              // chunked plans: ubits_kernel
    const long long ld_bytes = p->ld * 4;
    return p->fmt == MSQ_FMT_BITS && p->batch == 1 && p->nbands > 1 && !p->deterministic &&
           p->words >= 2 * msq::STRIP_WORDS && p->words % 4 == 0 && p->row_stage_bytes % 16 == 0 &&
           ld_bytes % 16 == 0 && (strip_warps(p) + 1) * 32 <= 640 && strip_slots(p) >= 2 &&
           ceil_div(p->rows, p->nbands) <= 65535;
}

// ---- u8 / bit-packed strip passes (msq_ustrip.cuh, msq_ubits.cuh): single
// matrices, several bands; a band may be split into column chunks (one CTA each)
// so short bands still fill the GPU with few bands
struct StripGeom {
    int chunks, cw, warps, row_bytes;  // chunks per band, own words per chunk, warps, ring row bytes
};
StripGeom strip_geom(const msq_plan* p, int stride, int halo, int bpw) {
    StripGeom g{};
    g.chunks = std::max(1, p->col_chunks);
    g.cw = (int)round_up(ceil_div(p->words, g.chunks), 4);
    g.warps = (int)ceil_div(g.cw, stride);
    g.row_bytes = (int)std::min<long long>(p->words, (long long)g.cw + halo) * bpw;
    return g;
}
StripGeom ustrip_geom(const msq_plan* p) { return strip_geom(p, msq::USTRIP_STRIDE, msq::USTRIP_HALO, 32); }
StripGeom ubits_geom(const msq_plan* p) { return strip_geom(p, msq::UB_STRIDE, msq::UB_HALO, 4); }
int ustrip_warps(const msq_plan* p) { return ustrip_geom(p).warps; }
int ustrip_fixed_smem() { return 2 * msq::USTRIP_MAXSLOTS * 8 + 64; }
// rows per ring slot: the largest of 8/4/2/1 that leaves >= 3 slots
int ustrip_rows_per_slot(int row_bytes) {
    const long long avail = kSmemMax - 256 - ustrip_fixed_smem();
    for (int R = 8; R >= 1; R /= 2)
        if (avail / ((long long)R * row_bytes) >= 3) return R;
    return 0;
}
int ustrip_slots(int row_bytes) {
    const int R = ustrip_rows_per_slot(row_bytes);
    if (!R) return 0;
    const long long avail = kSmemMax - 256 - ustrip_fixed_smem();
    return (int)std::min<long long>(msq::USTRIP_MAXSLOTS, avail / ((long long)R * row_bytes));
}
int ustrip_smem(int row_bytes) {
    return ustrip_slots(row_bytes) * ustrip_rows_per_slot(row_bytes) * row_bytes + ustrip_fixed_smem();
}
// ---- bit-packed strip pass (msq_ubits.cuh): any threshold, bands <= 504 rows
int ubits_warps(const msq_plan* p) { return ubits_geom(p).warps; }
bool ubits_applies(const msq_plan* p) {
    if (p->flags & MSQ_PLAN_PASS1) return false;  // experiments
    const int R = ustrip_rows_per_slot(ubits_geom(p).row_bytes);
    return p->fmt == MSQ_FMT_BITS && p->batch == 1 && p->nbands > 1 && R > 0 && p->words % 4 == 0 &&
           (p->ld * 4) % 16 == 0 && p->row_stage_bytes == p->words * 4 && ubits_warps(p) <= msq::UB_MAXWARPS &&
           p->words >= 32 && ceil_div(p->rows, p->nbands) <= msq::ubits_maxh(R);
}

bool ustrip_applies(const msq_plan* p) {
    if (p->flags & MSQ_PLAN_NO_STRIP) return false;  // experiments
    const int R = ustrip_rows_per_slot(ustrip_geom(p).row_bytes);
    return p->fmt == MSQ_FMT_U8 && p->batch == 1 && p->nbands > 1 && R > 0 && p->cols % 32 == 0 &&
           p->ld % 16 == 0 && p->row_stage_bytes == p->cols && ustrip_warps(p) <= msq::USTRIP_MAXWARPS &&
           p->words >= msq::USTRIP_WORDS && ceil_div(p->rows, p->nbands) <= msq::ustrip_maxh(R);
}

WsLayout ws_layout(const msq_plan* p) {
    WsLayout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += round_up((long long)bytes, 256);
        return o;
    };
    const size_t nb = (size_t)p->nbands;
    const size_t cols_pad = (size_t)p->words * 32;
    L.band_keys = take((size_t)p->batch * nb * 8);
    L.fix_keys = take(nb * 8);
    const bool summaries = p->batch == 1;
    // per unit: last-zero rows during pass 1 (global scratch), bottom runs after
    L.zb = take((size_t)p->batch * nb * cols_pad * 2);
    L.e = take(summaries ? nb * cols_pad * 2 : 0);
    L.ao = take(summaries ? nb * (size_t)p->words * 4 : 0);
    L.carry = take(summaries ? nb * cols_pad * 2 : 0);
    const bool strip = strip_applies(p);
    L.zw = take(strip ? nb * (size_t)strip_warps(p) * msq::STRIP_WORDS * 32 * 2 : 0);
    L.redo = take(strip ? nb * 4 : 0);
    L.total = off;
    return L;
}

// ------------------------------------------------------------- dispatch
int zplanes_for(const msq_plan* pl) {
    if (pl->fmt != MSQ_FMT_U8) return 0;  // bits inputs keep last-zero rows in global scratch
    const long long hmax = ceil_div(pl->rows, pl->nbands);
    int P = 1;
    while ((1ll << P) <= hmax) ++P;
    return P;
}

// CTA-team plans reserve smem for the optional phase-cycle counters
bool cta_plan(const msq_plan* pl) { return pl->teams_per_cta == 1 && pl->team == pl->threads; }


template <class K>
cudaError_t set_smem_attr(K kern, bool* done) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
        if (e != cudaSuccess) return e;
        done[dev] = true;
    }
    return cudaSuccess;
}

template <int WPT, bool U8, bool TMA, bool SUB>
cudaError_t launch_pass1_t(const msq_plan* pl, const msq::Pass1Params& prm, cudaStream_t st) {
    auto kern = msq::pass1_kernel<WPT, U8, TMA, SUB>;
    static bool attr_set[64] = {false};
    cudaError_t e = set_smem_attr(kern, attr_set);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};  // programmatic dependent of the seed / strip pass
    cfg.gridDim = dim3((unsigned)pl->grid);
    cfg.blockDim = dim3((unsigned)pl->threads);
    cfg.dynamicSmemBytes = (size_t)pl->smem_pass1;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, kern, prm);
    if (e2 != cudaSuccess) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        snprintf(g_last_err, sizeof(g_last_err), "%s (pass1: regs %d, maxThreads %d, localBytes %zu, block %d, smem %d)",
                 cudaGetErrorString(e2), fa.numRegs, fa.maxThreadsPerBlock, fa.localSizeBytes, pl->threads,
                 pl->smem_pass1);
        return e2;
    }
    return cudaSuccess;
}

template <int WPT>
cudaError_t launch_fixup_t(const msq_plan* pl, const msq::FixParams& prm, int nblocks, cudaStream_t st) {
    auto kern = msq::fixup_kernel<WPT>;
    static bool attr_set[64] = {false};
    cudaError_t e = set_smem_attr(kern, attr_set);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};  // programmatic dependent of the carry scan
    cfg.gridDim = dim3((unsigned)nblocks);
    cfg.blockDim = dim3((unsigned)pl->fix_threads);
    cfg.dynamicSmemBytes = (size_t)pl->smem_fixup;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, prm);
    return cudaGetLastError();
}

cudaError_t launch_pass1(const msq_plan* pl, const msq::Pass1Params& prm, cudaStream_t st) {
    const bool u8 = pl->fmt == MSQ_FMT_U8;
    const bool tma = pl->nstage > 0;
    const bool sub = !cta_plan(pl);
#define MSQ_P1(W_, U_, T_, S_) \
    if (pl->wpt == W_ && u8 == U_ && tma == T_ && sub == S_) return launch_pass1_t<W_, U_, T_, S_>(pl, prm, st);
    MSQ_P1(1, true, true, true) MSQ_P1(1, true, false, true) MSQ_P1(1, false, true, true)
    MSQ_P1(1, false, false, true)
    MSQ_P1(1, true, true, false) MSQ_P1(1, true, false, false) MSQ_P1(1, false, true, false)
    MSQ_P1(1, false, false, false)
    MSQ_P1(2, true, true, false) MSQ_P1(2, true, false, false) MSQ_P1(2, false, true, false)
    MSQ_P1(2, false, false, false)
    MSQ_P1(4, true, true, false) MSQ_P1(4, true, false, false) MSQ_P1(4, false, true, false)
    MSQ_P1(4, false, false, false)
#undef MSQ_P1
    return cudaErrorInvalidValue;
}

// band passes: the strip pass (when it applies) and pass1_kernel for the bands it left
template <int R>
cudaError_t launch_ubits_t(const msq_plan* pl, const msq::UStripParams& up, cudaStream_t st) {
    static bool attr_set[64] = {false};
    cudaError_t e = set_smem_attr(msq::ubits_kernel<R>, attr_set);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};  // programmatic dependent of the seed
    cfg.gridDim = dim3((unsigned)(pl->nbands * up.nchunks));
    cfg.blockDim = dim3((unsigned)((up.nwarps + 1) * 32));
    cfg.dynamicSmemBytes = (size_t)ustrip_smem(up.row_bytes);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, msq::ubits_kernel<R>, up);
}

template <int R>
cudaError_t launch_ustrip_t(const msq_plan* pl, const msq::UStripParams& up, cudaStream_t st) {
    static bool attr_set[64] = {false};
    cudaError_t e = set_smem_attr(msq::ustrip_kernel<R>, attr_set);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};  // programmatic dependent of the seed
    cfg.gridDim = dim3((unsigned)(pl->nbands * up.nchunks));
    cfg.blockDim = dim3((unsigned)((up.nwarps + 1) * 32));
    cfg.dynamicSmemBytes = (size_t)ustrip_smem(up.row_bytes);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, msq::ustrip_kernel<R>, up);
}

cudaError_t launch_ubits(const msq_plan* pl, const msq::Pass1Params& prm, const void* src, const int* redo,
                         cudaStream_t st) {
    {
        msq::UStripParams up{};
        up.src = (const uint8_t*)src;
        up.ld = pl->ld * 4;
        up.rows = (int)pl->rows;
        up.cols = (int)pl->cols;
        up.W = pl->words;
        up.nbands = pl->nbands;
        up.cols_pad = pl->words * 32;
        up.row_base = pl->row_base;
        const StripGeom g = ubits_geom(pl);
        up.nslots = ustrip_slots(g.row_bytes);
        up.row_bytes = g.row_bytes;
        up.nwarps = g.warps;
        up.nchunks = g.chunks;
        up.cw = g.cw;
        up.share = pl->deterministic ? 0 : 1;
        up.zb = prm.zb;
        up.e_out = prm.e_out;
        up.ao_out = prm.ao_out;
        up.band_keys = prm.band_keys;
        up.results = prm.results;
        up.redo = redo;
        if (g.chunks > 1 &&
            cudaMemsetAsync(prm.band_keys, 0, sizeof(unsigned long long) * (size_t)pl->nbands, st) != cudaSuccess)
            return cudaGetLastError();
        switch (ustrip_rows_per_slot(g.row_bytes)) {
            case 8: return launch_ubits_t<8>(pl, up, st);
            case 4: return launch_ubits_t<4>(pl, up, st);
            case 2: return launch_ubits_t<2>(pl, up, st);
            default: return launch_ubits_t<1>(pl, up, st);
        }
    }
}

cudaError_t launch_band_pass(const msq_plan* pl, msq::Pass1Params prm, void* ws, const void* src, cudaStream_t st,
                             int* nlaunch) {
    *nlaunch = 1;
    if (prm.write_summaries && ustrip_applies(pl) && ((uintptr_t)src % 16) == 0) {
        msq::UStripParams up{};
        up.src = (const uint8_t*)src;
        up.ld = pl->ld;
        up.rows = (int)pl->rows;
        up.cols = (int)pl->cols;
        up.W = pl->words;
        up.nbands = pl->nbands;
        up.cols_pad = pl->words * 32;
        up.row_base = pl->row_base;
        const StripGeom g = ustrip_geom(pl);
        up.nslots = ustrip_slots(g.row_bytes);
        up.row_bytes = g.row_bytes;
        up.nwarps = g.warps;
        up.nchunks = g.chunks;
        up.cw = g.cw;
        up.share = pl->deterministic ? 0 : 1;
        up.zb = prm.zb;
        up.e_out = prm.e_out;
        up.ao_out = prm.ao_out;
        up.band_keys = prm.band_keys;
        up.results = prm.results;
        if (g.chunks > 1 &&
            cudaMemsetAsync(prm.band_keys, 0, sizeof(unsigned long long) * (size_t)pl->nbands, st) != cudaSuccess)
            return cudaGetLastError();
        switch (ustrip_rows_per_slot(g.row_bytes)) {
            case 8: return launch_ustrip_t<8>(pl, up, st);
            case 4: return launch_ustrip_t<4>(pl, up, st);
            case 2: return launch_ustrip_t<2>(pl, up, st);
            default: return launch_ustrip_t<1>(pl, up, st);
        }
    }
    if (prm.write_summaries && strip_applies(pl) && ((uintptr_t)src % 16) == 0) {
        WsLayout L = ws_layout(pl);
        uint8_t* w = (uint8_t*)ws;
        msq::StripParams sp{};
        sp.src = (const uint8_t*)src;
        sp.ld_bytes = pl->ld * 4;
        sp.rows = (int)pl->rows;
        sp.cols = (int)pl->cols;
        sp.W = pl->words;
        sp.nbands = pl->nbands;
        sp.cols_pad = pl->words * 32;
        sp.row_base = pl->row_base;
        sp.nslots = strip_slots(pl);
        sp.row_bytes = pl->row_stage_bytes;
        sp.nwarps = strip_warps(pl);
        sp.zw = (uint16_t*)(w + L.zw);
        sp.zb = prm.zb;
        sp.e_out = prm.e_out;
        sp.ao_out = prm.ao_out;
        sp.band_keys = prm.band_keys;
        sp.results = prm.results;
        sp.redo = (int*)(w + L.redo);
        static bool attr_set[64] = {false};
        cudaError_t e = set_smem_attr(msq::strip_kernel, attr_set);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg{};  // programmatic dependent of the seed
        cfg.gridDim = dim3((unsigned)pl->nbands);
        cfg.blockDim = dim3((unsigned)((sp.nwarps + 1) * 32));
        cfg.dynamicSmemBytes = (size_t)strip_smem(pl);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, msq::strip_kernel, sp);
        if (e != cudaSuccess) return e;
        prm.redo = sp.redo;
        *nlaunch = 2;
        // bands the strip pass left (start threshold outside [96, 222] or passed 222)
        if (ubits_applies(pl)) return launch_ubits(pl, prm, src, sp.redo, st);
    } else if (prm.write_summaries && ubits_applies(pl) && ((uintptr_t)src % 16) == 0) {
        return launch_ubits(pl, prm, src, nullptr, st);
    }
    return launch_pass1(pl, prm, st);
}

// tests only: plan->test_floor = k presets the shared best side to k (a lower
// bound the caller vouches for, k <= answer), as if the seed had found it
cudaError_t apply_test_floor(const msq_plan* pl, msq_devresult* d_result, cudaStream_t st) {
    if (pl->test_floor <= 0 || pl->batch != 1) return cudaSuccess;
    return cudaMemcpyAsync(&d_result->best_side, &pl->test_floor, sizeof(int32_t), cudaMemcpyHostToDevice, st);
}

cudaError_t launch_fixup(const msq_plan* pl, const msq::FixParams& prm, int nblocks, cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    if (!(pl->flags & MSQ_PLAN_CLIMB_FIXUP)) {  // window-search fix-up (msq_fixup2.cuh)
        static bool attr_set[64] = {false};
        cudaError_t e = set_smem_attr(msq::fixup2_kernel, attr_set);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg{};  // programmatic dependent of the carry scan
        cfg.gridDim = dim3((unsigned)nblocks);
        cfg.blockDim = dim3((unsigned)msq::FIX2_THREADS);
        cfg.dynamicSmemBytes = (size_t)msq::fix2_layout(pl->words).total;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, msq::fixup2_kernel, prm);
        return cudaGetLastError();
    }
    switch (pl->fix_wpt) {
        case 1: return launch_fixup_t<1>(pl, prm, nblocks, st);
        case 2: return launch_fixup_t<2>(pl, prm, nblocks, st);
        case 4: return launch_fixup_t<4>(pl, prm, nblocks, st);
        default: return cudaErrorInvalidValue;
    }
}

int team_layout_bytes(const msq_plan* pl) {
    return msq::p1_layout(pl->team, pl->wpt, pl->nstage, pl->row_stage_bytes, pl->tile_rows, zplanes_for(pl),
                          pl->nstage > 0, cta_plan(pl))
        .total;
}

msq::Pass1Params make_pass1(const msq_plan* pl, const void* src, void* ws, msq_devresult* res,
                            bool summaries) {
    WsLayout L = ws_layout(pl);
    uint8_t* w = (uint8_t*)ws;
    msq::Pass1Params p{};
    p.src = (const uint8_t*)src;
    const long long esz = pl->fmt == MSQ_FMT_U8 ? 1 : 4;
    p.ld_bytes = pl->ld * esz;
    p.batch_stride = pl->rows * pl->ld * esz;
    p.rows = (int)pl->rows;
    p.cols = (int)pl->cols;
    p.W = pl->words;
    p.nbands = pl->nbands;
    p.cols_pad = pl->words * 32;
    p.row_base = pl->row_base;
    p.nstage = pl->nstage;
    p.rs = pl->row_stage_bytes;
    p.row_bytes = pl->row_stage_bytes;
    p.bs = pl->tile_rows;
    p.bl = pl->tile_rows_l;
    p.tl = pl->tl;
    p.share = (pl->deterministic || pl->nbands == 1) ? 0 : 1;
    p.write_summaries = summaries ? 1 : 0;
    p.team = pl->team;
    p.teams_per_cta = pl->teams_per_cta;
    p.zplanes = zplanes_for(pl);
    p.units = pl->nbands * pl->batch;
    p.layout_bytes = team_layout_bytes(pl);
    p.zb = (uint16_t*)(w + L.zb);
    p.e_out = summaries ? (uint16_t*)(w + L.e) : nullptr;
    p.ao_out = summaries ? (uint32_t*)(w + L.ao) : nullptr;
    p.band_keys = (unsigned long long*)(w + L.band_keys);
    p.results = (unsigned char*)res;
    p.prof = g_prof;
    return p;
}

msq::FixParams make_fix(const msq_plan* pl, void* ws, const uint32_t* base, msq_devresult* res) {
    WsLayout L = ws_layout(pl);
    uint8_t* w = (uint8_t*)ws;
    msq::FixParams f{};
    f.rows = (int)pl->rows;
    f.cols = (int)pl->cols;
    f.W = pl->words;
    f.nbands = pl->nbands;
    f.cols_pad = pl->words * 32;
    f.row_base = pl->row_base;
    f.band_begin = base ? 0 : 1;
    f.bs = pl->tile_rows;
    f.bl = pl->tile_rows_l;
    f.e_in = (const uint16_t*)(w + L.e);
    f.carry_in = (const uint16_t*)(w + L.carry);
    f.share = pl->deterministic ? 0 : 1;
    f.fix_keys = (unsigned long long*)(w + L.fix_keys);
    f.results = (unsigned char*)res;
    return f;
}

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return MSQ_OK;
    if (g_last_err[0] && e == cudaErrorLaunchOutOfResources) return MSQ_ECUDA;
    snprintf(g_last_err, sizeof(g_last_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return MSQ_ECUDA;
}

cudaError_t launch_carry(const msq_plan* pl, void* ws, const uint32_t* base, cudaStream_t st) {
    WsLayout L = ws_layout(pl);
    uint8_t* w = (uint8_t*)ws;
    // programmatic dependent launch: the CTAs launch while the band pass drains
    // and wait (griddepcontrol.wait) for its writes
    cudaLaunchConfig_t cfg{};
    const int lanes = pl->words * 32 <= 32768 ? 16 : 32;  // columns per CTA = 8 * lanes
    cfg.gridDim = dim3((unsigned)ceil_div(pl->words * 32, 8 * lanes));
    cfg.blockDim = dim3(lanes, msq::CARRY_SEG);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (lanes == 16)
        return cudaLaunchKernelEx(&cfg, msq::carry_scan_kernel<16>, (int)pl->rows, (int)pl->cols, pl->words,
                                  pl->nbands, pl->words * 32, (const uint16_t*)(w + L.zb),
                                  (const uint32_t*)(w + L.ao), base, (uint16_t*)(w + L.carry));
    return cudaLaunchKernelEx(&cfg, msq::carry_scan_kernel<32>, (int)pl->rows, (int)pl->cols, pl->words, pl->nbands,
                              pl->words * 32, (const uint16_t*)(w + L.zb), (const uint32_t*)(w + L.ao), base,
                              (uint16_t*)(w + L.carry));
}

// Lower-bound seed before pass 1 (shared-threshold mode only): strips of
// SEED_ROWS rows x 1024-column chunks, one warp each; about 2% of the input
// bytes.  Skipped for small matrices, batches and deterministic plans.
bool seed_disabled(const msq_plan* pl) { return (pl->flags & MSQ_PLAN_NO_SEED) != 0; }  // experiments
int seeds_launched(const msq_plan* pl) {
    return (seed_disabled(pl) || pl->deterministic || pl->batch != 1 || pl->rows < 8 * msq::SEED_ROWS || pl->cols < 256) ? 0 : 1;
}
cudaError_t launch_seed(const msq_plan* pl, const void* d_src, msq_devresult* d_result, cudaStream_t st) {
    if (seed_disabled(pl) || pl->deterministic || pl->batch != 1 || pl->rows < 8 * msq::SEED_ROWS || pl->cols < 256) return cudaSuccess;
    const int chunks = (int)ceil_div(pl->words, 32);
    const long long nstrips = std::max<long long>(1, std::min<long long>(pl->rows / 6400, std::max(1, 1024 / chunks)));
    const long long warps = nstrips * chunks;
    const long long ld_bytes = pl->fmt == MSQ_FMT_U8 ? pl->ld : pl->ld * 4;
    // 2 warps per CTA: the strips spread over every SM (the seed is latency-bound)
    const int blocks = (int)ceil_div(warps * 32, 64);
    if (pl->fmt == MSQ_FMT_U8)
        msq::seed_climb_kernel<true><<<blocks, 64, 0, st>>>((const uint8_t*)d_src, ld_bytes, (int)pl->rows,
                                                              (int)pl->cols, pl->words, (int)nstrips, chunks,
                                                              (unsigned char*)d_result);
    else
        msq::seed_climb_kernel<false><<<blocks, 64, 0, st>>>((const uint8_t*)d_src, ld_bytes, (int)pl->rows,
                                                               (int)pl->cols, pl->words, (int)nstrips, chunks,
                                                               (unsigned char*)d_result);
    return cudaGetLastError();
}


bool key_range_ok(const msq_plan* pl);

// ---- sieve engine (msq_sieve.cuh): bit-packed single matrices, sparse zeros
struct SieveGeom {
    int CR, CC, CWn, WC, nbands, nchunks, wmax, nslots, slot_row_bytes, smem, nunits;
    size_t ctl, cand, G, total;  // workspace offsets (after the band engine's layout)
};
int g_sieve_wpc = 8;  // most consumer warps per CTA of the streaming pass (instrumentation)
int g_sieve_phases = 0;  // > 0: sweeps of the streaming pass whatever the height (tests)

bool sieve_shape_ok(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld) {
    const int64_t words = ceil_div(cols, 32);
    return fmt == MSQ_FMT_BITS && batch == 1 && rows >= 64 && cols >= 64 && rows < (1ll << 21) - 1 - msq::SV_HALO_ROWS &&
           cols <= 65536 && ld >= words && (ld * 4) % 16 == 0;
}

// geometry for `rows` rows (halo rows included); nbands_fixed > 0 keeps the plan's band count
SieveGeom sieve_geom(int64_t rows, int64_t cols, int nbands_fixed) {
    SieveGeom g{};
    const int W = (int)round_up(ceil_div(cols, 32), 4);  // rows are copied in 16-byte units
    g.CR = (int)(rows / 8);
    g.CC = (int)(cols / 8);
    g.CWn = (int)ceil_div(g.CC, 32);
    g.WC = (int)ceil_div(g.CWn, 31);
    g.nunits = (int)ceil_div(g.CR, msq::SV_OWN);
    const int WF = (int)ceil_div(W, 256);  // streaming warps per row
    g.nchunks = (int)ceil_div(WF, std::max(1, g_sieve_wpc));
    g.wmax = (int)ceil_div(WF, g.nchunks);
    g.nbands = nbands_fixed > 0 ? nbands_fixed
                                : (int)std::max<long long>(1, std::min<long long>(num_sms() / g.nchunks, g.CR));
    int rb = 0;
    for (int c = 0; c < g.nchunks; ++c) {
        const int wc0 = WF * c / g.nchunks, wc1 = WF * (c + 1) / g.nchunks;
        rb = std::max(rb, (std::min(W, 256 * wc1) - 256 * wc0) * 4);
    }
    g.slot_row_bytes = rb;
    const int fixed = 2 * msq::SV_MAXSLOTS * 8 + 64;
    g.nslots = (int)std::min<long long>(msq::SV_MAXSLOTS, (kSmemMax - 256 - fixed) / ((long long)msq::SV_TR * rb));
    g.smem = g.nslots * msq::SV_TR * rb + fixed;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (size_t)round_up((long long)bytes, 256);
        return o;
    };
    g.ctl = take(sizeof(msq::SieveCtl) + msq::SV_PHASES * 4);  // + phase counters, zeroed together
    g.cand = take((size_t)msq::SV_CAP * 8);
    g.G = take((size_t)g.CR * g.CWn * 4);
    g.total = off;
    return g;
}

msq::SieveParams make_sieve(const msq_plan* pl, const void* d_src, const void* d_halo, int64_t halo_rows,
                            int64_t halo_ld, void* d_ws, msq_devresult* res) {
    const SieveGeom g = sieve_geom(pl->rows + halo_rows, pl->cols, pl->sv_bands);
    uint8_t* w = (uint8_t*)d_ws + pl->sv_ws_off;
    msq::SieveParams p{};
    p.src = (const uint8_t*)d_src;
    p.halo = (const uint8_t*)d_halo;
    p.ld_bytes = pl->ld * 4;
    p.halo_ld_bytes = halo_ld * 4;
    p.halo_rows = (int)halo_rows;
    p.rows = (int)(pl->rows + halo_rows);
    p.cols = (int)pl->cols;
    p.W = pl->words;
    p.row_base = pl->row_base - halo_rows;
    p.CR = g.CR;
    p.CC = g.CC;
    p.CWn = g.CWn;
    p.WC = g.WC;
    p.nbands = g.nbands;
    p.nchunks = g.nchunks;
    p.wmax = g.wmax;
    p.nslots = g.nslots;
    p.slot_row_bytes = g.slot_row_bytes;
    p.nunits = g.nunits;
    p.coarse_warps = (int)ceil_div((long long)g.nunits * g.WC, msq::SV_EWARPS) * msq::SV_EWARPS;
    p.ctl = (msq::SieveCtl*)(w + g.ctl);
    p.cand = (unsigned long long*)(w + g.cand);
    p.G = (uint32_t*)(w + g.G);
    // a sweep should give every CTA a few tiles: short slices (one rank of many) take fewer
    // (measured on slices of cfg4, tools/time_slice_phases.py: 8192 rows 0.042 ms with 2
    // sweeps against 0.045 with 1; 16384 rows 0.049 with 4 against 0.053 with 1)
    p.nphases = g_sieve_phases > 0 ? std::min(g_sieve_phases, msq::SV_PHASES)
                                   : (int)std::max<long long>(1, std::min<long long>(msq::SV_PHASES, g.CR / (3ll * g.nbands)));
    // equal sweeps.  (A short last sweep -- 3:3:3:1 or 4:3:2:1 of the rows, to leave less
    // of the coarse pass behind the streaming pass -- measured slower on cfg4: 0.114 and
    // 0.107 ms against 0.1045: the short pieces cost the streaming pass more than the
    // coarse pass gains.)
    for (int k = 0; k <= msq::SV_PHASES; ++k)
        p.prow[k] = (int)((long long)g.CR * std::min(k, p.nphases) / p.nphases);
    p.prow[p.nphases] = g.CR;
    p.pcnt = (int*)(w + g.ctl + sizeof(msq::SieveCtl));
    p.ptarget = g.nbands * (int)ceil_div(round_up(pl->words, 4), 256);
    p.result = (unsigned char*)res;
    return p;
}

bool sieve_args_ok(const msq_plan* pl, const void* d_src, const void* d_halo, int64_t halo_rows, int64_t halo_ld,
                   const void* d_ws, const msq_devresult* d_result) {
    if (!pl || pl->engine != 2 || !d_src || !d_ws || !d_result || ((uintptr_t)d_src % 16) != 0) return false;
    if (halo_rows < 0 || halo_rows % 8 != 0 || halo_rows > msq::SV_HALO_ROWS) return false;
    if (halo_rows > 0 && (!d_halo || ((uintptr_t)d_halo % 16) != 0 || halo_ld < pl->words || (halo_ld * 4) % 16 != 0))
        return false;
    return pl->row_base - halo_rows >= 0 && key_range_ok(pl);
}

// memsets + the streaming pass
cudaError_t launch_sieve_pass(const msq_plan* pl, const msq::SieveParams& sp, cudaStream_t st) {
    const SieveGeom g = sieve_geom(sp.rows, sp.cols, pl->sv_bands);
    // one memset: control block, phase counters and the candidate list behind them
    // (the result block is zeroed by the streaming pass itself)
    if (cudaMemsetAsync(sp.ctl, 0, g.cand - g.ctl + (size_t)msq::SV_CAP * 8, st) != cudaSuccess)
        return cudaGetLastError();
    static bool attr_set[64] = {false};
    cudaError_t e = set_smem_attr(msq::sieve_pass_kernel, attr_set);
    if (e != cudaSuccess) return e;
    msq::sieve_pass_kernel<<<g.nbands * g.nchunks, (g.wmax + 1) * 32, (size_t)g.smem, st>>>(sp);
    return cudaGetLastError();
}

// Algorithm 1 on the block bitmap, then the exact windows of its candidates
cudaError_t launch_sieve_finish(const msq::SieveParams& sp, cudaStream_t st) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)ceil_div((long long)sp.nunits * sp.WC, msq::SV_EWARPS));
    cfg.blockDim = dim3(32 * msq::SV_EWARPS);
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, msq::sieve_coarse_kernel, sp);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3((unsigned)(num_sms() * 2));
    cfg.blockDim = dim3(32 * msq::SV_VWARPS);
    return cudaLaunchKernelEx(&cfg, msq::sieve_verify_kernel, sp);
}

// --------------------------------------------------- internal workspace
struct DevCache {
    std::mutex mu;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    void* in = nullptr;  // staging for host-buffer calls
    size_t in_bytes = 0;
    msq_devresult* res = nullptr;
    size_t res_cap = 0;
    msq_devresult* hres = nullptr;  // pinned
    size_t hres_cap = 0;
    unsigned* flag = nullptr;  // 16 bytes of device flags (cube probe)
    void* dpws = nullptr;      // row-DP / brute-force workspace
    size_t dpws_bytes = 0;
    // pageable host -> device staging (host-buffer calls): per worker thread two
    // pinned chunks, their events and a copy stream
    static constexpr int kStageWorkers = 16, kStageBufs = 4;
    void* stage[kStageWorkers][kStageBufs] = {};
    cudaEvent_t stage_ev[kStageWorkers][kStageBufs] = {};
    cudaEvent_t stage_done[kStageWorkers] = {};
    cudaStream_t stage_st[kStageWorkers] = {};
    int stage_ready = 0;
    size_t stage_chunk = 0;  // bytes per pinned buffer (allocated for every worker and buffer)
};
DevCache g_cache[64];

int grow(void** p, size_t* cap, size_t need) {
    if (*cap >= need) return MSQ_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc(p, need) != cudaSuccess) {
        cudaGetLastError();
        return MSQ_ENOMEM;
    }
    *cap = need;
    return MSQ_OK;
}

// Solve with the per-device cache; the caller holds C.mu from its own staging
// (if any) through the result copy, so no other thread's input or workspace
// can land in between.
// keys pack global rows and columns into KEY_DIM_BITS each (msq_engine.cuh)
bool key_range_ok(const msq_plan* pl) {
    return pl->row_base >= 0 && pl->row_base + pl->rows <= (1ll << msq::KEY_DIM_BITS) - 1 &&
           pl->cols <= (1ll << msq::KEY_DIM_BITS) - 1;
}

int dp_solve_locked(DevCache& C, int32_t fmt, const void* d_src, int64_t rows, int64_t cols, int64_t ld,
                    uint32_t* d_heights, int32_t* d_rowmax, msq_result* out, void* stream);
bool dp_shape_ok(int32_t fmt, int64_t rows, int64_t cols, int64_t ld);

// shapes past the band engine's key and carry ranges (cols > 65536 or
// rows >= 2^21 - 1): solved by the row-parallel DP kernel (msq_rowdp.cuh),
// whose 40-bit linear-index key covers any matrix that fits in memory
bool beyond_band_engine(int64_t rows, int64_t cols) {
    return cols > (int64_t)kMaxWords * 32 || rows >= (1ll << msq::KEY_DIM_BITS) - 1;
}

int solve_locked(DevCache& C, int32_t fmt, int64_t batch, const void* d_src, int64_t rows, int64_t cols, int64_t ld,
                 msq_result* out, void* stream) {
    if (batch == 1 && beyond_band_engine(rows, cols) && dp_shape_ok(fmt, rows, cols, ld))
        return dp_solve_locked(C, fmt, d_src, rows, cols, ld, nullptr, nullptr, out, stream);
    msq_plan pl;
    int rc = msq_plan_make(fmt, (int32_t)batch, rows, cols, ld, 0, 0, &pl);
    if (rc) return rc;
    if ((rc = grow(&C.ws, &C.ws_bytes, (size_t)std::max<int64_t>(pl.ws_bytes, 256)))) return rc;
    if ((rc = grow((void**)&C.res, &C.res_cap, sizeof(msq_devresult) * (size_t)batch))) return rc;
    if (C.hres_cap < (size_t)batch) {
        if (C.hres) cudaFreeHost(C.hres);
        C.hres = nullptr;
        C.hres_cap = 0;
        if (cudaMallocHost((void**)&C.hres, sizeof(msq_devresult) * (size_t)batch) != cudaSuccess)
            return MSQ_ENOMEM;
        C.hres_cap = (size_t)batch;
    }
    cudaStream_t st = (cudaStream_t)stream;
    rc = msq_launch(&pl, d_src, C.ws, C.res, stream);
    if (rc) return rc;
    if (cudaMemcpyAsync(C.hres, C.res, sizeof(msq_devresult) * (size_t)batch, cudaMemcpyDeviceToHost,
                        st) != cudaSuccess)
        return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    if (pl.engine == 2 && (C.hres[0].status & 6u)) {  // the sieve could not decide: band engine
        pl.engine = 0;
        rc = msq_launch(&pl, d_src, C.ws, C.res, stream);
        if (rc) return rc;
        if (cudaMemcpyAsync(C.hres, C.res, sizeof(msq_devresult), cudaMemcpyDeviceToHost, st) != cudaSuccess)
            return MSQ_ECUDA;
        if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    }
    int worst = MSQ_OK;
    for (int64_t k = 0; k < batch; ++k) {
        int r = msq_decode(&C.hres[k], rows, cols, &out[k]);
        if (r) worst = r;
    }
    return worst;
}

bool empty_shape(int64_t batch, int64_t rows, int64_t cols, msq_result* out, int* rc) {
    if (rows != 0 && cols != 0) return false;
    if (rows < 0 || cols < 0 || (rows == 0 && cols != 0)) {
        *rc = MSQ_EINVAL;
        return true;
    }
    for (int64_t k = 0; k < std::max<int64_t>(batch, 1); ++k) out[k] = msq_result{0, 0, 0, -1, -1};
    *rc = MSQ_OK;
    return true;
}

int solve_sync(int32_t fmt, int64_t batch, const void* d_src, int64_t rows, int64_t cols, int64_t ld,
               msq_result* out, void* stream) {
    if (!out) return MSQ_EINVAL;
    int rc;
    if (empty_shape(batch, rows, cols, out, &rc)) return rc;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    return solve_locked(C, fmt, batch, d_src, rows, cols, ld, out, stream);
}

}  // namespace


namespace {
int plan_band(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld, int32_t nbands,
              int32_t deterministic, msq_plan* plan);

// ---- register team engine (msq_team.cuh): small matrices, one team per matrix
constexpr int kTeamThreads = 32;  // one warp per CTA: fine-grained spread over the SMs

int team_planes(long long rows) { return rows <= 504 ? 9 : 11; }  // rows <= 2^PB - 8
constexpr int kTeamMaxRows = 2040;  // one team walks <= 2^11 - 8 rows (11 last-zero planes)
int g_team_band_rows = 16;           // band height of the team engine's row-band mode (instrumentation)

// engine: -1 automatic, 0 band engine, 1 team engine (where it applies)
bool team_applies(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int32_t nbands, int32_t engine) {
    if (engine == 0) return false;
    const bool forced = engine == 1;
    if (nbands > 0 || cols > 1024) return false;
    (void)fmt;
    // batches: one team per matrix (rows <= 2040).  Single matrices: one team
    // per row band of the band plan (carry scan + fix-up behind), measured
    // faster than the band engine for every width <= 1024 (512^2 44 vs 152 us,
    // 1024^2 41 vs 158 us, 2000x1000 82 vs 485 us); the single-team chain only
    // when the plan has one band.
    if (batch > 1) return rows <= kTeamMaxRows;
    return forced || rows <= 600 || rows <= (long long)kTeamMaxRows * std::min<long long>(num_sms(), std::max<long long>(1, rows / 64));
}

template <int TEAM, int PB, bool BANDS>
cudaError_t launch_team_t(const msq_plan* pl, const void* d_src, msq_devresult* d_result, cudaStream_t st,
                          const msq::TeamBands& tb) {
    const int mpb = (kTeamThreads / 32) * (32 / TEAM);
    const int units = BANDS ? tb.nbands : pl->batch;
    const int blocks = (int)ceil_div(units, mpb);
    const bool u8 = pl->fmt == MSQ_FMT_U8;
    const long long ld_bytes = u8 ? pl->ld : pl->ld * 4;
    // band mode: the kernel takes the matrix's rows in mat_stride and the tallest band in rows
    const long long mstride = BANDS ? pl->rows : pl->rows * ld_bytes;
    const bool vec = u8 && pl->cols % 32 == 0 && ld_bytes % 16 == 0 && ((uintptr_t)d_src % 16) == 0;
    const uint8_t* s = (const uint8_t*)d_src;
    unsigned char* r = (unsigned char*)d_result;
    const int R = BANDS ? (int)ceil_div(pl->rows, tb.nbands) : (int)pl->rows;
    const int C = (int)pl->cols, W = pl->words, B = units;
    if (!u8)
        msq::team_kernel<TEAM, PB, false, false, 16, BANDS><<<blocks, kTeamThreads, 0, st>>>(s, mstride, ld_bytes, R, C, W, B, r, tb);
    else if (vec)
        msq::team_kernel<TEAM, PB, true, true, 8, BANDS><<<blocks, kTeamThreads, 0, st>>>(s, mstride, ld_bytes, R, C, W, B, r, tb);
    else
        msq::team_kernel<TEAM, PB, true, false, 8, BANDS><<<blocks, kTeamThreads, 0, st>>>(s, mstride, ld_bytes, R, C, W, B, r, tb);
    return cudaGetLastError();
}

template <int PB>
cudaError_t launch_team_pb(const msq_plan* pl, const void* d_src, msq_devresult* d_result, cudaStream_t st,
                           const msq::TeamBands* tb) {
    int ts = 1;
    while (ts < pl->words) ts *= 2;
    const msq::TeamBands none{};
    if (tb) {  // row-band mode: teams of 8..32 lanes
        switch (ts) {
            case 1: case 2: case 4: case 8: return launch_team_t<8, PB, true>(pl, d_src, d_result, st, *tb);
            case 16: return launch_team_t<16, PB, true>(pl, d_src, d_result, st, *tb);
            case 32: return launch_team_t<32, PB, true>(pl, d_src, d_result, st, *tb);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (ts) {
        case 1: return launch_team_t<1, PB, false>(pl, d_src, d_result, st, none);
        case 2: return launch_team_t<2, PB, false>(pl, d_src, d_result, st, none);
        case 4: return launch_team_t<4, PB, false>(pl, d_src, d_result, st, none);
        case 8: return launch_team_t<8, PB, false>(pl, d_src, d_result, st, none);
        case 16: return launch_team_t<16, PB, false>(pl, d_src, d_result, st, none);
        case 32: return launch_team_t<32, PB, false>(pl, d_src, d_result, st, none);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_team(const msq_plan* pl, const void* d_src, msq_devresult* d_result, cudaStream_t st,
                        const msq::TeamBands* tb = nullptr) {
    const long long h = tb ? ceil_div(pl->rows, tb->nbands) : pl->rows;  // rows one team walks
    return team_planes(h) == 9 ? launch_team_pb<9>(pl, d_src, d_result, st, tb)
                               : launch_team_pb<11>(pl, d_src, d_result, st, tb);
}
}  // namespace

extern "C" int msq_plan_make(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld, int32_t nbands,
                             int32_t deterministic, msq_plan* plan) {
    return msq_plan_make_ex(fmt, batch, rows, cols, ld, nbands, deterministic, -1, plan);
}

extern "C" int msq_plan_make_ex(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld, int32_t nbands,
                                int32_t deterministic, int32_t engine, msq_plan* plan) {
    if (!plan || engine < -1 || engine > 2) return MSQ_EINVAL;
    msq_plan p{};
    int rc = plan_band(fmt, batch, rows, cols, ld, nbands, deterministic, &p);
    const bool shape_ok = (fmt == MSQ_FMT_U8 || fmt == MSQ_FMT_BITS) && batch >= 1 && rows >= 1 && cols >= 1 &&
                          (fmt == MSQ_FMT_U8 ? ld >= cols : ld >= (cols + 31) / 32);
    // sieve engine: large bit-packed single matrices try it first (the band fields
    // stay valid: they are the fall-back when the sieve cannot decide)
    const bool sieve_auto = engine == -1 && nbands <= 0 && !deterministic && rows >= 4096 && cols >= 4096;
    if (engine == 2 || sieve_auto) {
        const bool ok = rc == MSQ_OK && shape_ok && sieve_shape_ok(fmt, batch, rows, cols, ld);
        if (ok) {
            const SieveGeom g = sieve_geom(rows, cols, 0);
            if (g.nslots >= 2 && g.wmax <= 8) {
                p.engine = 2;
                p.sv_bands = g.nbands;
                p.sv_ws_off = round_up(p.ws_bytes, 256);
                // the bitmap also covers the halo rows a rank may pass (msq_rank_sieve)
                p.ws_bytes = p.sv_ws_off + (int64_t)sieve_geom(rows + msq::SV_HALO_ROWS, cols, g.nbands).total;
                *plan = p;
                return MSQ_OK;
            }
        }
        if (engine == 2) return MSQ_EINVAL;
    }
    if (engine == 1 && !(shape_ok && team_applies(fmt, batch, rows, cols, nbands, engine))) return MSQ_EINVAL;
    if (shape_ok && team_applies(fmt, batch, rows, cols, nbands, engine)) {
        // one matrix on row bands: short bands (a team walks its rows one by one,
        // so the band height is the latency), the carry scan and fix-up behind
        if (rc == MSQ_OK && batch == 1 && nbands <= 0 && rows >= 2 * g_team_band_rows) {
            msq_plan q{};
            const int nbt = (int)std::min<long long>(num_sms(), rows / g_team_band_rows);
            if (nbt > p.nbands && plan_band(fmt, batch, rows, cols, ld, nbt, deterministic, &q) == MSQ_OK) p = q;
        }
        if (rc != MSQ_OK) {  // the band plan does not fit: the team engine needs no workspace
            p = msq_plan{};
            p.fmt = fmt;
            p.batch = batch;
            p.rows = rows;
            p.cols = cols;
            p.ld = ld;
            p.words = (int32_t)ceil_div(cols, 32);
            p.nbands = 1;
            p.deterministic = deterministic ? 1 : 0;
        }
        p.engine = 1;  // the band fields stay valid for the rank (row-band) entry points
        *plan = p;
        return MSQ_OK;
    }
    if (rc == MSQ_OK) *plan = p;
    return rc;
}

namespace {
int plan_band(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld, int32_t nbands,
              int32_t deterministic, msq_plan* plan) {
    if (!plan || (fmt != MSQ_FMT_U8 && fmt != MSQ_FMT_BITS) || batch < 1) return MSQ_EINVAL;
    if (rows < 1 || cols < 1 || rows >= (1ll << 21) || cols > 65536) return MSQ_EINVAL;
    const int64_t words = ceil_div(cols, 32);
    if (fmt == MSQ_FMT_U8 && ld < cols) return MSQ_EINVAL;
    if (fmt == MSQ_FMT_BITS && ld < words) return MSQ_EINVAL;
    if (words > kMaxWords) return MSQ_EINVAL;
    msq_plan p{};
    p.fmt = fmt;
    p.batch = batch;
    p.rows = rows;
    p.cols = cols;
    p.ld = ld;
    p.words = (int32_t)words;
    p.deterministic = deterministic ? 1 : 0;
    p.row_base = 0;
    p.tl = kModeLThreshold;
    const long long row_bytes = fmt == MSQ_FMT_U8 ? cols : words * 4;
    const long long ld_bytes = fmt == MSQ_FMT_U8 ? ld : ld * 4;
    p.row_stage_bytes = (int32_t)row_bytes;
    const bool tma_ok = (row_bytes % 16 == 0) && (ld_bytes % 16 == 0) && row_bytes <= 65536;
    const int sms = num_sms();
    if (batch > 1 && words <= 32) {
        // ---- sub-warp teams: one small matrix per team, several teams per CTA
        p.wpt = 1;
        int ts = 1;
        while (ts < words) ts *= 2;
        p.team = ts;
        p.nbands = 1;
        p.tile_rows = 4;
        p.tile_rows_l = 4;
        long long tpc = std::max<long long>(1, ceil_div(batch, sms));
        const long long gran = std::max(1, 32 / ts);  // teams per warp
        tpc = round_up(tpc, gran);
        tpc = std::min<long long>(tpc, 512 / ts);
        p.nstage = tma_ok ? 2 * 4 : 0;  // ring holds the previous and the current tile
        for (;;) {
            const long long per = msq::p1_layout(ts, 1, p.nstage, (int)row_bytes, p.tile_rows, zplanes_for(&p),
                                                 p.nstage > 0, tpc == 1 && ts >= 32)  // == cta_plan()
                                      .total;
            if (per * tpc <= kSmemMax) break;
            if (p.nstage > 0) {
                p.nstage = 0;
            } else {
                tpc -= gran;
                if (tpc < gran) return MSQ_EINVAL;
            }
        }
        p.teams_per_cta = (int32_t)tpc;
        p.threads = (int32_t)round_up(tpc * ts, 32);
        p.grid = (int32_t)ceil_div(batch, tpc);
        p.smem_pass1 = (int32_t)(tpc * team_layout_bytes(&p));
        p.smem_fixup = 0;
        p.ws_bytes = (int64_t)ws_layout(&p).total;
        *plan = p;
        return MSQ_OK;
    }
    // ---- CTA teams: one band of one matrix per CTA (512 consumer threads max)
    p.wpt = words <= 512 ? 1 : (words <= 1024 ? 2 : 4);
    p.threads = (int32_t)std::max<long long>(32, round_up(ceil_div(words, p.wpt), 32));
    p.fix_wpt = words <= 512 ? 1 : (words <= 1024 ? 2 : 4);
    p.fix_threads = (int32_t)std::max<long long>(32, round_up(ceil_div(words, p.fix_wpt), 32));
    p.team = p.threads;
    p.teams_per_cta = 1;
    int nb = nbands;
    const int chunks = 1;  // callers may split the strip passes' bands into column chunks
    if (batch > 1) {
        nb = 1;
    } else if (nb <= 0) {
        nb = (int)std::min<long long>(sms, std::max<long long>(1, rows / 64));
    }
    nb = (int)std::max<long long>(nb, ceil_div(rows, 4095));  // band heights fit MAXP=12 planes
    if (nb > rows) nb = (int)rows;
    if (nb > 2048) return MSQ_EINVAL;
    if (batch > 1 && nb != 1) return MSQ_EINVAL;
    p.nbands = nb;
    p.col_chunks = chunks;
    p.grid = nb * batch;
    p.tile_rows = 2;
    p.tile_rows_l = msq::BMAX;
    p.nstage = 0;
    const int P = zplanes_for(&p);
    if (tma_ok) {
        // refills happen after the next tile's first barrier, so the ring must
        // hold the previous tile plus the current one (more = deeper prefetch);
        // a single-row small-threshold tile frees one row of E history for it
        auto stages = [&](int bs) {
            const int base = msq::p1_layout(p.threads, p.wpt, 0, (int)row_bytes, bs, P, true, true).total;
            return std::min<long long>((kSmemMax - base - 512) / row_bytes, 32);
        };
        long long ns = stages(p.tile_rows);
        if (ns < 2 * p.tile_rows_l && stages(1) >= 2 * p.tile_rows_l) {
            p.tile_rows = 1;
            ns = stages(1);
        }
        while (p.tile_rows_l > p.tile_rows && ns < 2 * p.tile_rows_l) p.tile_rows_l /= 2;
        // the ring is a whole number of tile-sized slots (one mbarrier, one bulk copy each)
        if (ns >= 2 * p.tile_rows_l) p.nstage = (int32_t)(ns / p.tile_rows_l * p.tile_rows_l);
    }
    p.smem_pass1 = team_layout_bytes(&p);
    p.smem_fixup = msq::fix_layout(p.fix_threads, p.fix_wpt, p.tile_rows).total;
    if (p.smem_pass1 > kSmemMax || p.smem_fixup > kSmemMax) return MSQ_EINVAL;
    p.ws_bytes = (int64_t)ws_layout(&p).total;
    *plan = p;
    return MSQ_OK;
}

}  // namespace

extern "C" {

int msq_launch(const msq_plan* pl, const void* d_src, void* d_ws, msq_devresult* d_result, void* stream) {
    if (!pl || !key_range_ok(pl)) return MSQ_EINVAL;
    if (pl && pl->engine == 1) {  // register team engine: one launch, no workspace
        if (!d_src || !d_result) return MSQ_EINVAL;
        cudaStream_t st = (cudaStream_t)stream;
        g_last_launches = 0;
        if (cudaMemsetAsync(d_result, 0, sizeof(msq_devresult) * (size_t)pl->batch, st) != cudaSuccess)
            return MSQ_ECUDA;
        const bool single = (pl->flags & MSQ_PLAN_SINGLE_TEAM) != 0;  // experiments
        if (pl->batch == 1 && pl->nbands > 1 && !single) {
            // one matrix on row bands (the plan keeps every band <= kTeamMaxRows)
            if (!d_ws || pl->ws_bytes <= 0 || ceil_div(pl->rows, pl->nbands) > kTeamMaxRows) return MSQ_EINVAL;
            // one matrix on row bands: a team per band, then carry scan + fix-up
            WsLayout L = ws_layout(pl);
            uint8_t* w = (uint8_t*)d_ws;
            msq::TeamBands tb{};
            tb.nbands = pl->nbands;
            tb.cols_pad = pl->words * 32;
            tb.row_base = pl->row_base;
            tb.e_out = (uint16_t*)(w + L.e);
            tb.zb = (uint16_t*)(w + L.zb);
            tb.ao_out = (uint32_t*)(w + L.ao);
            tb.band_keys = (unsigned long long*)(w + L.band_keys);
            cudaError_t e = launch_team(pl, d_src, d_result, st, &tb);
            if (e != cudaSuccess) return cuda_status(e);
            e = launch_carry(pl, d_ws, nullptr, st);
            if (e != cudaSuccess) return cuda_status(e);
            msq::FixParams f = make_fix(pl, d_ws, nullptr, d_result);
            e = launch_fixup(pl, f, pl->nbands - 1, st);
            if (e != cudaSuccess) return cuda_status(e);
            g_last_launches = 3;
            return MSQ_OK;
        }
        if (pl->rows > kTeamMaxRows) return MSQ_EINVAL;  // one team walks every row
        cudaError_t e = launch_team(pl, d_src, d_result, st);
        if (e != cudaSuccess) return cuda_status(e);
        g_last_launches = 1;
        return MSQ_OK;
    }
    if (!pl || !d_src || !d_result || (!d_ws && pl->ws_bytes > 0)) return MSQ_EINVAL;
    if (pl->engine == 2) {
        if (((uintptr_t)d_src % 16) != 0) {  // the sieve's bulk copies need an aligned base
            msq_plan q = *pl;
            q.engine = 0;
            return msq_launch(&q, d_src, d_ws, d_result, stream);
        }
        return msq_rank_sieve(pl, d_src, nullptr, 0, 0, d_ws, d_result, stream);
    }
    if (pl->nstage > 0 && ((uintptr_t)d_src % 16) != 0) {
        msq_plan q = *pl;  // misaligned base: fall back to direct loads
        q.nstage = 0;
        return msq_launch(&q, d_src, d_ws, d_result, stream);
    }
    cudaStream_t st = (cudaStream_t)stream;
    g_last_launches = 0;
    if (cudaMemsetAsync(d_result, 0, sizeof(msq_devresult) * (size_t)pl->batch, st) != cudaSuccess)
        return MSQ_ECUDA;
    const bool multi = pl->batch == 1 && pl->nbands > 1;
    cudaError_t e = apply_test_floor(pl, d_result, st);
    if (e != cudaSuccess) return cuda_status(e);
    e = launch_seed(pl, d_src, d_result, st);
    if (e != cudaSuccess) return cuda_status(e);
    msq::Pass1Params p1 = make_pass1(pl, d_src, d_ws, d_result, multi);
    int nl = 1;
    e = launch_band_pass(pl, p1, d_ws, d_src, st, &nl);
    if (e != cudaSuccess) return cuda_status(e);
    g_last_launches = nl + seeds_launched(pl);
    if (multi) {
        e = launch_carry(pl, d_ws, nullptr, st);
        if (e != cudaSuccess) return cuda_status(e);
        msq::FixParams f = make_fix(pl, d_ws, nullptr, d_result);
        e = launch_fixup(pl, f, pl->nbands - 1, st);
        if (e != cudaSuccess) return cuda_status(e);
        g_last_launches = nl + 2 + seeds_launched(pl);
    }
    return MSQ_OK;
}

int msq_decode(const msq_devresult* r, int64_t rows, int64_t cols, msq_result* out) {
    if (!r || !out) return MSQ_EINVAL;
    const unsigned long long key = std::max(r->key_pass1, r->key_fix);
    if (key == 0) {
        *out = msq_result{0, 0, rows * cols, -1, -1};
    } else {
        const int64_t side = (int64_t)(key >> (2 * msq::KEY_DIM_BITS));
        const int64_t bottom = (int64_t)(msq::KEY_DIM_MASK - ((key >> msq::KEY_DIM_BITS) & msq::KEY_DIM_MASK));
        const int64_t right = (int64_t)(msq::KEY_DIM_MASK - (key & msq::KEY_DIM_MASK));
        *out = msq_result{side, side * side, rows * cols, bottom - side + 1, right - side + 1};
    }
    if (r->status & 1u) return MSQ_EVALUE;
    return (r->status & 6u) ? MSQ_EAGAIN : MSQ_OK;
}

int msq_solve_u8(const uint8_t* d_cells, int64_t rows, int64_t cols, int64_t ld, msq_result* out,
                 void* stream) {
    return solve_sync(MSQ_FMT_U8, 1, d_cells, rows, cols, ld, out, stream);
}

int msq_solve_bits(const uint32_t* d_words, int64_t rows, int64_t cols, int64_t ld_words, msq_result* out,
                   void* stream) {
    return solve_sync(MSQ_FMT_BITS, 1, d_words, rows, cols, ld_words, out, stream);
}

int msq_parse_text(const char* d_text, int64_t nbytes, int64_t rows, int64_t cols, int32_t fmt, void* d_out,
                   int64_t ld, int64_t* bad_line, void* stream) {
    if (!bad_line || nbytes < 0 || rows < 1 || cols < 1 || rows > 65535 || cols > (1ll << 31) - 2 ||
        (fmt != MSQ_FMT_U8 && fmt != MSQ_FMT_BITS))
        return MSQ_EINVAL;
    if (!d_text || !d_out) return MSQ_EINVAL;
    if (fmt == MSQ_FMT_U8 ? ld < cols : ld < ceil_div(cols, 32)) return MSQ_EINVAL;
    *bad_line = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    int rc;
    if ((rc = grow(&C.ws, &C.ws_bytes, 256))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* d_bad = (unsigned long long*)C.ws;
    if (cudaMemsetAsync(d_bad, 0xFF, 8, st) != cudaSuccess) return MSQ_ECUDA;
    const dim3 grid((unsigned)ceil_div(cols, msq::INGEST_CHARS), (unsigned)rows);
    if (fmt == MSQ_FMT_BITS)
        msq::ingest_text_kernel<true><<<grid, 256, 0, st>>>((const uint8_t*)d_text, nbytes, (int)rows, (int)cols,
                                                           (uint8_t*)d_out, ld * 4, d_bad);
    else
        msq::ingest_text_kernel<false><<<grid, 256, 0, st>>>((const uint8_t*)d_text, nbytes, (int)rows, (int)cols,
                                                            (uint8_t*)d_out, ld, d_bad);
    g_last_launches = 1;
    if (cudaGetLastError() != cudaSuccess) return MSQ_ECUDA;
    unsigned long long h = 0;
    if (cudaMemcpyAsync(&h, d_bad, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    if (h != ~0ull) {
        *bad_line = (int64_t)h;
        return MSQ_EVALUE;
    }
    return MSQ_OK;
}

int msq_cube_probe(const uint8_t* d_vol, int64_t depth, int64_t rows, int64_t cols, int64_t k, uint8_t* d_scratch,
                   int64_t* first_depth, void* stream) {
    if (!first_depth || !d_vol || !d_scratch || depth < 1 || rows < 1 || cols < 1 || k < 1 || depth > (1 << 20))
        return MSQ_EINVAL;
    *first_depth = -1;
    if (k > depth || k > rows || k > cols) return MSQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const long long layer = rows * cols;
    unsigned* d_bad = nullptr;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
        DevCache& C = g_cache[dev];
        std::lock_guard<std::mutex> lk(C.mu);
        if (!C.flag && cudaMalloc((void**)&C.flag, 16) != cudaSuccess) return MSQ_ENOMEM;
        d_bad = C.flag;
    }
    if (cudaMemsetAsync(d_bad, 0, 4, st) != cudaSuccess) return MSQ_ECUDA;
    msq::cube_threshold_kernel<<<(unsigned)ceil_div(layer, 256), 256, 0, st>>>(d_vol, (int)depth, layer, (int)k,
                                                                              d_scratch, d_bad);
    if (cudaGetLastError() != cudaSuccess) return MSQ_ECUDA;
    unsigned hbad = 0;
    if (cudaMemcpyAsync(&hbad, d_bad, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    if (hbad) return MSQ_EVALUE;
    // layers below depth k-1 cannot hold a k-cube (their runs are < k): skip them
    const int64_t d0 = k - 1, nd = depth - d0;
    std::vector<msq_result> res((size_t)nd);
    const int rc = solve_sync(MSQ_FMT_U8, nd, d_scratch + d0 * layer, rows, cols, cols, res.data(), stream);
    if (rc) return rc;
    for (int64_t d = 0; d < nd; ++d)
        if (res[(size_t)d].side >= k) {
            *first_depth = d0 + d;
            break;
        }
    return MSQ_OK;
}

int msq_max_rectangle_u8(const uint8_t* d_cells, int64_t rows, int64_t cols, int64_t ld, void* d_scratch,
                         int64_t* area, int64_t* height, int64_t* width, void* stream) {
    if (!area || !height || !width || rows < 0 || cols < 0 || rows >= (1 << 24) || cols > 65535 ||
        (rows > 0 && cols > 0 && (!d_cells || !d_scratch || ld < cols)))
        return MSQ_EINVAL;
    *area = *height = *width = 0;
    if (rows == 0 || cols == 0) return MSQ_OK;
    cudaStream_t st = (cudaStream_t)stream;
    // scratch: heights [rows][cols] u16, stacks [rows][cols] u16, row (h, w) [rows] u64, key u64, flag
    uint8_t* w = (uint8_t*)d_scratch;
    const size_t hb = (size_t)rows * cols * 2;
    uint16_t* hh = (uint16_t*)w;
    uint16_t* stk = (uint16_t*)(w + hb);
    unsigned long long* rowhw = (unsigned long long*)(w + ((2 * hb + 15) & ~(size_t)15));
    unsigned long long* key = rowhw + rows;
    unsigned* bad = (unsigned*)(key + 1);
    if (cudaMemsetAsync(key, 0, 16, st) != cudaSuccess) return MSQ_ECUDA;
    msq::hist_heights_kernel<<<(unsigned)ceil_div(cols, 256), 256, 0, st>>>(d_cells, ld, (int)rows, (int)cols, hh,
                                                                           bad);
    msq::hist_rows_kernel<<<(unsigned)ceil_div(rows, 128), 128, 0, st>>>(hh, (int)rows, (int)cols, stk, key, rowhw);
    g_last_launches = 2;
    if (cudaGetLastError() != cudaSuccess) return MSQ_ECUDA;
    unsigned long long hk[2] = {0, 0};
    if (cudaMemcpyAsync(hk, key, 16, cudaMemcpyDeviceToHost, st) != cudaSuccess) return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    if ((unsigned)hk[1]) return MSQ_EVALUE;
    if (hk[0] == 0) return MSQ_OK;
    const long long row = 0xFFFFFF - (long long)(hk[0] & 0xFFFFFF);
    unsigned long long hw = 0;
    if (cudaMemcpy(&hw, rowhw + row, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return MSQ_ECUDA;
    *area = (int64_t)(hk[0] >> 24);
    *height = (int64_t)(hw >> 32);
    *width = (int64_t)(hw & 0xFFFFFFFFu);
    return MSQ_OK;
}
int64_t msq_max_rectangle_scratch_bytes(int64_t rows, int64_t cols) {
    const size_t hb = (size_t)rows * cols * 2;
    return (int64_t)(((2 * hb + 15) & ~(size_t)15) + (size_t)rows * 8 + 32);
}

int msq_dp_batch_u8(const uint8_t* d_cells, int64_t batch, int64_t rows, int64_t cols, msq_result* out,
                    void* stream) {
    if (!out || batch < 1 || rows < 0 || cols < 0 || cols > msq::DP_MAXCOLS || rows >= (1 << 20) ||
        batch > (1 << 30))
        return MSQ_EINVAL;
    if (rows == 0 || cols == 0) {
        for (int64_t k = 0; k < batch; ++k) out[k] = msq_result{0, 0, 0, -1, -1};
        return MSQ_OK;
    }
    if (!d_cells) return MSQ_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    int rc;
    if ((rc = grow((void**)&C.res, &C.res_cap, sizeof(msq_devresult) * (size_t)batch))) return rc;
    if (C.hres_cap < (size_t)batch) {
        if (C.hres) cudaFreeHost(C.hres);
        C.hres = nullptr;
        C.hres_cap = 0;
        if (cudaMallocHost((void**)&C.hres, sizeof(msq_devresult) * (size_t)batch) != cudaSuccess)
            return MSQ_ENOMEM;
        C.hres_cap = (size_t)batch;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(C.res, 0, sizeof(msq_devresult) * (size_t)batch, st) != cudaSuccess) return MSQ_ECUDA;
    msq::dp_batch_kernel<<<(int)ceil_div(batch, 128), 128, 0, st>>>(d_cells, (int)batch, (int)rows, (int)cols,
                                                                    (unsigned char*)C.res);
    g_last_launches = 1;
    if (cudaGetLastError() != cudaSuccess) return MSQ_ECUDA;
    if (cudaMemcpyAsync(C.hres, C.res, sizeof(msq_devresult) * (size_t)batch, cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
        return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    int worst = MSQ_OK;
    for (int64_t k = 0; k < batch; ++k) {
        int r = msq_decode(&C.hres[k], rows, cols, &out[k]);
        if (r) worst = r;
    }
    return worst;
}

int msq_solve_batch_u8(const uint8_t* d_cells, int64_t batch, int64_t rows, int64_t cols, msq_result* out,
                       void* stream) {
    if (batch < 1) return MSQ_EINVAL;
    return solve_sync(MSQ_FMT_U8, batch, d_cells, rows, cols, cols, out, stream);
}

namespace {
// staging shape for pageable host buffers (instrumentation can change it:
// msq_debug_set_staging); workers <= 0 means half the hardware threads
struct StageCfg {  // measured on a 16-core B200 host: 41 GB/s (pinned direct: 50 GB/s)
    int workers = 8, bufs = 4;
    size_t chunk = 4u << 20;
} g_stage;

// Host -> device copy of a caller's buffer, ordered before later work on `st`.
// Pinned buffers go straight to cudaMemcpyAsync.  Pageable ones are staged by
// worker threads: each memcpy's its chunks (c = w, w + T, ...) into one of its
// pinned buffers while the others' DMAs run on its own stream, so the host
// copies and PCIe transfers of all workers overlap; `st` then waits on every
// worker stream.  Caller holds C.mu.
int h2d_copy(DevCache& C, int dev, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    cudaPointerAttributes at;
    const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const size_t chunk = g_stage.chunk;
    if (pinned || bytes < 2 * chunk)
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess ? MSQ_OK : MSQ_ECUDA;
    const int hw = (int)std::thread::hardware_concurrency();
    const int T = std::max(1, std::min<int>(DevCache::kStageWorkers, g_stage.workers > 0 ? g_stage.workers : hw / 2));
    const int NB = std::max(2, std::min(DevCache::kStageBufs, g_stage.bufs));
    if (C.stage_ready && C.stage_chunk != chunk) {  // re-shaped: drop the old buffers
        cudaDeviceSynchronize();
        for (int w = 0; w < DevCache::kStageWorkers; ++w)
            for (int b = 0; b < DevCache::kStageBufs; ++b)
                if (C.stage[w][b]) {
                    cudaFreeHost(C.stage[w][b]);
                    C.stage[w][b] = nullptr;
                }
        C.stage_chunk = chunk;
    }
    if (!C.stage_ready) {
        for (int w = 0; w < DevCache::kStageWorkers; ++w) {
            for (int b = 0; b < DevCache::kStageBufs; ++b)
                if (cudaEventCreateWithFlags(&C.stage_ev[w][b], cudaEventDisableTiming) != cudaSuccess)
                    return MSQ_ECUDA;
            if (cudaEventCreateWithFlags(&C.stage_done[w], cudaEventDisableTiming) != cudaSuccess ||
                cudaStreamCreateWithFlags(&C.stage_st[w], cudaStreamNonBlocking) != cudaSuccess)
                return MSQ_ECUDA;
        }
        C.stage_ready = 1;
        C.stage_chunk = chunk;
    }
    for (int w = 0; w < T; ++w)
        for (int b = 0; b < NB; ++b)
            if (!C.stage[w][b] && cudaMallocHost(&C.stage[w][b], chunk) != cudaSuccess) return MSQ_ENOMEM;
    // the destination may still be read by earlier work on `st`
    cudaEvent_t ready;
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) return MSQ_ECUDA;
    cudaEventRecord(ready, st);
    const size_t nchunks = (bytes + chunk - 1) / chunk;
    std::vector<int> rcs(T, MSQ_OK);
    std::vector<std::thread> pool;
    for (int w = 0; w < T; ++w) {
        pool.emplace_back([&, w]() {
            cudaSetDevice(dev);
            cudaStreamWaitEvent(C.stage_st[w], ready, 0);
            int it = 0;
            for (size_t c = (size_t)w; c < nchunks; c += (size_t)T, ++it) {
                const int b = it % NB;
                const size_t off = c * chunk, n = std::min(chunk, bytes - off);
                if (cudaEventSynchronize(C.stage_ev[w][b]) != cudaSuccess) { rcs[w] = MSQ_ECUDA; return; }
                std::memcpy(C.stage[w][b], (const char*)src + off, n);
                if (cudaMemcpyAsync((char*)dst + off, C.stage[w][b], n, cudaMemcpyHostToDevice, C.stage_st[w]) !=
                        cudaSuccess ||
                    cudaEventRecord(C.stage_ev[w][b], C.stage_st[w]) != cudaSuccess) {
                    rcs[w] = MSQ_ECUDA;
                    return;
                }
            }
            if (cudaEventRecord(C.stage_done[w], C.stage_st[w]) != cudaSuccess) rcs[w] = MSQ_ECUDA;
        });
    }
    for (auto& t : pool) t.join();
    cudaEventDestroy(ready);
    for (int w = 0; w < T; ++w) {
        if (rcs[w]) return rcs[w];
        if (cudaStreamWaitEvent(st, C.stage_done[w], 0) != cudaSuccess) return MSQ_ECUDA;
    }
    return MSQ_OK;
}
}  // namespace

static int solve_host(int32_t fmt, const void* h, int64_t rows, int64_t cols, int64_t ld, msq_result* out,
                      void* stream) {
    if (!out) return MSQ_EINVAL;
    int rc;
    if (empty_shape(1, rows, cols, out, &rc)) return rc;
    if (!h) return MSQ_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    const size_t bytes = (size_t)rows * (size_t)ld * (fmt == MSQ_FMT_U8 ? 1 : 4);
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);  // held through the solve: the staging buffer is shared
    if ((rc = grow(&C.in, &C.in_bytes, bytes))) return rc;
    if ((rc = h2d_copy(C, dev, C.in, h, bytes, (cudaStream_t)stream))) return rc;
    return solve_locked(C, fmt, 1, C.in, rows, cols, ld, out, stream);
}

int msq_solve_batch_u8_host(const uint8_t* h_cells, int64_t batch, int64_t rows, int64_t cols,
                            msq_result* out, void* stream) {
    if (!out || batch < 1) return MSQ_EINVAL;
    int rc;
    if (empty_shape(batch, rows, cols, out, &rc)) return rc;
    if (!h_cells) return MSQ_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    const size_t bytes = (size_t)batch * (size_t)rows * (size_t)cols;
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    if ((rc = grow(&C.in, &C.in_bytes, bytes))) return rc;
    if ((rc = h2d_copy(C, dev, C.in, h_cells, bytes, (cudaStream_t)stream))) return rc;
    return solve_locked(C, MSQ_FMT_U8, batch, C.in, rows, cols, cols, out, stream);
}

int msq_solve_u8_host(const uint8_t* h_cells, int64_t rows, int64_t cols, int64_t ld, msq_result* out,
                      void* stream) {
    return solve_host(MSQ_FMT_U8, h_cells, rows, cols, ld, out, stream);
}

int msq_solve_bits_host(const uint32_t* h_words, int64_t rows, int64_t cols, int64_t ld_words,
                        msq_result* out, void* stream) {
    return solve_host(MSQ_FMT_BITS, h_words, rows, cols, ld_words, out, stream);
}

int msq_rank_pass1(const msq_plan* pl, const void* d_src, void* d_ws, msq_devresult* d_result, void* stream) {
    if (pl && !key_range_ok(pl)) return MSQ_EINVAL;
    if (!pl || pl->batch != 1 || !d_src || !d_ws || !d_result || pl->ws_bytes <= 0) return MSQ_EINVAL;
    if (pl->nstage > 0 && ((uintptr_t)d_src % 16) != 0) {
        msq_plan q = *pl;
        q.nstage = 0;
        return msq_rank_pass1(&q, d_src, d_ws, d_result, stream);
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(d_result, 0, sizeof(msq_devresult), st) != cudaSuccess) return MSQ_ECUDA;
    cudaError_t e = apply_test_floor(pl, d_result, st);
    if (e != cudaSuccess) return cuda_status(e);
    e = launch_seed(pl, d_src, d_result, st);
    if (e != cudaSuccess) return cuda_status(e);
    msq::Pass1Params p1 = make_pass1(pl, d_src, d_ws, d_result, true);
    int nl = 1;
    e = launch_band_pass(pl, p1, d_ws, d_src, st, &nl);
    g_last_launches = nl + seeds_launched(pl);
    return cuda_status(e);
}

int msq_rank_seed(const msq_plan* pl, const void* d_src, msq_devresult* d_result, void* stream) {
    if (pl && !key_range_ok(pl)) return MSQ_EINVAL;
    if (!pl || pl->batch != 1 || !d_src || !d_result) return MSQ_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(d_result, 0, sizeof(msq_devresult), st) != cudaSuccess) return MSQ_ECUDA;
    cudaError_t e = apply_test_floor(pl, d_result, st);
    if (e != cudaSuccess) return cuda_status(e);
    e = launch_seed(pl, d_src, d_result, st);
    g_last_launches = seeds_launched(pl);
    return cuda_status(e);
}

int msq_rank_band_pass(const msq_plan* pl, const void* d_src, void* d_ws, msq_devresult* d_result, void* stream) {
    if (pl && !key_range_ok(pl)) return MSQ_EINVAL;
    if (!pl || pl->batch != 1 || !d_src || !d_ws || !d_result || pl->ws_bytes <= 0) return MSQ_EINVAL;
    if (pl->nstage > 0 && ((uintptr_t)d_src % 16) != 0) {
        msq_plan q = *pl;
        q.nstage = 0;
        return msq_rank_band_pass(&q, d_src, d_ws, d_result, stream);
    }
    msq::Pass1Params p1 = make_pass1(pl, d_src, d_ws, d_result, true);
    int nl = 1;
    const cudaError_t e = launch_band_pass(pl, p1, d_ws, d_src, (cudaStream_t)stream, &nl);
    g_last_launches = nl;
    return cuda_status(e);
}

int msq_rank_sieve_pass(const msq_plan* pl, const void* d_src, const void* d_halo, int64_t halo_rows,
                        int64_t halo_ld, void* d_ws, msq_devresult* d_result, void* stream) {
    if (!sieve_args_ok(pl, d_src, d_halo, halo_rows, halo_ld, d_ws, d_result)) return MSQ_EINVAL;
    const msq::SieveParams sp = make_sieve(pl, d_src, d_halo, halo_rows, halo_ld, d_ws, d_result);
    g_last_launches = 1;
    return cuda_status(launch_sieve_pass(pl, sp, (cudaStream_t)stream));
}

int msq_rank_sieve_finish(const msq_plan* pl, const void* d_src, const void* d_halo, int64_t halo_rows,
                          int64_t halo_ld, void* d_ws, msq_devresult* d_result, void* stream) {
    if (!sieve_args_ok(pl, d_src, d_halo, halo_rows, halo_ld, d_ws, d_result)) return MSQ_EINVAL;
    const msq::SieveParams sp = make_sieve(pl, d_src, d_halo, halo_rows, halo_ld, d_ws, d_result);
    g_last_launches = 2;
    return cuda_status(launch_sieve_finish(sp, (cudaStream_t)stream));
}

int msq_rank_sieve(const msq_plan* pl, const void* d_src, const void* d_halo, int64_t halo_rows, int64_t halo_ld,
                   void* d_ws, msq_devresult* d_result, void* stream) {
    int rc = msq_rank_sieve_pass(pl, d_src, d_halo, halo_rows, halo_ld, d_ws, d_result, stream);
    if (rc) return rc;
    rc = msq_rank_sieve_finish(pl, d_src, d_halo, halo_rows, halo_ld, d_ws, d_result, stream);
    g_last_launches = 3;
    return rc;
}

int msq_rank_key_status(const msq_devresult* d_result, int64_t* d_out, void* stream) {
    if (!d_result || !d_out) return MSQ_EINVAL;
    msq::key_status_kernel<<<1, 1, 0, (cudaStream_t)stream>>>((const unsigned char*)d_result, (long long*)d_out);
    g_last_launches = 1;
    return cuda_status(cudaGetLastError());
}

int msq_rank_summary(const msq_plan* pl, const void* d_ws, uint32_t* d_summary, void* stream) {
    if (!pl || !d_ws || !d_summary || pl->batch != 1) return MSQ_EINVAL;
    WsLayout L = ws_layout(pl);
    const uint8_t* w = (const uint8_t*)d_ws;
    const int threads = 256;  // one warp per 32-column word
    const int blocks = (int)ceil_div((long long)pl->words * 32, threads);
    msq::rank_summary_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
        (int)pl->rows, (int)pl->cols, pl->words, pl->nbands, pl->words * 32, (const uint16_t*)(w + L.zb),
        (const uint32_t*)(w + L.ao), d_summary);
    return cuda_status(cudaGetLastError());
}

int msq_compose_carry(const uint32_t* d_summaries, const int64_t* h_rank_rows, int32_t nranks, int32_t rank,
                      int64_t cols, uint32_t* d_base_carry, void* stream) {
    if (!d_summaries || !h_rank_rows || !d_base_carry || nranks < 1 || nranks > 64 || rank < 0 ||
        rank >= nranks || cols < 1)
        return MSQ_EINVAL;
    msq::RankRows rr{};
    for (int q = 0; q < nranks; ++q) rr.r[q] = h_rank_rows[q];
    const int threads = 256;
    msq::compose_carry_kernel<<<(int)ceil_div(cols, threads), threads, 0, (cudaStream_t)stream>>>(
        d_summaries, rr, rank, (int)cols, d_base_carry);
    return cuda_status(cudaGetLastError());
}

int msq_rank_fixup(const msq_plan* pl, void* d_ws, const uint32_t* d_base_carry, msq_devresult* d_result,
                   void* stream) {
    if (pl && !key_range_ok(pl)) return MSQ_EINVAL;
    if (!pl || !d_ws || !d_result || pl->batch != 1) return MSQ_EINVAL;
    cudaError_t e = launch_carry(pl, d_ws, d_base_carry, (cudaStream_t)stream);
    if (e != cudaSuccess) return MSQ_ECUDA;
    msq::FixParams f = make_fix(pl, d_ws, d_base_carry, d_result);
    const int nblocks = pl->nbands - f.band_begin;
    return cuda_status(launch_fixup(pl, f, nblocks, (cudaStream_t)stream));
}

int msq_ws_views(const msq_plan* pl, void* d_ws, uint16_t** e, uint16_t** b, uint32_t** allones,
                 uint64_t** band_keys) {
    if (!pl || !d_ws) return MSQ_EINVAL;
    WsLayout L = ws_layout(pl);
    uint8_t* w = (uint8_t*)d_ws;
    if (e) *e = (uint16_t*)(w + L.e);
    if (b) *b = (uint16_t*)(w + L.zb);
    if (allones) *allones = (uint32_t*)(w + L.ao);
    if (band_keys) *band_keys = (uint64_t*)(w + L.band_keys);
    return MSQ_OK;
}

int msq_gen_hash(int32_t fmt, uint64_t seed, uint64_t thr53, int64_t row0, int64_t nrows, int64_t cols,
                 int64_t ld, void* d_out, void* stream) {
    if (!d_out || nrows < 0 || cols < 1) return MSQ_EINVAL;
    const int threads = 256, blocks = 148 * 8;
    if (fmt == MSQ_FMT_U8)
        msq::gen_hash_u8_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(seed, thr53, row0, nrows, cols,
                                                                              ld, (uint8_t*)d_out);
    else if (fmt == MSQ_FMT_BITS)
        msq::gen_hash_bits_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(seed, thr53, row0, nrows,
                                                                                cols, ld, (uint32_t*)d_out);
    else
        return MSQ_EINVAL;
    return cuda_status(cudaGetLastError());
}

int32_t msq_last_launch_count(void) { return g_last_launches; }

void msq_debug_set_profile(void* d_counters) { g_prof = (unsigned long long*)d_counters; }

const char* msq_strerror(int code) {
    switch (code) {
        case MSQ_OK: return "ok";
        case MSQ_EINVAL: return "invalid argument (shape, stride or unsupported width)";
        case MSQ_EVALUE: return "cells must contain only 0 or 1";
        case MSQ_ECUDA: return "CUDA runtime error";
        case MSQ_EAGAIN: return "the sieve engine could not decide; solve with the band engine (plan.engine = 0)";
        case MSQ_ENOMEM: return "device memory allocation failed";
        default: return "unknown error";
    }
}

const char* msq_version(void) { return "msq 0.1.0 sm_100a"; }

const char* msq_last_cuda_error(void) { return g_last_err; }

}  // extern "C"

// ------------------------------------------------------ DP baselines, traced
namespace {
int64_t rowdp_strips(int32_t fmt, int64_t cols) { return ceil_div(cols, 32 * (fmt == MSQ_FMT_BITS ? 32 : 16)); }

void decode_rowdp(unsigned long long key, int64_t rows, int64_t cols, bool key_is_anchor, msq_result* out) {
    if (!key) {
        *out = msq_result{0, 0, rows * cols, -1, -1};
        return;
    }
    const int64_t side = (int64_t)(key >> msq::ROWDP_LIN_BITS);
    const int64_t lin = (int64_t)(((1ull << msq::ROWDP_LIN_BITS) - 1ull) - (key & ((1ull << msq::ROWDP_LIN_BITS) - 1ull)));
    const int64_t r = lin / cols, c = lin % cols;
    if (key_is_anchor) *out = msq_result{side, side * side, rows * cols, r, c};
    else *out = msq_result{side, side * side, rows * cols, r - side + 1, c - side + 1};
}
}  // namespace

namespace {
// caller holds C.mu
int dp_solve_locked(DevCache& C, int32_t fmt, const void* d_src, int64_t rows, int64_t cols, int64_t ld,
                    uint32_t* d_heights, int32_t* d_rowmax, msq_result* out, void* stream) {
    int rc;
    const int64_t nstrips = rowdp_strips(fmt, cols);
    const size_t bnd_bytes = (size_t)std::max<int64_t>(nstrips - 1, 0) * (size_t)rows * 8;
    const size_t need = 64 + bnd_bytes;
    if ((rc = grow(&C.dpws, &C.dpws_bytes, need))) return rc;
    if (C.hres_cap < 1) {
        if (cudaMallocHost((void**)&C.hres, sizeof(msq_devresult)) != cudaSuccess) return MSQ_ENOMEM;
        C.hres_cap = 1;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(C.dpws, 0, need, st) != cudaSuccess) return MSQ_ECUDA;
    if (d_rowmax && cudaMemsetAsync(d_rowmax, 0, sizeof(int32_t) * (size_t)rows, st) != cudaSuccess)
        return MSQ_ECUDA;
    unsigned char* base = (unsigned char*)C.dpws;
    msq::RowDpParams p;
    p.src = (const uint8_t*)d_src;
    p.ld = ld;
    p.rows = rows;
    p.cols = cols;
    p.nstrips = (int)nstrips;
    p.vec = (fmt == MSQ_FMT_U8 && ((uintptr_t)d_src % 16) == 0 && ld % 16 == 0 && cols % 16 == 0) ? 1 : 0;
    p.key = (unsigned long long*)base;
    p.status = (unsigned int*)(base + 16);
    p.ticket = (unsigned int*)(base + 20);
    p.bnd = (unsigned long long*)(base + 64);
    p.heights = d_heights;
    p.rowmax = d_rowmax;
    const int grid = (int)ceil_div(nstrips, msq::ROWDP_WARPS);
    if (fmt == MSQ_FMT_BITS) msq::rowdp_kernel<true><<<grid, 32 * msq::ROWDP_WARPS, 0, st>>>(p);
    else msq::rowdp_kernel<false><<<grid, 32 * msq::ROWDP_WARPS, 0, st>>>(p);
    g_last_launches = 1;
    if (cudaGetLastError() != cudaSuccess) return MSQ_ECUDA;
    if (cudaMemcpyAsync(C.hres, base, 32, cudaMemcpyDeviceToHost, st) != cudaSuccess) return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    const unsigned long long key = *(const unsigned long long*)C.hres;
    const unsigned status = *(const unsigned*)((const unsigned char*)C.hres + 16);
    decode_rowdp(key, rows, cols, false, out);
    return (status & 1u) ? MSQ_EVALUE : MSQ_OK;
}

bool dp_shape_ok(int32_t fmt, int64_t rows, int64_t cols, int64_t ld) {
    const int64_t words = ceil_div(cols, 32);
    return ld >= (fmt == MSQ_FMT_U8 ? cols : words) && rows * cols < (1ll << msq::ROWDP_LIN_BITS) &&
           cols < (1ll << 31) - 64;
}
}  // namespace

extern "C" int msq_dp_solve(int32_t fmt, const void* d_src, int64_t rows, int64_t cols, int64_t ld,
                            uint32_t* d_heights, int32_t* d_rowmax, msq_result* out, void* stream) {
    if (!out || (fmt != MSQ_FMT_U8 && fmt != MSQ_FMT_BITS)) return MSQ_EINVAL;
    int rc;
    if (empty_shape(1, rows, cols, out, &rc)) return rc;
    if (!d_src || !dp_shape_ok(fmt, rows, cols, ld)) return MSQ_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    return dp_solve_locked(C, fmt, d_src, rows, cols, ld, d_heights, d_rowmax, out, stream);
}

extern "C" int msq_brute_u8(const uint8_t* d_cells, int64_t rows, int64_t cols, int64_t ld, msq_result* out,
                            void* stream) {
    if (!out) return MSQ_EINVAL;
    int rc;
    if (empty_shape(1, rows, cols, out, &rc)) return rc;
    if (!d_cells || ld < cols || rows * cols > (1ll << 24)) return MSQ_EINVAL;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return MSQ_ECUDA;
    DevCache& C = g_cache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    if ((rc = grow(&C.dpws, &C.dpws_bytes, 64))) return rc;
    if (C.hres_cap < 1) {
        if (cudaMallocHost((void**)&C.hres, sizeof(msq_devresult)) != cudaSuccess) return MSQ_ENOMEM;
        C.hres_cap = 1;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(C.dpws, 0, 64, st) != cudaSuccess) return MSQ_ECUDA;
    unsigned char* base = (unsigned char*)C.dpws;
    const int64_t n = rows * cols;
    msq::brute_kernel<<<(int)ceil_div(n, 256), 256, 0, st>>>(d_cells, ld, (int)rows, (int)cols,
                                                             (unsigned long long*)base,
                                                             (unsigned long long*)(base + 8),
                                                             (unsigned int*)(base + 16));
    g_last_launches = 1;
    if (cudaGetLastError() != cudaSuccess) return MSQ_ECUDA;
    if (cudaMemcpyAsync(C.hres, base, 32, cudaMemcpyDeviceToHost, st) != cudaSuccess) return MSQ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MSQ_ECUDA;
    const unsigned long long key = *(const unsigned long long*)C.hres;
    const unsigned long long visited = *(const unsigned long long*)((const unsigned char*)C.hres + 8);
    const unsigned status = *(const unsigned*)((const unsigned char*)C.hres + 16);
    decode_rowdp(key, rows, cols, true, out);
    out->cells_visited = (int64_t)visited;
    return (status & 1u) ? MSQ_EVALUE : MSQ_OK;
}

extern "C" void msq_debug_set_staging(int32_t workers, int32_t buffers, int64_t chunk_bytes) {
    g_stage.workers = workers;
    g_stage.bufs = buffers > 0 ? buffers : 4;
    g_stage.chunk = chunk_bytes > 0 ? (size_t)chunk_bytes : (4u << 20);
}

extern "C" void msq_debug_set_sieve_phases(int32_t phases) { g_sieve_phases = phases > 0 ? phases : 0; }
extern "C" void msq_debug_set_sieve_wpc(int32_t warps) { g_sieve_wpc = warps >= 1 && warps <= 8 ? warps : 8; }
extern "C" void msq_debug_set_team_band_rows(int32_t rows) { g_team_band_rows = rows > 0 ? rows : 16; }
