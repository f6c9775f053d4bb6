/*
 * msq.h -- C ABI of the B200 maximal-square library (libmsq.so).
 *
 * The hot path is the reference's frequency algorithm,
 * /root/reference/pkg/src/squarelab/squares.py:68-114 (_freq_core), reached
 * through freq_square(m, audit=None) -> SquareResult (squares.py:117-126).
 * The reference has no FFI of its own (it is pure Python); these entry points
 * are what its Python solver signature binds to through ctypes (see
 * INTEGRATION.md).  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - Device pointers are caller-owned; the library never frees them.
 *   - u8 cells must be 0 or 1 (grid.py:61-62); any other byte -> MSQ_EVALUE.
 *   - Bit-packed rows: bit b of uint32 word w is column 32*w + b (LSB = lowest
 *     column); padding bits past `cols` are ignored.
 *   - Results: side, area = side^2, cells_visited = rows*cols (squares.py:114),
 *     top/left = the top-left corner of the first maximal square in row-major
 *     order of its bottom-right cell (the cell of Algorithm 1's final threshold
 *     raise, squares.py:93-97); top = left = -1 when side == 0.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every call is reentrant per stream as long as concurrent calls use
 *     distinct workspaces (the msq_solve_* convenience calls share one
 *     internal per-device workspace and serialise on it).
 */
#ifndef MSQ_H
#define MSQ_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MSQ_OK 0
#define MSQ_EINVAL 1   /* bad shape / stride / alignment / unsupported width */
#define MSQ_EVALUE 2   /* a u8 cell outside {0,1} -> Python ValueError       */
#define MSQ_ECUDA 3    /* CUDA runtime error -> Python RuntimeError          */
#define MSQ_ENOMEM 4   /* workspace allocation failed                        */
#define MSQ_EAGAIN 5   /* msq_decode of a sieve-engine launch that could not decide
                          (status bits 1, 2): launch again with plan.engine = 0; the
                          msq_solve_* calls do that themselves                  */

/* input formats */
#define MSQ_FMT_U8 0
#define MSQ_FMT_BITS 1

typedef struct {
    int64_t side;
    int64_t area;
    int64_t cells_visited;
    int64_t top;
    int64_t left;
} msq_result;

/* Device-side result block written by a launch (one per matrix). */
typedef struct {
    uint64_t key_pass1;  /* best key from band passes                     */
    uint64_t key_fix;    /* best key from band-boundary fix-ups            */
    uint32_t status;     /* bit 0: invalid u8 cell; bits 1, 2: the sieve engine
                            could not decide (bit 1: block squares beyond its
                            windows or too many candidates; bit 2: nothing
                            above side 62 in these rows): run the band engine */
    int32_t best_side;   /* running best side shared between bands         */
    uint64_t reserved;
} msq_devresult;

/* Launch plan: everything the kernels need that depends only on the shape. */
typedef struct {
    int32_t fmt;          /* MSQ_FMT_U8 / MSQ_FMT_BITS                      */
    int32_t batch;        /* matrices (stacked, contiguous) >= 1            */
    int64_t rows, cols;   /* per matrix                                     */
    int64_t ld;           /* row stride in elements (bytes / uint32 words)  */
    int32_t words;        /* ceil(cols / 32)                                */
    int32_t wpt;          /* words per thread                               */
    int32_t threads;      /* CTA size                                       */
    int32_t tile_rows;    /* rows per test tile                             */
    int32_t nbands;       /* row bands per matrix (1 for batch)             */
    int32_t nstage;       /* TMA ring depth in tiles (0 = direct loads)     */
    int32_t row_stage_bytes;
    int32_t smem_pass1, smem_fixup;
    int32_t deterministic;/* 1: no cross-band threshold sharing             */
    int64_t row_base;     /* global row index of row 0 (row-band sharding)  */
    int64_t ws_bytes;     /* required workspace bytes                       */
    int32_t team;         /* threads per band team (sub-warp for batches)   */
    int32_t teams_per_cta;
    int32_t tile_rows_l;  /* rows per tile once the threshold is >= tl      */
    int32_t tl;           /* threshold where the word-level filter takes over */
    int32_t grid;         /* pass-1 CTAs                                    */
    int32_t fix_threads;  /* fix-up CTA size                                */
    int32_t fix_wpt;      /* fix-up words per thread                        */
    int32_t engine;       /* 0: band engine; 1: register team engine (small matrices);
                             2: sieve engine (large bit-packed matrices, msq_sieve.cuh):
                             one streaming pass over 8x8-cell blocks + exact windows of
                             the few candidates; exact for answers 56..222, otherwise the
                             result block says so (status bit 1) and the same plan with
                             engine = 0 runs the band engine */
    int32_t flags;        /* MSQ_PLAN_* experiment switches; 0 from msq_plan_make */
    int32_t test_floor;   /* TEST ONLY: > 0 presets the shared best side (the caller
                             vouches that the answer is >= it); 0 from msq_plan_make */
    int32_t col_chunks;   /* column chunks per band for the u8 / any-threshold bit-packed
                             strip passes (one CTA per band and chunk; 1 from
                             msq_plan_make): fewer, taller bands with the same CTA count,
                             so the band summaries (carry scan, fix-up) shrink -- the
                             tile strip pass then stands aside */
    int32_t sv_bands;     /* sieve engine: row bands of the streaming pass */
    int64_t sv_ws_off;    /* sieve engine: its part of the workspace starts here */
} msq_plan;

/* msq_plan.flags: experiment switches a caller may set on its own plan
 * (per call, no global state); production plans leave them 0. */
#define MSQ_PLAN_NO_STRIP 1     /* bit-packed bands: skip the strip pass        */
#define MSQ_PLAN_NO_SEED 2      /* skip the lower-bound seed                     */
#define MSQ_PLAN_SINGLE_TEAM 4  /* team engine: one team per matrix (rows <= 2040) */
#define MSQ_PLAN_CLIMB_FIXUP 8  /* band-boundary fix-up by the per-depth climb (fixup_kernel)
                                   instead of the window search (fixup2_kernel) */
#define MSQ_PLAN_PASS1 16       /* bit-packed bands the strip pass leaves (or all of them):
                                   pass1_kernel instead of ubits_kernel */

/* Build a plan.  nbands <= 0 picks a default (one band per SM, bands of
 * >= 64 rows, <= 65535 rows each).  Returns MSQ_EINVAL for unsupported
 * shapes (cols > 65536, rows >= 2^21, misaligned TMA-incompatible strides
 * are handled by the direct-load path, not rejected). */
int msq_plan_make(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld,
                  int32_t nbands, int32_t deterministic, msq_plan* plan);
/* Same with an engine choice: -1 = automatic (msq_plan_make), 0 = band
 * engine, 1 = register team engine (cols <= 1024; MSQ_EINVAL otherwise),
 * 2 = sieve engine (bit-packed, one matrix, rows and cols >= 64, row stride a
 * multiple of 16 bytes; automatic from 4096 x 4096). */
int msq_plan_make_ex(int32_t fmt, int32_t batch, int64_t rows, int64_t cols, int64_t ld,
                     int32_t nbands, int32_t deterministic, int32_t engine, msq_plan* plan);

/* Enqueue a solve on `stream`.  d_ws: >= plan->ws_bytes of device memory
 * (required for every plan with ws_bytes > 0, team-engine plans included);
 * d_result: plan->batch msq_devresult blocks (device memory).  Nothing is
 * synchronised; decode with msq_decode after the stream completes. */
int msq_launch(const msq_plan* plan, const void* d_src, void* d_ws, msq_devresult* d_result,
               void* stream);

/* Decode a (host copy of a) device result block. Returns MSQ_EVALUE if the
 * status flags an invalid cell. */
int msq_decode(const msq_devresult* r, int64_t rows, int64_t cols, msq_result* out);

/* Synchronous convenience calls (internal per-device workspace).  Single
 * matrices past the band engine's ranges (cols > 65536 or rows >= 2^21 - 1)
 * are solved by the row-parallel DP kernel (msq_dp_solve): same result, any
 * shape with rows * cols < 2^40. */
int msq_solve_u8(const uint8_t* d_cells, int64_t rows, int64_t cols, int64_t ld,
                 msq_result* out, void* stream);
int msq_solve_bits(const uint32_t* d_words, int64_t rows, int64_t cols, int64_t ld_words,
                   msq_result* out, void* stream);
int msq_solve_batch_u8(const uint8_t* d_cells, int64_t batch, int64_t rows, int64_t cols,
                       msq_result* out, void* stream);

/* Text ingest (grid.py:172-206 parse_matrix format: one '0'/'1' line per
 * row, '\n'-separated, trailing newline optional) on the device: d_text holds
 * nbytes of text, rows x cols as the caller derived them from the first line
 * (cols = its length, rows = lines).  Writes u8 cells (ld bytes per row) or
 * LSB-first packed words (ld words per row) to d_out.  On a malformed text
 * returns MSQ_EVALUE with *bad_line = the first (1-based) line that is ragged
 * or holds a character outside {'0','1'}: where the reference's sequential
 * parse raises RaggedRowsError / InvalidCharError. */
int msq_parse_text(const char* d_text, int64_t nbytes, int64_t rows, int64_t cols, int32_t fmt,
                   void* d_out, int64_t ld, int64_t* bad_line, void* stream);

/* Cube extension (cubes.py:92-125): one probe of max_cube's binary search.
 * d_vol: depth x rows x cols u8 voxels (depth-major, then row-major, the
 * reference's BinaryVolume layout); d_scratch: depth*rows*cols bytes.
 * *first_depth = the first depth d >= k-1 at which the depth-frequency matrix
 * holds a k x k window of values >= k (exists_cube_at_depth, cubes.py:75-89),
 * or -1.  The reference's probe reads (d+1)*rows*cols voxels when it finds one
 * at d, all of them otherwise.  MSQ_EVALUE for a voxel outside {0,1}. */
int msq_cube_probe(const uint8_t* d_vol, int64_t depth, int64_t rows, int64_t cols, int64_t k,
                   uint8_t* d_scratch, int64_t* first_depth, void* stream);

/* Histogram maximal rectangle (histogram.py:60-70 maximal_rectangle): the
 * largest all-ones rectangle of a u8 matrix as (area, height, width) of the
 * first largest rectangle in the reference's sweep order.  d_scratch holds
 * msq_max_rectangle_scratch_bytes(rows, cols) bytes; cols <= 65535. */
int64_t msq_max_rectangle_scratch_bytes(int64_t rows, int64_t cols);
int msq_max_rectangle_u8(const uint8_t* d_cells, int64_t rows, int64_t cols, int64_t ld, void* d_scratch,
                         int64_t* area, int64_t* height, int64_t* width, void* stream);

/* The three-way-min DP (dp_full, squares.py:142-171) over a batch of small
 * matrices (cols <= 256), one thread per matrix: the independent second
 * solver of the GPU verification campaigns (the reference's verify.py:32-37
 * runs dp_full beside freq_square).  Same result convention. */
int msq_dp_batch_u8(const uint8_t* d_cells, int64_t batch, int64_t rows, int64_t cols,
                    msq_result* out, void* stream);

/* The DP baselines on any shape (dp_full / dp_rows, squares.py:142-200) by the
 * row-parallel form dp[i][j] = min(h, w, dp[i-1][j-1] + 1) (msq_rowdp.cuh),
 * u8 or bit-packed input, rows * cols < 2^40.  Optional outputs for the traced
 * mode (freq_square_traced, squares.py:129-139): d_heights = [rows][cols]
 * uint32 column heights after each row (the reference's freq snapshots),
 * d_rowmax = [rows] int32 largest square ending in each row (found_max_width
 * after row i = max of rowmax[0..i]).  NULL skips them.  Synchronous. */
int msq_dp_solve(int32_t fmt, const void* d_src, int64_t rows, int64_t cols, int64_t ld,
                 uint32_t* d_heights, int32_t* d_rowmax, msq_result* out, void* stream);

/* brute_force_square (squares.py:203-249): one thread per anchor; out->
 * cells_visited = the reference's raw cell-read count.  rows*cols <= 2^24 (the
 * Python wrapper applies the reference's cap first).  Synchronous. */
int msq_brute_u8(const uint8_t* d_cells, int64_t rows, int64_t cols, int64_t ld, msq_result* out,
                 void* stream);

/* Host-buffer entry points: copy H2D on `stream`, solve, copy the result
 * back (the path a CPU caller of freq_square takes). */
int msq_solve_u8_host(const uint8_t* h_cells, int64_t rows, int64_t cols, int64_t ld,
                      msq_result* out, void* stream);
int msq_solve_bits_host(const uint32_t* h_words, int64_t rows, int64_t cols, int64_t ld_words,
                        msq_result* out, void* stream);
int msq_solve_batch_u8_host(const uint8_t* h_cells, int64_t batch, int64_t rows, int64_t cols,
                            msq_result* out, void* stream);
/* (Pageable host buffers are staged through pinned chunks by worker threads,
 * host copies overlapping the PCIe transfers; pinned ones are copied directly.) */

/* ---- row-band sharding across GPUs (one process per GPU) ----------------
 * A rank owns rows [row_base, row_base + plan->rows) of the global matrix.
 *   1. msq_rank_pass1   : band passes over the local rows (fills d_ws)
 *   2. msq_rank_summary : per column bottom run of the local slice
 *                         (uint32; == plan->rows means all ones)
 *   3. (caller) all-gather the summaries of all ranks
 *   4. msq_compose_carry: carry-in heights for this rank from the gathered
 *                         summaries of the ranks above it
 *   5. msq_rank_fixup   : data-free band-boundary fix-ups, including the top
 *                         boundary of the slice when d_base_carry != NULL
 *   6. (caller) all-reduce(max) of max(key_pass1, key_fix) over ranks      */
int msq_rank_pass1(const msq_plan* plan, const void* d_src, void* d_ws,
                   msq_devresult* d_result, void* stream);
int msq_rank_summary(const msq_plan* plan, const void* d_ws, uint32_t* d_summary, void* stream);
/* msq_rank_pass1 in two halves, so the ranks can pool their lower bounds:
 * msq_rank_seed resets d_result and runs the lower-bound seed over the local
 * rows (best side in d_result->best_side); the caller all-reduces(max)
 * best_side over the ranks in place; msq_rank_band_pass then runs the band
 * passes from that shared lower bound. */
int msq_rank_seed(const msq_plan* plan, const void* d_src, msq_devresult* d_result, void* stream);
int msq_rank_band_pass(const msq_plan* plan, const void* d_src, void* d_ws, msq_devresult* d_result,
                       void* stream);
int msq_compose_carry(const uint32_t* d_summaries, const int64_t* h_rank_rows, int32_t nranks,
                      int32_t rank, int64_t cols, uint32_t* d_base_carry, void* stream);
int msq_rank_fixup(const msq_plan* plan, void* d_ws, const uint32_t* d_base_carry,
                   msq_devresult* d_result, void* stream);
/* Sieve engine across ranks (plan->engine == 2): a rank passes its local rows
 * and, when it is not the first, the last halo_rows (a multiple of 8, <= 256;
 * 256 unless the rank above is shorter) rows of the rank above (d_halo,
 * halo_ld words per row).  Every square the sieve can report (side <= 222)
 * then lies inside the rows of the rank that holds its bottom row, so the only
 * exchange is that halo before the solve and the all-reduce(max) of the key
 * after it.  msq_rank_sieve = msq_rank_sieve_pass (the streaming kernel) +
 * msq_rank_sieve_finish (band-top block rows, exact candidate windows).
 * Status bit 1 on any rank, or bit 2 on some rank while the reduced key's side
 * is <= 62: all ranks run steps 1-6 above instead. */
int msq_rank_sieve(const msq_plan* plan, const void* d_src, const void* d_halo, int64_t halo_rows,
                   int64_t halo_ld, void* d_ws, msq_devresult* d_result, void* stream);
int msq_rank_sieve_pass(const msq_plan* plan, const void* d_src, const void* d_halo, int64_t halo_rows,
                        int64_t halo_ld, void* d_ws, msq_devresult* d_result, void* stream);
int msq_rank_sieve_finish(const msq_plan* plan, const void* d_src, const void* d_halo, int64_t halo_rows,
                          int64_t halo_ld, void* d_ws, msq_devresult* d_result, void* stream);
/* d_out[0] = max(key_pass1, key_fix), d_out[1] = 3 for an invalid cell, 2 when
 * the sieve could not decide (status bit 1), 1 when it found nothing above side
 * 62 in this rank's rows (bit 2), else 0: the two int64 the ranks all-reduce(max)
 * (one tiny kernel on `stream`). */
int msq_rank_key_status(const msq_devresult* d_result, int64_t* d_out, void* stream);

/* Intermediate outputs (tests): per band leading-ones depth e, bottom run b
 * (uint16 [nbands][words*32]) and all-ones masks (uint32 [nbands][words]),
 * pass-1 band keys (uint64 [nbands]); device pointers into d_ws. */
int msq_ws_views(const msq_plan* plan, void* d_ws, uint16_t** e, uint16_t** b, uint32_t** allones,
                 uint64_t** band_keys);

/* Seeded counter-hash matrix generator (bench / test inputs, not the hot
 * path): cell (i,j) = mix64(seed + (i*cols+j+1)*0x9E3779B97F4A7C15)>>11 < thr53. */
int msq_gen_hash(int32_t fmt, uint64_t seed, uint64_t thr53, int64_t row0, int64_t nrows,
                 int64_t cols, int64_t ld, void* d_out, void* stream);

/* Number of kernel launches the last msq_launch enqueued (instrumentation). */
int32_t msq_last_launch_count(void);

/* Debug instrumentation: when set, each pass-1 unit writes 16 uint64 phase
 * cycle counters to d_counters[unit*16..] (NULL disables; tools only). */
void msq_debug_set_profile(void* d_counters);

/* Instrumentation: the pageable-buffer staging of the host-buffer calls
 * (worker threads, pinned buffers per worker, bytes per buffer; workers <= 0 =
 * half the hardware threads).  Tools only; the defaults are the measured best. */
void msq_debug_set_staging(int32_t workers, int32_t buffers, int64_t chunk_bytes);
/* Instrumentation: consumer warps per CTA of the sieve engine's streaming pass (plans made after the call). */
void msq_debug_set_sieve_wpc(int32_t warps);
/* Tests: sweeps of the sieve engine's streaming pass (1..4; 0 = by the height: the coarse pass
 * and the verifier run beside the streaming pass from the second sweep on). */
void msq_debug_set_sieve_phases(int32_t phases);
/* Instrumentation: band height of the team engine's row-band mode (plans made after the call). */
void msq_debug_set_team_band_rows(int32_t rows);

const char* msq_strerror(int code);
/* Name and text of the last CUDA error seen by this thread ("" if none). */
const char* msq_last_cuda_error(void);
const char* msq_version(void);

#ifdef __cplusplus
}
#endif
#endif
