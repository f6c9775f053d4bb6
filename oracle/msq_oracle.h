/*
 * msq_oracle.h -- CPU ORACLE for the maximal-square hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2503_18974_b200/) links, loads or calls this code.  It is used by
 * tests/, by __graft_entry__.smoke() as the checker, and by bench.py's
 * cpu_baseline / --impl reference legs.
 *
 * It restates the reference algorithm of /root/reference/pkg/src/squarelab/
 * squares.py (_freq_core :68-114, dp_rows :174-200) in plain C, adds the
 * location the reference implies (the cell of the final threshold raise,
 * squares.py:93-97 == dp_full's first strict improvement, squares.py:168-169),
 * and restates the row-band decomposition that
 * the GPU kernels implement, so every intermediate the kernels produce can be
 * checked bit for bit.
 *
 * Parity pinning: tests/test_oracle.py checks this file against golden vectors
 * produced by importing the reference itself (tests/golden/make_golden.py).
 */
#ifndef MSQ_ORACLE_H
#define MSQ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t side;
    int64_t area;
    int64_t cells_visited;
    int64_t top;   /* -1 when side == 0 */
    int64_t left;  /* -1 when side == 0 */
} orc_result;

/* 64-bit result key: larger key = better answer (side, then smaller bottom
 * row, then smaller right column).  Same packing as the CUDA library. */
uint64_t orc_pack_key(int64_t side, int64_t bottom, int64_t right);
void orc_unpack_key(uint64_t key, int64_t* side, int64_t* bottom, int64_t* right);

/* Algorithm 1 (squares.py:68-114) on row-major bytes, ld = row stride. */
int orc_freq_u8(const uint8_t* cells, int64_t rows, int64_t cols, int64_t ld, orc_result* out);
/* Same on bit-packed rows: bit b of word w = column 32w+b, ld in words. */
int orc_freq_bits(const uint32_t* words, int64_t rows, int64_t cols, int64_t ld, orc_result* out);
/* Row-rolling DP (squares.py:174-200); location = first strict improvement. */
int orc_dp_u8(const uint8_t* cells, int64_t rows, int64_t cols, int64_t ld, orc_result* out);

/* Batched Algorithm 1 over `batch` stacked rows x cols matrices. */
int orc_freq_batch_u8(const uint8_t* cells, int64_t batch, int64_t rows, int64_t cols,
                      orc_result* out);

/* ---- band decomposition (P5/P6) ------------------------------------------
 * Pass 1: Algorithm 1 on rows [r0, r1) as a standalone matrix, starting with
 * found = t0 - 1.  Writes per column e[j] = leading-ones depth from the band
 * top (H if none), b[j] = bottom run (local height at r1-1), allones bitmask,
 * and the band key (0 if nothing was found at threshold >= t0).
 * fmt: 0 = u8 (ld bytes), 1 = bits (ld words). */
int orc_band_pass(const void* src, int fmt, int64_t ld, int64_t r0, int64_t r1, int64_t cols,
                  int64_t t0, uint16_t* e, uint16_t* b, uint32_t* allones, uint64_t* key);

/* Carry-in heights for band k: c[j] = true height of column j at row
 * r0(k)-1 (P5 composition over bands 0..k-1 starting from base[] (may be NULL
 * = zeros)).  bvec/allones are [nbands][cols] / [nbands][words]. */
int orc_band_carry(int64_t k, const int64_t* heights, const uint16_t* bvec,
                   const uint32_t* allones, int64_t cols, const uint32_t* base, uint32_t* c);

/* Data-free fix-up (P6): virtual rows d=1..H with heights (e_j>=d ? c_j+d : 0),
 * exact seeding at d=1, single-threshold rows after, stop at d >= threshold.
 * r0 = band top row (global) for the key. */
int orc_fixup(const uint32_t* c, const uint16_t* e, int64_t cols, int64_t H, int64_t r0,
              int64_t t0, uint64_t* key);

/* Whole-matrix solve through the band decomposition (nbands >= 1). */
int orc_solve_banded_mt(const void* src, int fmt, int64_t ld, int64_t rows, int64_t cols,
                        int64_t nbands, int64_t nthreads, orc_result* out);
int orc_solve_banded(const void* src, int fmt, int64_t ld, int64_t rows, int64_t cols,
                     int64_t nbands, orc_result* out);

/* ---- seeded counter-hash generator (cfg3/cfg4 inputs) --------------------
 * cell(i,j) = (mix64(seed + (i*cols+j+1)*golden) >> 11) < thr53. */
uint64_t orc_mix64(uint64_t z);
void orc_gen_hash_u8(uint64_t seed, uint64_t thr53, int64_t row0, int64_t nrows, int64_t cols,
                     uint8_t* out);
void orc_gen_hash_bits(uint64_t seed, uint64_t thr53, int64_t row0, int64_t nrows, int64_t cols,
                       int64_t ld_words, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
