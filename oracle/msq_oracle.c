/*
 * msq_oracle.c -- CPU ORACLE (test infrastructure only; see msq_oracle.h).
 *
 * Every function cites the reference line it restates.  This file is a plain
 * C restatement of the reference's published algorithm; it is the checker for
 * the CUDA library, never part of it.
 */
#include "msq_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define KEY_DIM_BITS 21
#define KEY_DIM_MASK ((1ULL << KEY_DIM_BITS) - 1ULL)

uint64_t orc_pack_key(int64_t side, int64_t bottom, int64_t right) {
    if (side <= 0) return 0;
    return ((uint64_t)side << (2 * KEY_DIM_BITS)) |
           ((KEY_DIM_MASK - (uint64_t)bottom) << KEY_DIM_BITS) |
           (KEY_DIM_MASK - (uint64_t)right);
}

void orc_unpack_key(uint64_t key, int64_t* side, int64_t* bottom, int64_t* right) {
    if (key == 0) { *side = 0; *bottom = -1; *right = -1; return; }
    *side = (int64_t)(key >> (2 * KEY_DIM_BITS));
    *bottom = (int64_t)(KEY_DIM_MASK - ((key >> KEY_DIM_BITS) & KEY_DIM_MASK));
    *right = (int64_t)(KEY_DIM_MASK - (key & KEY_DIM_MASK));
}

static void result_from_key(uint64_t key, int64_t rows, int64_t cols, orc_result* out) {
    int64_t side, bottom, right;
    orc_unpack_key(key, &side, &bottom, &right);
    out->side = side;
    out->area = side * side;
    out->cells_visited = rows * cols;
    out->top = side ? bottom - side + 1 : -1;
    out->left = side ? right - side + 1 : -1;
}

/* Row fetch into a byte buffer: fmt 0 = bytes, fmt 1 = LSB-first bit words. */
static inline void fetch_row(const void* src, int fmt, int64_t ld, int64_t i, int64_t cols,
                             uint8_t* buf) {
    if (fmt == 0) {
        memcpy(buf, (const uint8_t*)src + i * ld, (size_t)cols);
    } else {
        const uint32_t* w = (const uint32_t*)src + i * ld;
        for (int64_t j = 0; j < cols; ++j) buf[j] = (uint8_t)((w[j >> 5] >> (j & 31)) & 1u);
    }
}

/*
 * Algorithm 1, restated from squares.py:68-114 (_freq_core):
 *   freq[j] += 1 on a one, reset on a zero (:88-90, :100-101);
 *   counter counts consecutive columns with freq >= check_max_height (:91-92);
 *   counter == check_max_width confirms a square, both thresholds grow,
 *   counter resets and the trailing reset is skipped (:93-99);
 *   counter resets on a miss and at each row end (:102-103).
 * Location: the cell (i, j) of the last confirmation (:93-97), i.e. the bottom
 * row / right column of the first maximal square in row-major order.
 * `found0` seeds found_max_width (the band pass starts at t0 - 1; 0 = plain).
 * Returns the packed key of the last confirmation (0 if none).
 */
static uint64_t freq_core(const void* src, int fmt, int64_t ld, int64_t r0, int64_t r1,
                          int64_t cols, int64_t found0, int64_t* freq, uint8_t* buf,
                          int64_t* found_out, int64_t* last_ij) {
    int64_t found = found0;
    int64_t check_w = found0 + 1, check_h = found0 + 1;
    int64_t counter = 0;
    uint64_t key = 0;
    for (int64_t i = r0; i < r1; ++i) {
        fetch_row(src, fmt, ld, i, cols, buf);
        for (int64_t j = 0; j < cols; ++j) {
            if (buf[j]) {
                int64_t f = freq[j] + 1;
                freq[j] = f;
                if (check_h <= f) {
                    counter += 1;
                    if (check_w == counter) {
                        found += 1;
                        check_w += 1;
                        check_h += 1;
                        counter = 0;
                        key = orc_pack_key(found, i, j);
                        if (last_ij) { last_ij[0] = i; last_ij[1] = j; }
                    }
                    continue; /* a satisfied column skips the trailing reset */
                }
            } else {
                freq[j] = 0;
            }
            counter = 0;
        }
        counter = 0;
    }
    if (found_out) *found_out = found;
    return key;
}

static int solve_freq(const void* src, int fmt, int64_t ld, int64_t rows, int64_t cols,
                      orc_result* out) {
    if (rows < 0 || cols < 0 || (rows == 0 && cols != 0)) return 1;
    if (rows == 0 || cols == 0) { /* squares.py:74-75 */
        out->side = out->area = out->cells_visited = 0;
        out->top = out->left = -1;
        return 0;
    }
    int64_t* freq = (int64_t*)calloc((size_t)cols, sizeof(int64_t));
    uint8_t* buf = (uint8_t*)malloc((size_t)cols);
    if (!freq || !buf) { free(freq); free(buf); return 2; }
    /* the location is kept unpacked: any shape (the key packs 21-bit rows) */
    int64_t found = 0, ij[2] = {-1, -1};
    freq_core(src, fmt, ld, 0, rows, cols, 0, freq, buf, &found, ij);
    free(freq);
    free(buf);
    out->side = found;
    out->area = found * found;
    out->cells_visited = rows * cols;
    out->top = found ? ij[0] - found + 1 : -1;
    out->left = found ? ij[1] - found + 1 : -1;
    return 0;
}

int orc_freq_u8(const uint8_t* cells, int64_t rows, int64_t cols, int64_t ld, orc_result* out) {
    return solve_freq(cells, 0, ld, rows, cols, out);
}

int orc_freq_bits(const uint32_t* words, int64_t rows, int64_t cols, int64_t ld,
                  orc_result* out) {
    return solve_freq(words, 1, ld, rows, cols, out);
}

int orc_freq_batch_u8(const uint8_t* cells, int64_t batch, int64_t rows, int64_t cols,
                      orc_result* out) {
    for (int64_t k = 0; k < batch; ++k) {
        int rc = orc_freq_u8(cells + k * rows * cols, rows, cols, cols, out + k);
        if (rc) return rc;
    }
    return 0;
}

/*
 * Row-rolling DP, restated from squares.py:174-200 (same recurrence as
 * dp_full :142-171): v = min(up, left, diag) + 1 on ones, border cells = 1;
 * best updated on strict v > best (:168-169 / :195-196) -> first maximal cell
 * in row-major order is the location.
 */
int orc_dp_u8(const uint8_t* cells, int64_t rows, int64_t cols, int64_t ld, orc_result* out) {
    if (rows < 0 || cols < 0 || (rows == 0 && cols != 0)) return 1;
    if (rows == 0 || cols == 0) {
        out->side = out->area = out->cells_visited = 0;
        out->top = out->left = -1;
        return 0;
    }
    int64_t* prev = (int64_t*)calloc((size_t)cols, sizeof(int64_t));
    int64_t* cur = (int64_t*)calloc((size_t)cols, sizeof(int64_t));
    if (!prev || !cur) { free(prev); free(cur); return 2; }
    int64_t best = 0, bi = -1, bj = -1;
    for (int64_t i = 0; i < rows; ++i) {
        const uint8_t* row = cells + i * ld;
        for (int64_t j = 0; j < cols; ++j) {
            if (row[j]) {
                int64_t v;
                if (i == 0 || j == 0) {
                    v = 1;
                } else {
                    int64_t m = prev[j];
                    if (cur[j - 1] < m) m = cur[j - 1];
                    if (prev[j - 1] < m) m = prev[j - 1];
                    v = m + 1;
                }
                cur[j] = v;
                if (v > best) { best = v; bi = i; bj = j; }
            } else {
                cur[j] = 0;
            }
        }
        int64_t* t = prev; prev = cur; cur = t;
    }
    free(prev);
    free(cur);
    out->side = best;
    out->area = best * best;
    out->cells_visited = rows * cols;
    out->top = best ? bi - best + 1 : -1;
    out->left = best ? bj - best + 1 : -1;
    return 0;
}

/*
 * P6 pass 1: Algorithm 1 on the band as a standalone matrix.
 * Starting at found = t0-1 stays exact because the band-local g(r0-1) = 0 and
 * g(i) <= g(i-1)+1 (P2), so one confirmation per row suffices.
 */
int orc_band_pass(const void* src, int fmt, int64_t ld, int64_t r0, int64_t r1, int64_t cols,
                  int64_t t0, uint16_t* e, uint16_t* b, uint32_t* allones, uint64_t* key) {
    int64_t H = r1 - r0;
    if (H <= 0 || H > 65535 || cols <= 0 || t0 < 1) return 1;
    int64_t* freq = (int64_t*)calloc((size_t)cols, sizeof(int64_t));
    uint8_t* buf = (uint8_t*)malloc((size_t)cols);
    int64_t* first0 = (int64_t*)malloc((size_t)cols * sizeof(int64_t));
    if (!freq || !buf || !first0) { free(freq); free(buf); free(first0); return 2; }
    for (int64_t j = 0; j < cols; ++j) first0[j] = H;
    /* leading-ones depth needs a second look at the rows; do it alongside */
    *key = freq_core(src, fmt, ld, r0, r1, cols, t0 - 1, freq, buf, NULL, NULL);
    for (int64_t i = r0; i < r1; ++i) {
        fetch_row(src, fmt, ld, i, cols, buf);
        for (int64_t j = 0; j < cols; ++j)
            if (!buf[j] && first0[j] == H) first0[j] = i - r0;
    }
    int64_t words = (cols + 31) / 32;
    memset(allones, 0, (size_t)words * sizeof(uint32_t));
    for (int64_t j = 0; j < cols; ++j) {
        e[j] = (uint16_t)first0[j];
        b[j] = (uint16_t)freq[j];
        if (freq[j] == H) allones[j >> 5] |= 1u << (j & 31);
    }
    free(freq);
    free(buf);
    free(first0);
    return 0;
}

/* P5: (b1,f1) o (b2,f2) = (f2 ? b1 + len2 : b2, f1 & f2), folded top-down. */
int orc_band_carry(int64_t k, const int64_t* heights, const uint16_t* bvec,
                   const uint32_t* allones, int64_t cols, const uint32_t* base, uint32_t* c) {
    int64_t words = (cols + 31) / 32;
    for (int64_t j = 0; j < cols; ++j) {
        uint64_t h = base ? base[j] : 0;
        for (int64_t q = 0; q < k; ++q) {
            int full = (allones[q * words + (j >> 5)] >> (j & 31)) & 1u;
            h = full ? h + (uint64_t)heights[q] : bvec[q * cols + j];
        }
        c[j] = h > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)h;
    }
    return 0;
}

/* virtual height of column j at depth d (P6) */
static inline int64_t vheight(const uint32_t* c, const uint16_t* e, int64_t j, int64_t d) {
    return (int64_t)e[j] >= d ? (int64_t)c[j] + d : 0;
}

/* first column closing a window of k consecutive virtual heights >= k, or -1 */
static int64_t vfirst_window(const uint32_t* c, const uint16_t* e, int64_t cols, int64_t d,
                             int64_t k) {
    int64_t run = 0;
    for (int64_t j = 0; j < cols; ++j) {
        if (vheight(c, e, j, d) >= k) {
            if (++run >= k) return j;
        } else {
            run = 0;
        }
    }
    return -1;
}

/*
 * P6 fix-up: Algorithm 1 on the virtual band top.  At d = 1 the running
 * maximum is seeded exactly (P3: the window test is monotone in k), because
 * g(r0-1) of the rows above is not bounded by t0.  From d = 2 on one test per
 * row at found+1 is exact (P2); stop at the first d >= found+1 (no crossing
 * square of a larger side can end deeper).
 */
int orc_fixup(const uint32_t* c, const uint16_t* e, int64_t cols, int64_t H, int64_t r0,
              int64_t t0, uint64_t* key) {
    *key = 0;
    if (H <= 0 || cols <= 0 || t0 < 1) return H <= 0 ? 0 : 1;
    int64_t found = t0 - 1;
    /* d = 1: exact seeding */
    int64_t j = vfirst_window(c, e, cols, 1, found + 1);
    if (j >= 0) {
        int64_t k = found + 1, jk = j;
        for (;;) {
            int64_t j2 = vfirst_window(c, e, cols, 1, k + 1);
            if (j2 < 0) break;
            k += 1;
            jk = j2;
        }
        found = k;
        *key = orc_pack_key(found, r0, jk);
    }
    for (int64_t d = 2; d <= H && d < found + 1; ++d) {
        /* Algorithm 1 row (squares.py:86-103) on virtual heights */
        int64_t t = found + 1, counter = 0;
        for (int64_t jj = 0; jj < cols; ++jj) {
            if (vheight(c, e, jj, d) >= t) {
                counter += 1;
                if (counter == t) {
                    found += 1;
                    *key = orc_pack_key(found, r0 + d - 1, jj);
                    t += 1;
                    counter = 0;
                }
            } else {
                counter = 0;
            }
        }
    }
    return 0;
}

int orc_solve_banded(const void* src, int fmt, int64_t ld, int64_t rows, int64_t cols,
                     int64_t nbands, orc_result* out) {
    if (rows == 0 || cols == 0) return solve_freq(src, fmt, ld, rows, cols, out);
    if (nbands < 1) return 1;
    if (nbands > rows) nbands = rows;
    int64_t words = (cols + 31) / 32;
    int64_t* hts = (int64_t*)malloc((size_t)nbands * sizeof(int64_t));
    int64_t* r0s = (int64_t*)malloc((size_t)nbands * sizeof(int64_t));
    uint16_t* e = (uint16_t*)malloc((size_t)(nbands * cols) * sizeof(uint16_t));
    uint16_t* b = (uint16_t*)malloc((size_t)(nbands * cols) * sizeof(uint16_t));
    uint32_t* ao = (uint32_t*)malloc((size_t)(nbands * words) * sizeof(uint32_t));
    uint32_t* c = (uint32_t*)malloc((size_t)cols * sizeof(uint32_t));
    uint64_t* keys = (uint64_t*)calloc((size_t)nbands, sizeof(uint64_t));
    int rc = 0;
    if (!hts || !r0s || !e || !b || !ao || !c || !keys) { rc = 2; goto done; }
    uint64_t best = 0;
    for (int64_t k = 0; k < nbands; ++k) {
        r0s[k] = rows * k / nbands;
        hts[k] = rows * (k + 1) / nbands - r0s[k];
        rc = orc_band_pass(src, fmt, ld, r0s[k], r0s[k] + hts[k], cols, 1, e + k * cols,
                           b + k * cols, ao + k * words, &keys[k]);
        if (rc) goto done;
        if (keys[k] > best) best = keys[k];
    }
    int64_t g = (int64_t)(best >> (2 * KEY_DIM_BITS));
    for (int64_t k = 1; k < nbands; ++k) {
        orc_band_carry(k, hts, b, ao, cols, NULL, c);
        uint64_t fk;
        rc = orc_fixup(c, e + k * cols, cols, hts[k], r0s[k], g > 0 ? g : 1, &fk);
        if (rc) goto done;
        if (fk > best) best = fk;
    }
    result_from_key(best, rows, cols, out);
done:
    free(hts); free(r0s); free(e); free(b); free(ao); free(c); free(keys);
    return rc;
}

/*
 * All-core variant for the benchmark's CPU arm: the same band algebra as
 * orc_solve_banded (Algorithm 1 per row band, P5 carry fold, P6 fix-up), the
 * band passes and the fix-ups spread over `nthreads` POSIX threads, the carry
 * fold sequential (O(nbands * cols)).  Whole-matrix exact.
 */
typedef struct {
    const void* src; int fmt; int64_t ld, cols, words, nbands, nthreads, tid;
    const int64_t* r0s; const int64_t* hts;
    uint16_t* e; uint16_t* b; uint32_t* ao; uint32_t* carry; uint64_t* keys; uint64_t* fkeys;
    int64_t g; int phase; int rc;
} mt_job;

static void* mt_worker(void* arg) {
    mt_job* j = (mt_job*)arg;
    for (int64_t k = j->tid; k < j->nbands; k += j->nthreads) {
        if (j->phase == 0) {
            int rc = orc_band_pass(j->src, j->fmt, j->ld, j->r0s[k], j->r0s[k] + j->hts[k], j->cols, 1,
                                   j->e + k * j->cols, j->b + k * j->cols, j->ao + k * j->words, &j->keys[k]);
            if (rc) j->rc = rc;
        } else if (k > 0) {
            int rc = orc_fixup(j->carry + k * j->cols, j->e + k * j->cols, j->cols, j->hts[k], j->r0s[k],
                               j->g > 0 ? j->g : 1, &j->fkeys[k]);
            if (rc) j->rc = rc;
        }
    }
    return NULL;
}

int orc_solve_banded_mt(const void* src, int fmt, int64_t ld, int64_t rows, int64_t cols,
                        int64_t nbands, int64_t nthreads, orc_result* out) {
    if (rows == 0 || cols == 0) return solve_freq(src, fmt, ld, rows, cols, out);
    if (nbands < 1 || nthreads < 1) return 1;
    if (nbands > rows) nbands = rows;
    if (nthreads > nbands) nthreads = nbands;
    const int64_t words = (cols + 31) / 32;
    int64_t* hts = (int64_t*)malloc((size_t)nbands * sizeof(int64_t));
    int64_t* r0s = (int64_t*)malloc((size_t)nbands * sizeof(int64_t));
    uint16_t* e = (uint16_t*)malloc((size_t)(nbands * cols) * sizeof(uint16_t));
    uint16_t* b = (uint16_t*)malloc((size_t)(nbands * cols) * sizeof(uint16_t));
    uint32_t* ao = (uint32_t*)malloc((size_t)(nbands * words) * sizeof(uint32_t));
    uint32_t* carry = (uint32_t*)calloc((size_t)(nbands * cols), sizeof(uint32_t));
    uint64_t* keys = (uint64_t*)calloc((size_t)nbands, sizeof(uint64_t));
    uint64_t* fkeys = (uint64_t*)calloc((size_t)nbands, sizeof(uint64_t));
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    int rc = 0;
    if (!hts || !r0s || !e || !b || !ao || !carry || !keys || !fkeys || !jobs || !th) { rc = 2; goto done; }
    for (int64_t k = 0; k < nbands; ++k) {
        r0s[k] = rows * k / nbands;
        hts[k] = rows * (k + 1) / nbands - r0s[k];
    }
    for (int phase = 0; phase < 2; ++phase) {
        uint64_t best = 0;
        if (phase == 1) {
            for (int64_t k = 0; k < nbands; ++k) if (keys[k] > best) best = keys[k];
            /* P5 fold: carry_k = f_{k-1} ? carry_{k-1} + H_{k-1} : b_{k-1} */
            for (int64_t k = 1; k < nbands; ++k)
                for (int64_t jj = 0; jj < cols; ++jj) {
                    const int full = (ao[(k - 1) * words + (jj >> 5)] >> (jj & 31)) & 1u;
                    const uint64_t h = full ? (uint64_t)carry[(k - 1) * cols + jj] + (uint64_t)hts[k - 1]
                                            : (uint64_t)b[(k - 1) * cols + jj];
                    carry[k * cols + jj] = h > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)h;
                }
        }
        for (int64_t t = 0; t < nthreads; ++t) {
            mt_job* j = &jobs[t];
            j->src = src; j->fmt = fmt; j->ld = ld; j->cols = cols; j->words = words;
            j->nbands = nbands; j->nthreads = nthreads; j->tid = t; j->r0s = r0s; j->hts = hts;
            j->e = e; j->b = b; j->ao = ao; j->carry = carry; j->keys = keys; j->fkeys = fkeys;
            j->g = (int64_t)(best >> (2 * KEY_DIM_BITS)); j->phase = phase;
            if (pthread_create(&th[t], NULL, mt_worker, j)) { rc = 3; goto done; }
        }
        for (int64_t t = 0; t < nthreads; ++t) {
            pthread_join(th[t], NULL);
            if (jobs[t].rc) rc = jobs[t].rc;
        }
        if (rc) goto done;
    }
    {
        uint64_t best = 0;
        for (int64_t k = 0; k < nbands; ++k) {
            if (keys[k] > best) best = keys[k];
            if (fkeys[k] > best) best = fkeys[k];
        }
        result_from_key(best, rows, cols, out);
    }
done:
    free(hts); free(r0s); free(e); free(b); free(ao); free(carry); free(keys); free(fkeys);
    free(jobs); free(th);
    return rc;
}

/* ---- seeded counter-hash generator -------------------------------------- */
uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline int hash_cell(uint64_t seed, uint64_t thr53, uint64_t idx) {
    return (orc_mix64(seed + (idx + 1ULL) * 0x9E3779B97F4A7C15ULL) >> 11) < thr53;
}

void orc_gen_hash_u8(uint64_t seed, uint64_t thr53, int64_t row0, int64_t nrows, int64_t cols,
                     uint8_t* out) {
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t j = 0; j < cols; ++j)
            out[i * cols + j] = (uint8_t)hash_cell(seed, thr53, (uint64_t)((row0 + i) * cols + j));
}

void orc_gen_hash_bits(uint64_t seed, uint64_t thr53, int64_t row0, int64_t nrows, int64_t cols,
                       int64_t ld_words, uint32_t* out) {
    for (int64_t i = 0; i < nrows; ++i) {
        uint32_t* w = out + i * ld_words;
        memset(w, 0, (size_t)ld_words * sizeof(uint32_t));
        for (int64_t j = 0; j < cols; ++j)
            if (hash_cell(seed, thr53, (uint64_t)((row0 + i) * cols + j)))
                w[j >> 5] |= 1u << (j & 31);
    }
}
