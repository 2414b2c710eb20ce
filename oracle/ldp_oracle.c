/*
 * ldp_oracle.c -- CPU restatement of the reference's LDP path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the B200
 * kernels. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it; the product path (paper_1810_11518_b200)
 * never links or calls it.
 *
 * Every function restates one reference function (paths relative to the
 * reference tree, proj/...):
 *   oracle_make_random      src/image.cpp:75-83      (std::mt19937, low byte)
 *   oracle_sample           src/image.cpp:36-40      (clamp-to-edge)
 *   oracle_responses        src/kirsch.cpp:63-84     (naive 3x3 dot products)
 *                           masks: src/kirsch.cpp:10-29 (ring + base ring)
 *   oracle_ldp_code         src/descriptors.cpp:83-102 (k selection passes,
 *                           strict '>' so the lowest direction wins ties)
 *   oracle_bin_index        src/descriptors.cpp:25-45,104-106 (ascending
 *                           rank among popcount-k codes; the reference only
 *                           defines k == 3 -- k != 3 is this repo's extension)
 *   oracle_code_map         the per-pixel loop of src/descriptors.cpp:129-136
 *   oracle_histogram        src/descriptors.cpp:123-139
 *   oracle_cell_histograms  src/windowing.cpp:8-19,35-63 (floor grid, each
 *                           cell clamped as its own image, row-major cells);
 *                           rectangular cells are this repo's extension.
 *   oracle_lbp_code         src/descriptors.cpp:141-157 (k == 0 selects LBP
 *                           in the map/histogram/batch functions: bit i set
 *                           when ring neighbour i >= the centre, 256 bins
 *                           indexed by the code, descriptors.cpp:159-168)
 *
 * Parity pins: tests/test_oracle.py checks this file against the reference's
 * golden fixtures (tests/golden/, converted by tests/golden/make_golden.py)
 * and against the reference library itself compiled into oracle/_ref/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* Ring positions clockwise from the top-left neighbour (kirsch.cpp:11-12). */
static const int kRing[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, 1},
                                {1, 1},   {1, 0},  {1, -1}, {0, -1}};
/* Mask 0's ring weights; mask i at ring slot j is kBase[(j + i) % 8]
 * (kirsch.cpp:15,25). */
static const int kBase[8] = {-3, -3, 5, 5, 5, -3, -3, -3};

static int g_masks[8][3][3];
static int g_masks_ready = 0;

static void build_masks(void) {
    if (g_masks_ready) return;
    for (int i = 0; i < 8; ++i) {
        g_masks[i][1][1] = 0;
        for (int j = 0; j < 8; ++j)
            g_masks[i][kRing[j][0] + 1][kRing[j][1] + 1] = kBase[(j + i) % 8];
    }
    g_masks_ready = 1;
}

/* ---- std::mt19937 (image.cpp:75-83 uses its low 8 bits per pixel) ---- */
typedef struct { uint32_t mt[624]; int idx; } mt19937;

static void mt_seed(mt19937* s, uint32_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
    s->idx = 624;
}

static uint32_t mt_next(mt19937* s) {
    if (s->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            uint32_t y = (s->mt[i] & 0x80000000u) | (s->mt[(i + 1) % 624] & 0x7fffffffu);
            s->mt[i] = s->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        s->idx = 0;
    }
    uint32_t y = s->mt[s->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

void oracle_make_random(int rows, int cols, uint32_t seed, uint8_t* out) {
    mt19937 s;
    mt_seed(&s, seed);
    const size_t n = (size_t)rows * (size_t)cols;
    for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)(mt_next(&s) & 0xFFu);
}

/* ---- sampling / responses ---- */
static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Clamp-to-edge inside the window [x0, x0+rows) x [y0, y0+cols) of an image
 * with row pitch `pitch` (image.cpp:36-40; a window is a cropped image,
 * windowing.cpp:21-33,42). */
static inline int sample_win(const uint8_t* px, int pitch, int x0, int y0, int rows,
                             int cols, int x, int y) {
    const int cx = clampi(x, x0, x0 + rows - 1);
    const int cy = clampi(y, y0, y0 + cols - 1);
    return px[(size_t)cx * (size_t)pitch + (size_t)cy];
}

int oracle_sample(const uint8_t* px, int rows, int cols, int x, int y) {
    return sample_win(px, cols, 0, 0, rows, cols, x, y);
}

static void responses_win(const uint8_t* px, int pitch, int x0, int y0, int rows, int cols,
                          int x, int y, int m[8]) {
    build_masks();
    int nb[3][3];
    for (int k = -1; k <= 1; ++k)
        for (int l = -1; l <= 1; ++l)
            nb[k + 1][l + 1] = sample_win(px, pitch, x0, y0, rows, cols, x + k, y + l);
    for (int i = 0; i < 8; ++i) {
        int acc = 0;
        for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l) acc += g_masks[i][k][l] * nb[k][l];
        m[i] = acc;
    }
}

/* kirsch.cpp:63-84: eight signed responses at (x, y), clamped borders. */
void oracle_responses(const uint8_t* px, int rows, int cols, int x, int y, int32_t* out8) {
    int m[8];
    responses_win(px, cols, 0, 0, rows, cols, x, y, m);
    for (int i = 0; i < 8; ++i) out8[i] = m[i];
}

/* descriptors.cpp:83-102: k passes, each picks the largest unused response
 * with strict '>', so ties keep the lowest direction index. Returns -1 for
 * k outside [1, 7] (the reference throws std::invalid_argument). */
int oracle_ldp_code(const int32_t* m, int k) {
    if (k < 1 || k > 7) return -1;
    int used[8] = {0};
    unsigned code = 0;
    for (int picked = 0; picked < k; ++picked) {
        int best = -1;
        for (int i = 0; i < 8; ++i)
            if (!used[i] && (best < 0 || m[i] > m[best])) best = i;
        used[best] = 1;
        code |= 1u << best;
    }
    return (int)code;
}

static int popcount8(unsigned c) {
    int n = 0;
    for (int b = 0; b < 8; ++b) n += (c >> b) & 1u;
    return n;
}

/* descriptors.cpp:25-45,104-106: rank of `code` among the codes with the same
 * popcount k, ascending by value; -1 if popcount(code) != k. */
int oracle_bin_index(int code, int k) {
    if (k == 0) return (code >= 0 && code <= 255) ? code : -1;
    if (code < 0 || code > 255 || popcount8((unsigned)code) != k) return -1;
    int rank = 0;
    for (int c = 0; c < code; ++c)
        if (popcount8((unsigned)c) == k) ++rank;
    return rank;
}

/* C(8, k): number of bins for popcount-k codes (56 for k = 3); 256 for
 * k == 0 (LBP). */
int oracle_n_bins(int k) {
    if (k == 0) return 256;
    if (k < 1 || k > 7) return -1;
    int n = 0;
    for (int c = 0; c < 256; ++c) n += popcount8((unsigned)c) == k;
    return n;
}

/* descriptors.cpp:141-157: bit i set when ring neighbour i >= the centre. */
static int lbp_win(const uint8_t* px, int pitch, int x0, int y0, int rows, int cols, int x, int y) {
    const int centre = sample_win(px, pitch, x0, y0, rows, cols, x, y);
    int code = 0;
    for (int i = 0; i < 8; ++i)
        if (sample_win(px, pitch, x0, y0, rows, cols, x + kRing[i][0], y + kRing[i][1]) >= centre)
            code |= 1 << i;
    return code;
}

int oracle_lbp_code(const uint8_t* px, int rows, int cols, int x, int y) {
    return lbp_win(px, cols, 0, 0, rows, cols, x, y);
}

static int code_win(const uint8_t* px, int pitch, int x0, int y0, int rows, int cols, int x,
                    int y, int k) {
    if (k == 0) return lbp_win(px, pitch, x0, y0, rows, cols, x, y);
    int m[8];
    responses_win(px, pitch, x0, y0, rows, cols, x, y, m);
    return oracle_ldp_code(m, k);
}

/* The per-pixel code of descriptors.cpp:129-136 written out as a map:
 * codes[x * cols + y] = ldp_code(responses(img, x, y), k). Image clamp. */
int oracle_code_map(const uint8_t* px, int rows, int cols, int k, uint8_t* codes) {
    if (k < 0 || k > 7 || rows < 3 || cols < 3) return -1;
    for (int x = 0; x < rows; ++x)
        for (int y = 0; y < cols; ++y)
            codes[(size_t)x * cols + y] = (uint8_t)code_win(px, cols, 0, 0, rows, cols, x, y, k);
    return 0;
}

/* One histogram over a window (an independent image with its own clamp). */
static void hist_win(const uint8_t* px, int pitch, int x0, int y0, int rows, int cols, int k,
                     const int* rank, uint64_t* hist) {
    for (int x = x0; x < x0 + rows; ++x)
        for (int y = y0; y < y0 + cols; ++y)
            ++hist[rank[code_win(px, pitch, x0, y0, rows, cols, x, y, k)]];
}

static void rank_table(int k, int* rank) {
    for (int c = 0; c < 256; ++c) rank[c] = oracle_bin_index(c, k);
}

/* descriptors.cpp:123-139 (k == 3 there; any k in [1,7] here, C(8,k) bins). */
int oracle_histogram(const uint8_t* px, int rows, int cols, int k, uint64_t* hist) {
    if (k < 0 || k > 7 || rows < 3 || cols < 3) return -1;
    int rank[256];
    rank_table(k, rank);
    memset(hist, 0, sizeof(uint64_t) * (size_t)oracle_n_bins(k));
    hist_win(px, cols, 0, 0, rows, cols, k, rank, hist);
    return 0;
}

/* windowing.cpp:8-19,35-63 generalised to cell_rows x cell_cols cells:
 * grid = floor(rows / cell_rows) x floor(cols / cell_cols), remainder
 * dropped, cells row-major, each cell clamped as an independent image.
 * hist is [grid_rows * grid_cols][n_bins]. Returns the number of cells, or
 * -1 on invalid arguments (window < 3 or larger than the image throws in
 * make_grid, windowing.cpp:9-17). */
int oracle_cell_histograms(const uint8_t* px, int rows, int cols, int cell_rows,
                           int cell_cols, int k, uint64_t* hist) {
    if (k < 0 || k > 7 || rows < 3 || cols < 3) return -1;
    if (cell_rows < 3 || cell_cols < 3 || cell_rows > rows || cell_cols > cols) return -1;
    const int gr = rows / cell_rows, gc = cols / cell_cols, nb = oracle_n_bins(k);
    int rank[256];
    rank_table(k, rank);
    memset(hist, 0, sizeof(uint64_t) * (size_t)gr * gc * nb);
    for (int r = 0; r < gr; ++r)
        for (int c = 0; c < gc; ++c)
            hist_win(px, cols, r * cell_rows, c * cell_cols, cell_rows, cell_cols, k, rank,
                     hist + ((size_t)r * gc + c) * nb);
    return gr * gc;
}

/* ---- threaded batch driver (CPU baseline "port" leg and fast parity) ----
 * Images are independent (SPEC: functions are pure), so a batch shards by
 * image over `threads` POSIX threads. pixels: n x rows x cols contiguous;
 * codes (nullable): same layout; hist (nullable): n x cells x n_bins (u64).
 * cell_rows == 0 means one whole-image histogram per image. */
typedef struct {
    const uint8_t* px; int rows, cols, k, cell_rows, cell_cols;
    uint8_t* codes; uint64_t* hist; int64_t first, last; int cells, nb;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* j = (batch_job*)arg;
    const size_t plane = (size_t)j->rows * (size_t)j->cols;
    for (int64_t i = j->first; i < j->last; ++i) {
        const uint8_t* img = j->px + (size_t)i * plane;
        if (j->codes) oracle_code_map(img, j->rows, j->cols, j->k, j->codes + (size_t)i * plane);
        if (j->hist) {
            uint64_t* h = j->hist + (size_t)i * (size_t)j->cells * (size_t)j->nb;
            if (j->cell_rows == 0) oracle_histogram(img, j->rows, j->cols, j->k, h);
            else oracle_cell_histograms(img, j->rows, j->cols, j->cell_rows, j->cell_cols, j->k, h);
        }
    }
    return NULL;
}

int oracle_batch(const uint8_t* px, int64_t n, int rows, int cols, int k, int cell_rows,
                 int cell_cols, uint8_t* codes, uint64_t* hist, int threads) {
    if (k < 0 || k > 7 || rows < 3 || cols < 3 || n < 0) return -1;
    int cells = 1;
    if (cell_rows != 0) {
        if (cell_rows < 3 || cell_cols < 3 || cell_rows > rows || cell_cols > cols) return -1;
        cells = (rows / cell_rows) * (cols / cell_cols);
    }
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if ((int64_t)threads > n) threads = (int)(n > 0 ? n : 1);
    pthread_t tid[256];
    batch_job jobs[256];
    build_masks();
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (batch_job){px, rows, cols, k, cell_rows, cell_cols, codes, hist,
                              n * t / threads, n * (t + 1) / threads, cells, oracle_n_bins(k)};
        pthread_create(&tid[t], NULL, batch_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    return 0;
}

/* ---- column terms and the equivalence sweep ----
 * oracle_column_terms      src/kirsch.cpp:86-138 (fifteen signed column
 *                          partial sums; the centre weight is zero)
 * oracle_responses_terms   src/kirsch.cpp:140-157 (kResponseTerms: each
 *                          response is the sum of three column terms)
 * oracle_verify_image      src/verify.cpp:37-61
 * oracle_verify_equivalence src/verify.cpp:19-33,63-111 (corpus from one
 *                          mt19937; threads only shape the chunked
 *                          bookkeeping, run sequentially here)            */

/* term n: column offset dy and weights for rows x-1, x, x+1 */
static const int kTermCol[15] = {-1, 0, 1, 0, 1, -1, 1, -1, 1, -1, -1, 0, -1, 1, 1};
static const int kTermW[15][3] = {
    {-3, -3, -3}, {-3, 0, -3}, {5, 5, 5},    {5, 0, -3},   {5, 5, -3},
    {5, -3, -3},  {5, -3, -3}, {5, 5, -3},   {-3, -3, -3}, {5, 5, 5},
    {-3, 5, 5},   {-3, 0, 5},  {-3, -3, 5},  {-3, -3, 5},  {-3, 5, 5},
};
static const int kResponseTerms[8][3] = {{0, 1, 2},  {0, 3, 4},   {5, 3, 6},    {7, 3, 8},
                                         {9, 1, 8},  {10, 11, 8}, {12, 11, 13}, {0, 11, 14}};

void oracle_column_terms(const uint8_t* px, int rows, int cols, int x, int y, int32_t* a15) {
    for (int n = 0; n < 15; ++n) {
        int acc = 0;
        for (int k = 0; k < 3; ++k)
            acc += kTermW[n][k] * sample_win(px, cols, 0, 0, rows, cols, x + k - 1, y + kTermCol[n]);
        a15[n] = acc;
    }
}

void oracle_responses_terms(const int32_t* a15, int32_t* out8) {
    for (int i = 0; i < 8; ++i)
        out8[i] = a15[kResponseTerms[i][0]] + a15[kResponseTerms[i][1]] + a15[kResponseTerms[i][2]];
}

typedef struct {
    uint64_t images_checked, pixels_checked;
    int has_mismatch, image_index, x, y, direction, naive_value, accelerated_value;
} oracle_verify_result;

/* fault5 = {image_index, x, y, term_index, delta} or NULL */
int oracle_verify_image(const uint8_t* px, int rows, int cols, const int* fault5, int image_index,
                        oracle_verify_result* r) {
    memset(r, 0, sizeof(*r));
    if (fault5 && (fault5[3] < 0 || fault5[3] > 14)) return -1;
    r->images_checked = 1;
    for (int x = 0; x < rows; ++x)
        for (int y = 0; y < cols; ++y) {
            int32_t naive[8], a[15], accel[8];
            oracle_responses(px, rows, cols, x, y, naive);
            oracle_column_terms(px, rows, cols, x, y, a);
            if (fault5 && fault5[0] == image_index && fault5[1] == x && fault5[2] == y)
                a[fault5[3]] += fault5[4];
            oracle_responses_terms(a, accel);
            ++r->pixels_checked;
            for (int d = 0; d < 8; ++d)
                if (naive[d] != accel[d]) {
                    r->has_mismatch = 1;
                    r->image_index = image_index, r->x = x, r->y = y, r->direction = d;
                    r->naive_value = naive[d], r->accelerated_value = accel[d];
                    return 0;
                }
        }
    return 0;
}

int oracle_verify_equivalence(int images, uint32_t seed, const int* fault5, int threads,
                              oracle_verify_result* r) {
    memset(r, 0, sizeof(*r));
    if (fault5 && (fault5[3] < 0 || fault5[3] > 14)) return -1;
    if (images < 1) images = 1;
    int* dims = (int*)malloc(sizeof(int) * 2 * (size_t)images);
    uint32_t* seeds = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)images);
    mt19937 s;
    mt_seed(&s, seed);
    for (int i = 0; i < images; ++i) {
        dims[2 * i] = 3 + (int)(mt_next(&s) % 62);
        dims[2 * i + 1] = 3 + (int)(mt_next(&s) % 62);
        seeds[i] = mt_next(&s);
    }
    if (threads < 1) threads = 1;
    if (threads > images) threads = images;
    const int chunk = (images + threads - 1) / threads;
    uint8_t* img = (uint8_t*)malloc(64 * 64);
    for (int t = 0; t < threads; ++t) {
        const int lo = t * chunk, hi = lo + chunk < images ? lo + chunk : images;
        for (int i = lo; i < hi; ++i) {
            oracle_make_random(dims[2 * i], dims[2 * i + 1], seeds[i], img);
            oracle_verify_result one;
            oracle_verify_image(img, dims[2 * i], dims[2 * i + 1], fault5, i, &one);
            r->images_checked += one.images_checked;
            r->pixels_checked += one.pixels_checked;
            if (one.has_mismatch) {
                if (!r->has_mismatch) {
                    const uint64_t ic = r->images_checked, pc = r->pixels_checked;
                    *r = one;
                    r->images_checked = ic, r->pixels_checked = pc;
                }
                break;
            }
        }
    }
    free(img);
    free(seeds);
    free(dims);
    return 0;
}

/* kirsch.cpp:193-208: the naive responses of every pixel, [rows*cols][8]. */
void oracle_response_field(const uint8_t* px, int rows, int cols, int32_t* out) {
    for (int x = 0; x < rows; ++x)
        for (int y = 0; y < cols; ++y) oracle_responses(px, rows, cols, x, y, out + ((size_t)x * cols + y) * 8);
}
