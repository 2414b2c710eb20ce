// ldp_kernels.cu -- B200 (sm_100a) kernels for the LDP path and the C-ABI
// dispatch behind include/aldp_cuda.h.
//
// Two kernels, both CUDA, selected per call by layout:
//  * ldp_fast_kernel<K, NCL> -- the product hot path. One warp owns a
//    "tile" of band_rows x 128 columns; each lane owns four adjacent columns
//    and slides down the band keeping three rows of packed u16x2 ring values
//    in registers. Per output row and lane: 16 Kirsch keys (two pixel pairs),
//    an 18-op min/max top-k network per pair, a 6-bit XOR id, one shared-
//    memory table lookup per pixel for the code, one per-lane shared-memory
//    atomic per pixel for the histogram, one coalesced 4-byte code store.
//  * ldp_generic_kernel -- one thread per pixel, any geometry and any k.
//    Used for layouts the fast kernel does not take (pitches, strides or
//    base pointers that are not 8-byte aligned) and as the parity vehicle.
//
// Reference semantics: see ldp_common.cuh and include/aldp_cuda.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "aldp_cuda.h"
#include "ldp_common.cuh"

namespace aldp_b200 {

// --------------------------------------------------------------------------
// error plumbing
// --------------------------------------------------------------------------
static thread_local std::string t_last_error;
static thread_local int t_launches;  // kernels the last batch call launched (aldp_last_launch_count)
// aldp_debug_fault mode; ALDP_FAULT_INJECT sets the initial value
static std::atomic<int> g_fault{[] {
    const char* e = std::getenv("ALDP_FAULT_INJECT");
    return e ? std::atoi(e) : 0;
}()};
void count_launch() { ++t_launches; }

// Records `msg` as this host thread's last error (aldp_last_error) and
// returns `s`. Shared with ldp_host.cu.
aldp_status set_error(aldp_status s, const std::string& msg) {
    t_last_error = msg;
    return s;
}

static aldp_status fail(aldp_status s, const std::string& msg) { return set_error(s, msg); }

static aldp_status cuda_fail(cudaError_t e, const char* what) {
    return fail(ALDP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define ALDP_CUDA_TRY(expr)                                        \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);        \
    } while (0)

// --------------------------------------------------------------------------
// fast kernel (ldp_fast.cuh)
// --------------------------------------------------------------------------
}  // namespace aldp_b200
#include "ldp_fast.cuh"
#include "ldp_fast_launch.cuh"
namespace aldp_b200 {

// --------------------------------------------------------------------------
// generic kernel: one thread per pixel
// --------------------------------------------------------------------------
struct GenericParams {
    const uint8_t* px;
    int64_t img_stride;
    int pitch, rows, cols, n_images, k;
    uint8_t* codes;
    int64_t codes_img_stride;
    int codes_pitch;
    uint32_t* hist;
    int nbins;
    int hist16;                                // uint16 counts, two per word
    int cell_rows, cell_cols, grid_r, grid_c;  // cell_rows == 0: whole image
    int cell_clamp;                            // 0: cells cut from the whole-image code map
    int row_lo, row_hi;                        // neighbour rows readable (halo rows of a band view)
};

__global__ void ldp_generic_kernel(GenericParams p) {
    const int64_t plane = int64_t(p.rows) * p.cols;
    const int64_t total = plane * p.n_images;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int img = int(t / plane);
        const int64_t rem = t - int64_t(img) * plane;
        const int x = int(rem / p.cols), y = int(rem - int64_t(x) * p.cols);
        const uint8_t* base = p.px + img * p.img_stride;
        // k == 0: LBP (256 bins indexed by the code itself)
        const unsigned code = p.k ? clamped_code(base, p.pitch, x, y, p.row_lo, p.row_hi, 0, p.cols - 1, p.k)
                                  : clamped_lbp(base, p.pitch, x, y, p.row_lo, p.row_hi, 0, p.cols - 1);
        if (p.codes)
            p.codes[img * p.codes_img_stride + int64_t(x) * p.codes_pitch + y] = uint8_t(code);
        if (!p.hist) continue;
        if (p.cell_rows == 0) {
            hist_add(p.hist, p.hist16, int64_t(img) * p.nbins + (p.k ? colex_rank(code) : code), 1u);
        } else {
            const int cr = x / p.cell_rows, cc = y / p.cell_cols;
            if (cr >= p.grid_r || cc >= p.grid_c) continue;  // remainder dropped
            const int x0 = cr * p.cell_rows, y0 = cc * p.cell_cols;
            const bool edge = x == x0 || x == x0 + p.cell_rows - 1 || y == y0 ||
                              y == y0 + p.cell_cols - 1;
            unsigned hc = code;
            if (edge && p.cell_clamp)
                hc = p.k ? clamped_code(base, p.pitch, x, y, x0, x0 + p.cell_rows - 1, y0, y0 + p.cell_cols - 1, p.k)
                         : clamped_lbp(base, p.pitch, x, y, x0, x0 + p.cell_rows - 1, y0, y0 + p.cell_cols - 1);
            const int64_t cell = int64_t(img) * p.grid_r * p.grid_c + int64_t(cr) * p.grid_c + cc;
            hist_add(p.hist, p.hist16, cell * p.nbins + (p.k ? colex_rank(hc) : hc), 1u);
        }
    }
}


// Negative control (aldp_debug_fault): after a batch, corrupt image 0's code
// at (0, 0) and its first histogram's bin 0 -- a separate launch, so the
// product kernels carry no trace of it.
__global__ void fault_kernel(uint8_t* codes, uint32_t* hist, int hist16) {
    if (codes) codes[0] ^= 1;
    if (hist) hist_add(hist, hist16, 0, 1u);
}

// --------------------------------------------------------------------------
// dispatch
// --------------------------------------------------------------------------
static int n_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

// launch_fast_t<...> (ldp_fast_launch.cuh): the cell-histogram
// instantiations are compiled in ldp_fast_cells.cu (their own ptxas
// options), the rest here.
int fast_n_sms() { return n_sms(); }
ALDP_FAST_CELL_INSTANTIATIONS(extern template)
ALDP_FAST_NARROW_INSTANTIATIONS(extern template)

template <int K, int NW, bool HALO>
static aldp_status launch_fast_kw(const FastParams& p, bool cells, bool narrow, cudaStream_t st) {
    const bool codes = p.codes != nullptr, hist = p.hist != nullptr;
    if constexpr (K != 0 && K != 4) {
        if (cells && narrow)
            return codes ? launch_fast_t<K, NW, true, true, true, HALO, kNarrowTileCells>(p, st)
                         : launch_fast_t<K, NW, true, false, true, HALO, kNarrowTileCells>(p, st);
    }
    if (cells) {  // cell geometry only matters for histograms
        return codes ? launch_fast_t<K, NW, true, true, true, HALO>(p, st)
                     : launch_fast_t<K, NW, true, false, true, HALO>(p, st);
    }
    if (codes && hist) return launch_fast_t<K, NW, false, true, true, HALO>(p, st);
    if (codes) return launch_fast_t<K, NW, false, true, false, HALO>(p, st);
    return launch_fast_t<K, NW, false, false, true, HALO>(p, st);
}

// Two 4-byte words per lane (NW = 2; one word per lane measured slower).
constexpr int kLaneWords = 2;

template <int K>
static aldp_status launch_fast_k(const FastParams& p, bool cells, bool narrow, bool halo, cudaStream_t st) {
    return halo ? launch_fast_kw<K, kLaneWords, true>(p, cells, narrow, st)
                : launch_fast_kw<K, kLaneWords, false>(p, cells, narrow, st);
}

static aldp_status launch_fast(const FastParams& p, int k, bool cells, bool narrow, bool halo, cudaStream_t st) {
    switch (k) {
    case 0: return launch_fast_k<0>(p, cells, narrow, halo, st);  // LBP
    case 1: return launch_fast_k<1>(p, cells, narrow, halo, st);
    case 2: return launch_fast_k<2>(p, cells, narrow, halo, st);
    case 3: return launch_fast_k<3>(p, cells, narrow, halo, st);
    case 4: return launch_fast_k<4>(p, cells, narrow, halo, st);
    case 5: return launch_fast_k<5>(p, cells, narrow, halo, st);
    case 6: return launch_fast_k<6>(p, cells, narrow, halo, st);
    case 7: return launch_fast_k<7>(p, cells, narrow, halo, st);
    default: return fail(ALDP_EINVAL, "fast kernel: unsupported k");
    }
}

// Most cells a 128-column tile can touch for this geometry.
static int max_cells_per_tile(int cols, int cell_cols, int grid_c) {
    int worst = 0;
    for (int c0 = 0; c0 < cols; c0 += kTileCols) {
        const int end = std::min(std::min(c0 + kTileCols, cols), grid_c * cell_cols) - 1;
        if (end < c0) continue;
        worst = std::max(worst, end / cell_cols - c0 / cell_cols + 1);
    }
    return std::max(worst, 1);
}

static aldp_status validate(const aldp_ldp_args* a, int* grid_r, int* grid_c, bool lbp) {
    if (!a) return fail(ALDP_EINVAL, "null args");
    if (!lbp && (a->k < 1 || a->k > 7)) return fail(ALDP_EINVAL, "k must be in [1, 7]");
    if (a->rows < 3 || a->cols < 3)
        return fail(ALDP_EINVAL, "descriptor extraction needs at least a 3x3 image, got " +
                                     std::to_string(a->rows) + "x" + std::to_string(a->cols));
    if (a->n_images < 0) return fail(ALDP_EINVAL, "negative image count");
    if (a->pitch < a->cols) return fail(ALDP_EINVAL, "pitch smaller than cols");
    if (a->n_images > 1 && a->img_stride < int64_t(a->pitch) * a->rows)
        return fail(ALDP_EINVAL, "image stride smaller than an image");
    if (a->n_images > 0 && !a->d_pixels) return fail(ALDP_EINVAL, "null pixels");
    if (a->d_codes && a->codes_pitch < a->cols) return fail(ALDP_EINVAL, "codes pitch < cols");
    if ((a->cell_rows == 0) != (a->cell_cols == 0))
        return fail(ALDP_EINVAL, "cell_rows and cell_cols must both be 0 or both set");
    if (a->cell_rows) {
        if (a->cell_rows < 3 || a->cell_cols < 3)
            return fail(ALDP_EINVAL, "window side must be >= 3");
        if (a->cell_rows > a->rows || a->cell_cols > a->cols)
            return fail(ALDP_EINVAL, "window exceeds image");
        *grid_r = a->rows / a->cell_rows;
        *grid_c = a->cols / a->cell_cols;
    } else {
        *grid_r = *grid_c = 1;
    }
    return ALDP_OK;
}

// Exact unsigned division by d for dividends below 2^31 as (n * m) >> sh:
// sh = 32 + ceil(log2 d), m = floor(2^sh / d) + 1. The error term n(m - 2^sh/d)
// / 2^sh < 2^31 / 2^sh <= 1 / (2d) never crosses an integer (Granlund-Montgomery).
static void magic_div(uint32_t d, uint64_t& m, int& sh) {
    if (d == 0) d = 1;
    int l = 0;
    while ((uint64_t(1) << l) < d) ++l;
    sh = 32 + l;
    m = (uint64_t(1) << sh) / d + 1;  // < 2^33 + 1 (2^l < 2d), so n * m < 2^64
}

// Band geometry, tile order, exact-division constants and id tables of a
// fast-kernel launch over n_images frames of p.rows rows, then the launch.
// cells: cell histograms (the cell kernel and tag set 0); halo: p is a band
// view whose edge rows may see real rows (row_lo / row_hi).
static aldp_status finish_fast(FastParams& p, int n_images, int cell_rows, int cell_cols, int k, bool cells,
                               bool halo, cudaStream_t st, bool narrow = false) {
    p.band_rows = cell_rows ? cell_rows : 128;
    if (!cell_rows) {
        // Small batches (a few frames per call): shorter bands until the
        // tiles fill every warp slot once (2 tiles per warp, 2 CTAs of 8
        // warps per SM); each band costs two recounted edge rows.
        const int64_t slots = int64_t(n_sms()) * 2 * kFastWarps * 2;
        while (p.band_rows > 16 &&
               int64_t(n_images) * ((p.rows + p.band_rows - 1) / p.band_rows) * p.blocks < slots)
            p.band_rows /= 2;
    }
    p.bands = (p.rows + p.band_rows - 1) / p.band_rows;
    p.uniform_bands = p.rows % p.band_rows == 0 ? 1 : 0;
    p.n_tiles = int64_t(n_images) * p.bands * p.blocks;
    {
        const int G = (p.blocks & 1) ? 2 : 1;
        magic_div(uint32_t(int64_t(G) * p.bands * p.blocks), p.mg_group, p.sh_group);
        magic_div(uint32_t(G * p.blocks), p.mg_bandG, p.sh_bandG);
        magic_div(uint32_t(p.blocks), p.mg_band1, p.sh_band1);
        magic_div(uint32_t(p.blocks), p.mg_blocks, p.sh_blocks);
        magic_div(uint32_t(cell_cols ? cell_cols : 1), p.mg_cell, p.sh_cell);
    }
    p.one = 1;
    const int ts = fast_tag_set(cells);  // the tag set the launched kernel keys with
    for (int id = 0; id < 128; ++id) p.id_code[id] = p.id_bin[id] = 0;
    for (int c = 0; c < 256 && k; ++c)
        if (popcount8(c) == k) {
            // k == 4: the 6-bit XOR plus "direction 0 selected" (ldp_common.cuh top4_id)
            const int id = int(tag_xor(c, ts)) | (k == 4 ? (c & 1) << 6 : 0);
            if (p.id_code[id]) return fail(ALDP_EINVAL, "internal: code id collision");
            p.id_code[id] = uint8_t(c);
            p.id_bin[id] = uint8_t(colex_rank(c));
            if (k != 4) p.bin_id[colex_rank(c)] = uint8_t(id);
        }
    return launch_fast(p, k, cells, narrow, halo, st);
}

// How the narrow-cell kernel writes its histograms (ALDP_NARROW_HIST
// overrides, read per call so tests can toggle it):
//   0 = every bin added with global atomics into a memset histogram (round 1);
//   2 = cells wholly inside a 128-column tile stored, the few that straddle a
//       tile edge added after zero_straddling_cells (default).
// A/B on 2048 C5 frames (profiles/r02_narrow_ab.txt): window 10: 283 k -> 338 k
// Mpixel/s, window 25: 501 k -> 522 k. (Mode 1, tiles of whole cells with
// every bin stored, measured 301 k / 398 k and was dropped: its tiles
// recompute the columns they overlap.)
static int narrow_hist_mode() {
    const char* e = std::getenv("ALDP_NARROW_HIST");
    return e ? std::atoi(e) : 2;
}

// Zeroes the histograms of the cells that straddle a 128-column tile edge
// (narrow mode 2 adds into those; every other cell is stored whole).
__global__ void zero_straddling_cells(uint32_t* hist, int hist16, int64_t n_cells, int grid_c, int cell_cols,
                                      int nbins) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_cells;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int cf = int(i % grid_c) * cell_cols;
        if (cf / kTileCols == (cf + cell_cols - 1) / kTileCols) continue;
        if (hist16) {
            uint16_t* h = reinterpret_cast<uint16_t*>(hist) + i * nbins;
            for (int b = 0; b < nbins; ++b) h[b] = 0;
        } else {
            uint32_t* h = hist + i * nbins;
            for (int b = 0; b < nbins; ++b) h[b] = 0;
        }
    }
}

// lbp: the LBP descriptor (256 bins, k ignored); internally k == 0.
static aldp_status run_batch(const aldp_ldp_args* a, int kernel, cudaStream_t st, bool lbp) {
    t_launches = 0;
    int grid_r = 1, grid_c = 1;
    aldp_status s = validate(a, &grid_r, &grid_c, lbp);
    if (s != ALDP_OK) return s;
    const int k = lbp ? 0 : a->k;
    const int nbins = lbp ? 256 : aldp_n_bins(a->k);
    const int64_t cells = a->cell_rows ? int64_t(grid_r) * grid_c : 1;
    if (a->hist_u16) {
        const int64_t area = a->cell_rows ? int64_t(a->cell_rows) * a->cell_cols : int64_t(a->rows) * a->cols;
        if (area >= 65536) return fail(ALDP_EINVAL, "hist_u16: a histogram can reach 65536 counts");
        if (reinterpret_cast<uintptr_t>(a->d_hist) % 4) return fail(ALDP_EINVAL, "hist_u16: d_hist not 4-byte aligned");
    }
    const int al = 4 * kLaneWords;  // alignment the per-lane vector loads/stores need
    const bool aligned =
        a->pitch % al == 0 && (a->n_images <= 1 || a->img_stride % al == 0) &&
        (reinterpret_cast<uintptr_t>(a->d_pixels) % al) == 0 &&
        (!a->d_codes || (a->codes_pitch % al == 0 && (reinterpret_cast<uintptr_t>(a->d_codes) % al) == 0 &&
                         (a->n_images <= 1 || a->codes_img_stride % al == 0)));
    // cells per 128-column tile: up to kMaxTileCells on the regular layout,
    // kNarrowTileCells on the narrow one (LDP k != 4, cells of >= 9 columns)
    int ncl = 1;
    if (a->cell_rows && a->d_hist) ncl = max_cells_per_tile(a->cols, a->cell_cols, grid_c);
    const bool narrow = ncl > kMaxTileCells;
    const bool fast_ok = aligned && (!narrow || (ncl <= kNarrowTileCells && a->cell_cols >= 9 && !lbp && a->k != 4));
    // narrow cells: histograms stored four bins at a time (16-byte stores of
    // u32 bins, 8-byte of u16) -- mode 2 of narrow_hist_mode()
    const int nmode = (kernel != ALDP_KERNEL_GENERIC && fast_ok && narrow && !a->cell_from_map &&
                       reinterpret_cast<uintptr_t>(a->d_hist) % (a->hist_u16 ? 8 : 16) == 0)
                          ? narrow_hist_mode()
                          : 0;
    if (a->d_hist && nmode == 0)
        ALDP_CUDA_TRY(cudaMemsetAsync(a->d_hist, 0,
                                      (a->hist_u16 ? 2 : 4) * size_t(a->n_images) * cells * nbins, st));
    if (a->d_hist && nmode == 2 && a->n_images > 0) {
        const int64_t n_cells = int64_t(a->n_images) * cells;
        const int grid = int(std::min<int64_t>((n_cells + 255) / 256, 8LL * n_sms()));
        zero_straddling_cells<<<grid, 256, 0, st>>>(a->d_hist, a->hist_u16, n_cells, grid_c, a->cell_cols, nbins);
        count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "zero_straddling_cells launch");
    }
    if (a->n_images == 0 || (!a->d_codes && !a->d_hist)) return ALDP_OK;
    if (kernel == ALDP_KERNEL_FAST && !fast_ok)
        return fail(ALDP_EINVAL, "fast kernel needs 8-byte aligned pitches/strides and at most 5 cells per "
                                 "128 columns (16 for LDP k != 4 with cells of >= 9 columns)");
    if (kernel != ALDP_KERNEL_GENERIC && fast_ok) {
        FastParams p{};
        p.px = a->d_pixels;
        p.img_stride = a->img_stride;
        p.pitch = a->pitch;
        p.rows = a->rows;
        p.cols = a->cols;
        p.n_images = a->n_images;
        p.codes = a->d_codes;
        p.codes_img_stride = a->codes_img_stride;
        p.codes_pitch = a->codes_pitch;
        p.hist = a->d_hist;
        p.nbins = nbins;
        p.hist16 = a->hist_u16 ? 1 : 0;
        p.cell_rows = a->cell_rows;
        p.cell_cols = a->cell_cols;
        p.cell_clamp = a->cell_from_map ? 0 : 1;
        p.row_lo = a->rows_above ? -1 : 0;
        p.row_hi = a->rows - 1 + (a->rows_below ? 1 : 0);
        p.edge_lo = p.cell_clamp ? 0 : -1;
        p.edge_hi = p.cell_clamp ? a->cell_rows - 1 : -1;
        p.grid_r = grid_r;
        p.grid_c = grid_c;
        p.blocks = (a->cols + kTileCols - 1) / kTileCols;
        p.store_whole = nmode == 2 ? 1 : 0;
        // Cell histograms with rows below the cell grid (490 = 6 x 81 + 4 for
        // the 7x6 grid of a 640x490 frame): the grid rows run as one launch and
        // the short remainder as a second, codes-only launch. Warps take tiles
        // round-robin; with the short band mixed in, a warp that drew only
        // full-height tiles set the end of the kernel on small batches (C2:
        // its 8 tiles against a mean of 6.5). Only the grid launch's last row
        // sees a clamped row below it; it is a cell edge row (its histogram
        // uses the cell clamp anyway) and its code is rewritten by the second
        // launch, which starts two rows above the grid's end with a real row
        // above it. cell_from_map counts map codes, so it keeps one launch.
        // Round 1 split only small batches (C2 +4.7 %, full C5 -0.5 %); with
        // the round-2 row loop the split pays at every size (full C5: 762 k
        // -> 794 k Mpixel/s, profiles/r02_split_ab.txt): the remainder launch
        // recomputes ~1 % of the pixels, but the grid launch then runs tiles
        // of one height and one code path. ALDP_SPLIT_TILES (tiles per warp
        // segment below which to split) overrides it for A/B runs.
        // (validate() guarantees grid_r >= 1 here: cell_rows <= rows.)
        static const int64_t kSplitTiles = [] {
            const char* e = std::getenv("ALDP_SPLIT_TILES");
            return e ? int64_t(std::atoll(e)) : int64_t(1) << 40;
        }();
        const int grid_rows = grid_r * a->cell_rows;
        const int64_t tiles = int64_t(a->n_images) * ((a->rows + a->cell_rows - 1) / std::max(a->cell_rows, 1)) *
                              ((a->cols + kTileCols - 1) / kTileCols);
        const int64_t seg_slots = int64_t(n_sms()) * 2 * kFastWarps * 2;
        if (a->cell_rows && !a->cell_from_map && grid_rows < a->rows && tiles < kSplitTiles * seg_slots) {
            FastParams q = p;
            p.rows = grid_rows;
            p.row_hi = grid_rows - 1;
            if (aldp_status s1 = finish_fast(p, a->n_images, a->cell_rows, a->cell_cols, k, a->d_hist != nullptr,
                                             a->rows_above != 0, st, narrow);
                s1 != ALDP_OK)
                return s1;
            if (!a->d_codes) return ALDP_OK;
            const int start = grid_rows - 2;  // >= 1: cells are >= 3 rows
            q.px = a->d_pixels + int64_t(start) * a->pitch;
            q.rows = a->rows - start;
            q.codes = a->d_codes + int64_t(start) * a->codes_pitch;
            q.hist = nullptr;
            q.store_whole = 0;
            q.blocks = (a->cols + kTileCols - 1) / kTileCols;
            q.cell_rows = q.cell_cols = 0;
            q.grid_r = q.grid_c = 1;
            q.edge_lo = q.edge_hi = -1;
            q.row_lo = -1;
            q.row_hi = q.rows - 1 + (a->rows_below ? 1 : 0);
            return finish_fast(q, a->n_images, 0, 0, k, false, true, st);
        }
        return finish_fast(p, a->n_images, a->cell_rows, a->cell_cols, k, a->cell_rows != 0 && a->d_hist != nullptr,
                           a->rows_above || a->rows_below, st, narrow);
    }
    GenericParams g{};
    g.px = a->d_pixels;
    g.img_stride = a->img_stride;
    g.pitch = a->pitch;
    g.rows = a->rows;
    g.cols = a->cols;
    g.n_images = a->n_images;
    g.k = k;
    g.codes = a->d_codes;
    g.codes_img_stride = a->codes_img_stride;
    g.codes_pitch = a->codes_pitch;
    g.hist = a->d_hist;
    g.nbins = nbins;
    g.hist16 = a->hist_u16 ? 1 : 0;
    g.cell_rows = a->cell_rows;
    g.cell_cols = a->cell_cols;
    g.cell_clamp = a->cell_from_map ? 0 : 1;
    g.row_lo = a->rows_above ? -1 : 0;
    g.row_hi = a->rows - 1 + (a->rows_below ? 1 : 0);
    g.grid_r = grid_r;
    g.grid_c = grid_c;
    const int64_t total = int64_t(a->rows) * a->cols * a->n_images;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 32LL * n_sms())));
    ldp_generic_kernel<<<grid, 256, 0, st>>>(g);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "ldp_generic_kernel launch");
    return ALDP_OK;
}

// run_batch, then the negative control's corruption when it is on.
static aldp_status run_batch_checked(const aldp_ldp_args* a, int kernel, cudaStream_t st, bool lbp) {
    aldp_status s = run_batch(a, kernel, st, lbp);
    if (s == ALDP_OK && g_fault.load(std::memory_order_relaxed) && a->n_images > 0 && (a->d_codes || a->d_hist)) {
        fault_kernel<<<1, 1, 0, st>>>(a->d_codes, a->d_hist, a->hist_u16 ? 1 : 0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "fault_kernel launch");
    }
    return s;
}

}  // namespace aldp_b200

using namespace aldp_b200;

extern "C" {

aldp_status aldp_ldp_batch(const aldp_ldp_args* args, void* stream) {
    return run_batch_checked(args, ALDP_KERNEL_AUTO, static_cast<cudaStream_t>(stream), false);
}

aldp_status aldp_ldp_batch_ex(const aldp_ldp_args* args, int kernel, void* stream) {
    if (kernel < ALDP_KERNEL_AUTO || kernel > ALDP_KERNEL_GENERIC)
        return fail(ALDP_EINVAL, "unknown kernel selector");
    return run_batch_checked(args, kernel, static_cast<cudaStream_t>(stream), false);
}

aldp_status aldp_lbp_batch(const aldp_ldp_args* args, void* stream) {
    return run_batch_checked(args, ALDP_KERNEL_AUTO, static_cast<cudaStream_t>(stream), true);
}

aldp_status aldp_lbp_batch_ex(const aldp_ldp_args* args, int kernel, void* stream) {
    if (kernel < ALDP_KERNEL_AUTO || kernel > ALDP_KERNEL_GENERIC)
        return fail(ALDP_EINVAL, "unknown kernel selector");
    return run_batch_checked(args, kernel, static_cast<cudaStream_t>(stream), true);
}

int aldp_n_bins(int k) {
    if (k < 1 || k > 7) return 0;
    return binom(8, k);
}

int64_t aldp_grid_cells(int rows, int cols, int cell_rows, int cell_cols) {
    if (cell_rows == 0 && cell_cols == 0) return 1;
    if (cell_rows < 3 || cell_cols < 3 || cell_rows > rows || cell_cols > cols) return -1;
    return int64_t(rows / cell_rows) * (cols / cell_cols);
}

const char* aldp_last_error(void) { return t_last_error.c_str(); }

int aldp_last_launch_count(void) { return t_launches; }

int aldp_debug_fault(int mode) { return g_fault.exchange(mode); }

const char* aldp_version(void) { return "aldp_b200 0.1.0 sm_100a"; }

}  // extern "C"
