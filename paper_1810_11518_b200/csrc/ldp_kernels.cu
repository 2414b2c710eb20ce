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
//  * ldp_generic_kernel -- one thread per pixel, any geometry and any k
//    (including k == 4, which the XOR id cannot name). Used for layouts the
//    fast kernel does not take (odd widths/pitches) and tiny images.
//
// Reference semantics: see ldp_common.cuh and include/aldp_cuda.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
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
    int cell_rows, cell_cols, grid_r, grid_c;  // cell_rows == 0: whole image
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
        const unsigned code = clamped_code(base, p.pitch, x, y, 0, p.rows - 1, 0, p.cols - 1, p.k);
        if (p.codes)
            p.codes[img * p.codes_img_stride + int64_t(x) * p.codes_pitch + y] = uint8_t(code);
        if (!p.hist) continue;
        if (p.cell_rows == 0) {
            atomicAdd(p.hist + int64_t(img) * p.nbins + colex_rank(code), 1u);
        } else {
            const int cr = x / p.cell_rows, cc = y / p.cell_cols;
            if (cr >= p.grid_r || cc >= p.grid_c) continue;  // remainder dropped
            const int x0 = cr * p.cell_rows, y0 = cc * p.cell_cols;
            const bool edge = x == x0 || x == x0 + p.cell_rows - 1 || y == y0 ||
                              y == y0 + p.cell_cols - 1;
            const unsigned hc =
                edge ? clamped_code(base, p.pitch, x, y, x0, x0 + p.cell_rows - 1, y0,
                                    y0 + p.cell_cols - 1, p.k)
                     : code;
            const int64_t cell = int64_t(img) * p.grid_r * p.grid_c + int64_t(cr) * p.grid_c + cc;
            atomicAdd(p.hist + cell * p.nbins + colex_rank(hc), 1u);
        }
    }
}

// --------------------------------------------------------------------------
// fast kernel
// --------------------------------------------------------------------------
constexpr int kWarps = 4;          // warps per CTA
constexpr int kLaneCols = 4;       // columns per lane (one 32-bit word)
constexpr int kTileCols = 32 * kLaneCols;
constexpr int kIds = 64;           // 6-bit XOR ids
constexpr int kRegionBytes = kIds * 32 * 4;  // per-lane counters of one cell
constexpr uint32_t kScaleMask = 0x3FC03FC0u; // bytes 0/2 of a word, << 6

struct FastParams {
    const uint8_t* px;
    int64_t img_stride;
    int pitch, rows, cols, n_images;
    uint8_t* codes;
    int64_t codes_img_stride;
    int codes_pitch;
    uint32_t* hist;
    int nbins;
    int cell_mode;  // 0: whole image (one cell, image clamp)
    int cell_rows, cell_cols, grid_r, grid_c;
    int band_rows, bands, blocks;  // tiles = n_images * bands * blocks
    int64_t n_tiles;
};

// One input row as packed, pre-scaled (x64) u16x2 pairs. For a lane owning
// columns y..y+3: A = (y, y+2), B = (y+1, y+3), L = (y-1, y+1), R = (y+2, y+4).
struct Row {
    uint32_t A, B, L, R;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    return __byte_perm(a, b, s);
}

// Load the lane's word of image row `x` (already clamped), with the column
// clamp applied through the per-lane byte selector `sel`.
__device__ __forceinline__ uint32_t load_word(const uint8_t* rowp, int off, uint32_t sel) {
    const uint32_t raw = __ldg(reinterpret_cast<const uint32_t*>(rowp + off));
    return prmt(raw, raw, sel);
}

template <int K, int NCL>
__global__ void __launch_bounds__(kWarps * 32) ldp_fast_kernel(FastParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    // [0, 8 KB): id -> code table replicated per lane; [8 KB, 8 KB + 64 B):
    // id -> bin; then per warp NCL regions of per-lane counters.
    uint32_t* lut = reinterpret_cast<uint32_t*>(smem);
    uint8_t* id_bin = smem + kRegionBytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* region0 = smem + kRegionBytes + 64 + warp * NCL * kRegionBytes;

    // Table build: every popcount-K code -> its XOR id.
    for (int c = threadIdx.x; c < 256; c += blockDim.x) {
        if (popcount8(c) != K) continue;
        const uint32_t id = tag_xor(c);
        for (int l = 0; l < 32; ++l) lut[id * 32 + l] = uint32_t(c);
        id_bin[id] = uint8_t(colex_rank(c));
    }
    {
        uint32_t* cnt = reinterpret_cast<uint32_t*>(region0);
        for (int i = lane; i < NCL * kIds * 32; i += 32) cnt[i] = 0;
    }
    __syncthreads();

    const uint32_t lane4 = uint32_t(lane) * 4u;
    const uint32_t lut_base = uint32_t(__cvta_generic_to_shared(lut));
    const uint32_t reg_base = uint32_t(__cvta_generic_to_shared(region0));

    // Packed tag constants (both lanes of the u16x2 key).
    constexpr uint32_t T0 = kTag(0) * 0x10001u, T1 = kTag(1) * 0x10001u, T2 = kTag(2) * 0x10001u,
                       T3 = kTag(3) * 0x10001u, T4 = kTag(4) * 0x10001u, T5 = kTag(5) * 0x10001u,
                       T6 = kTag(6) * 0x10001u, T7 = kTag(7) * 0x10001u;

    const int64_t tiles_per_image = int64_t(p.bands) * p.blocks;
    for (int64_t tile = int64_t(blockIdx.x) * kWarps + warp; tile < p.n_tiles;
         tile += int64_t(gridDim.x) * kWarps) {
        const int img = int(tile / tiles_per_image);
        const int rem = int(tile - int64_t(img) * tiles_per_image);
        const int band = rem / p.blocks, blk = rem - band * p.blocks;
        const int r0 = band * p.band_rows;
        const int r1 = min(p.rows, r0 + p.band_rows);
        const int c0 = blk * kTileCols;
        const int y = c0 + lane * kLaneCols;
        const uint8_t* src = p.px + img * p.img_stride;

        // Column clamp: this lane's word (may lie partly/fully right of the
        // image) and the halo word (lane 31: left neighbour block word,
        // lane 0: right neighbour block word) as aligned offsets + byte
        // selectors replicating the edge pixel (image.cpp:36-40).
        const int last = p.cols - 1, last_al = last & ~3;
        auto clamp_word = [&](int col, int& off, uint32_t& sel) {
            const int a = min(max(col, 0), last_al);
            off = a;
            sel = 0;
            for (int j = 0; j < 4; ++j)
                sel |= uint32_t(min(max(col + j, 0), last) - a) << (4 * j);
        };
        int own_off, halo_off;
        uint32_t own_sel, halo_sel;
        clamp_word(y, own_off, own_sel);
        clamp_word(lane == 31 ? c0 - 4 : c0 + kTileCols, halo_off, halo_sel);
        // lane 31 needs the B form (bytes 1,3) of its halo word, lane 0 the
        // A form (bytes 0,2): rotate by 30 resp. 6 bits, then mask.
        const uint32_t halo_rot = lane == 31 ? 30u : 6u;
        const bool halo_lane = lane == 0 || lane == 31;

        auto load_row = [&](int x) -> Row {
            const uint8_t* rowp = src + int64_t(x) * p.pitch;
            const uint32_t w = load_word(rowp, own_off, own_sel);
            uint32_t h = 0;
            if (halo_lane) h = load_word(rowp, halo_off, halo_sel);
            h = __funnelshift_l(h, h, halo_rot) & kScaleMask;
            Row r;
            r.A = (w << 6) & kScaleMask;
            r.B = (w >> 2) & kScaleMask;
            // Rotating shuffles: lane 31 injects the left halo for lane 0,
            // lane 0 injects the right halo for lane 31.
            const uint32_t xb = lane == 31 ? h : r.B;
            const uint32_t ya = lane == 0 ? h : r.A;
            const uint32_t prevB = __shfl_sync(0xffffffffu, xb, (lane + 31) & 31);
            const uint32_t nextA = __shfl_sync(0xffffffffu, ya, (lane + 1) & 31);
            r.L = prmt(r.B, prevB, 0x1076);  // (y-1 <- prev.hi, y+1 <- B.lo)
            r.R = prmt(r.A, nextA, 0x5432);  // (y+2 <- A.hi, y+4 <- next.lo)
            return r;
        };

        // Histogram slots: per pixel a local cell region, or -1 (not counted
        // in the main pass: remainder, or a cell-edge column fixed up below).
        const int cell_c0 = p.cell_mode ? c0 / p.cell_cols : 0;
        uint32_t slot_base[4];
        bool slot_on[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int col = y + s;
            bool on = col < p.cols;
            int lc = 0;
            if (p.cell_mode) {
                const int cc = col / p.cell_cols, in = col - cc * p.cell_cols;
                on = on && cc < p.grid_c && in != 0 && in != p.cell_cols - 1;
                lc = cc - cell_c0;
            }
            slot_on[s] = on;
            slot_base[s] = reg_base + uint32_t(lc) * kRegionBytes + lane4;
        }
        const bool grid_band = !p.cell_mode || band < p.grid_r;

        uint8_t* dst = p.codes ? p.codes + img * p.codes_img_stride : nullptr;
        const bool lane_out = y < p.cols;

        Row ra = load_row(max(r0 - 1, 0));
        Row rb = load_row(r0);
        uint32_t psLA_a = ra.L + ra.A, psAB_a = ra.A + ra.B, psBR_a = ra.B + ra.R;
        uint32_t psLA_b = rb.L + rb.A, psAB_b = rb.A + rb.B, psBR_b = rb.B + rb.R;

        for (int x = r0; x < r1; ++x) {
            const Row rc = load_row(min(x + 1, p.rows - 1));
            const uint32_t psLA_c = rc.L + rc.A, psAB_c = rc.A + rc.B, psBR_c = rc.B + rc.R;

            // keys, pair A (pixels y, y+2): left L, centre A, right B
            uint32_t ka[8], kb[8];
            ka[0] = ra.B + rb.B + rc.B + T0;
            ka[1] = psAB_a + rb.B + T1;
            ka[2] = psLA_a + ra.B + T2;
            ka[3] = psLA_a + rb.L + T3;
            ka[4] = ra.L + rb.L + rc.L + T4;
            ka[5] = psLA_c + rb.L + T5;
            ka[6] = psLA_c + rc.B + T6;
            ka[7] = psAB_c + rb.B + T7;
            // keys, pair B (pixels y+1, y+3): left A, centre B, right R
            kb[0] = ra.R + rb.R + rc.R + T0;
            kb[1] = psBR_a + rb.R + T1;
            kb[2] = psAB_a + ra.R + T2;
            kb[3] = psAB_a + rb.A + T3;
            kb[4] = ra.A + rb.A + rc.A + T4;
            kb[5] = psAB_c + rb.A + T5;
            kb[6] = psAB_c + rc.R + T6;
            kb[7] = psBR_c + rb.R + T7;

            const uint32_t ida = topk_id<K>(ka);
            const uint32_t idb = topk_id<K>(kb);
            // per-pixel table offsets: id * 128 + lane * 4
            const uint32_t oa_lo = ((ida << 7) & 0x1F80u) | lane4;
            const uint32_t oa_hi = ((ida >> 9) & 0x1F80u) | lane4;
            const uint32_t ob_lo = ((idb << 7) & 0x1F80u) | lane4;
            const uint32_t ob_hi = ((idb >> 9) & 0x1F80u) | lane4;

            if (dst) {
                uint32_t ca_lo, ca_hi, cb_lo, cb_hi;
                asm("ld.shared.u32 %0, [%1];" : "=r"(ca_lo) : "r"(lut_base + oa_lo));
                asm("ld.shared.u32 %0, [%1];" : "=r"(cb_lo) : "r"(lut_base + ob_lo));
                asm("ld.shared.u32 %0, [%1];" : "=r"(ca_hi) : "r"(lut_base + oa_hi));
                asm("ld.shared.u32 %0, [%1];" : "=r"(cb_hi) : "r"(lut_base + ob_hi));
                const uint32_t word =
                    prmt(prmt(ca_lo, cb_lo, 0x0040), prmt(ca_hi, cb_hi, 0x0040), 0x5410);
                if (lane_out)
                    *reinterpret_cast<uint32_t*>(dst + int64_t(x) * p.codes_pitch + y) = word;
            }
            if (p.hist && grid_band) {
                const int in = x - r0;
                if (!p.cell_mode || (in != 0 && in != p.cell_rows - 1)) {
                    // slots: 0 = y (A lo), 1 = y+1 (B lo), 2 = y+2 (A hi), 3 = y+3 (B hi)
                    const uint32_t o[4] = {oa_lo, ob_lo, oa_hi, ob_hi};
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        if (slot_on[s]) {
                            const uint32_t addr = slot_base[s] + (o[s] - lane4);
                            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr));
                        }
                    }
                }
            }

            ra = rb;
            rb = rc;
            psLA_a = psLA_b; psAB_a = psAB_b; psBR_a = psBR_b;
            psLA_b = psLA_c; psAB_b = psAB_c; psBR_b = psBR_c;
        }

        asm volatile("" ::: "memory");
        if (!p.hist || !grid_band) continue;

        // ---- per-cell clamp fix-up (windowed_features semantics) ----
        // Pixels on a cell's border see a different neighbourhood than in the
        // whole-image map; count them with the cell-clamped code.
        int ncl = 1;
        if (p.cell_mode) {
            const int cmax = min(c0 + kTileCols, min(p.cols, p.grid_c * p.cell_cols)) - 1;
            ncl = cmax >= c0 ? cmax / p.cell_cols - cell_c0 + 1 : 0;
            const int x_lo = r0, x_hi = r0 + p.cell_rows - 1;
            const int c_end = min(c0 + kTileCols, p.grid_c * p.cell_cols);
            // (a) the band's first and last row, every in-grid column
            for (int i = lane; i < 2 * kTileCols; i += 32) {
                const int x = i < kTileCols ? x_lo : x_hi;
                const int col = c0 + (i & (kTileCols - 1));
                if (col >= c_end) continue;
                const int cc = col / p.cell_cols;
                const int y_lo = cc * p.cell_cols, y_hi = y_lo + p.cell_cols - 1;
                const unsigned code = clamped_code(src, p.pitch, x, col, x_lo, x_hi, y_lo, y_hi, K);
                atomicAdd(reinterpret_cast<uint32_t*>(region0 + (cc - cell_c0) * kRegionBytes) +
                              tag_xor(code) * 32 + lane, 1u);
            }
            // (b) interior rows of the cells' first and last columns
            const int inner = p.cell_rows - 2;
            for (int lc = 0; lc < ncl; ++lc) {
                const int cc = cell_c0 + lc;
                const int y_lo = cc * p.cell_cols, y_hi = y_lo + p.cell_cols - 1;
                for (int i = lane; i < 2 * inner; i += 32) {
                    const int col = i < inner ? y_lo : y_hi;
                    if (col < c0 || col >= c_end) continue;
                    const int x = x_lo + 1 + (i < inner ? i : i - inner);
                    const unsigned code =
                        clamped_code(src, p.pitch, x, col, x_lo, x_hi, y_lo, y_hi, K);
                    atomicAdd(reinterpret_cast<uint32_t*>(region0 + lc * kRegionBytes) +
                                  tag_xor(code) * 32 + lane, 1u);
                }
            }
        }
        __syncwarp();

        // ---- flush: sum the 32 per-lane counters of each id, one global
        // atomic per (cell, bin) that saw pixels, and re-zero ----
        for (int lc = 0; lc < ncl; ++lc) {
            uint32_t* cnt = reinterpret_cast<uint32_t*>(region0 + lc * kRegionBytes);
            const int64_t cell = p.cell_mode ? int64_t(band) * p.grid_c + cell_c0 + lc : 0;
            uint32_t* out = p.hist + (int64_t(img) * (p.cell_mode ? int64_t(p.grid_r) * p.grid_c : 1) +
                                      cell) * p.nbins;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int id = lane + 32 * h;
                uint4* row = reinterpret_cast<uint4*>(cnt + id * 32);
                uint32_t sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 v = row[q];
                    sum += v.x + v.y + v.z + v.w;
                    row[q] = make_uint4(0, 0, 0, 0);
                }
                if (sum) atomicAdd(out + id_bin[id], sum);
            }
        }
        __syncwarp();
    }
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

template <int K, int NCL>
static aldp_status launch_fast_t(const FastParams& p, cudaStream_t st) {
    const size_t smem = kRegionBytes + 64 + size_t(kWarps) * NCL * kRegionBytes;
    static std::once_flag once[1];
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once[0], [&] {
        attr_err = cudaFuncSetAttribute(ldp_fast_kernel<K, NCL>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    });
    if (attr_err != cudaSuccess) return cuda_fail(attr_err, "cudaFuncSetAttribute");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ldp_fast_kernel<K, NCL>, kWarps * 32,
                                                  smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t want = (p.n_tiles + kWarps - 1) / kWarps;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(per_sm) * n_sms())));
    ldp_fast_kernel<K, NCL><<<grid, kWarps * 32, smem, st>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "ldp_fast_kernel launch");
    return ALDP_OK;
}

template <int K>
static aldp_status launch_fast_k(const FastParams& p, int ncl, cudaStream_t st) {
    switch (ncl) {
    case 1: return launch_fast_t<K, 1>(p, st);
    case 2: return launch_fast_t<K, 2>(p, st);
    case 3: return launch_fast_t<K, 3>(p, st);
    default: return fail(ALDP_EINVAL, "fast kernel: too many cells per tile");
    }
}

static aldp_status launch_fast(const FastParams& p, int k, int ncl, cudaStream_t st) {
    switch (k) {
    case 1: return launch_fast_k<1>(p, ncl, st);
    case 2: return launch_fast_k<2>(p, ncl, st);
    case 3: return launch_fast_k<3>(p, ncl, st);
    case 5: return launch_fast_k<5>(p, ncl, st);
    case 6: return launch_fast_k<6>(p, ncl, st);
    case 7: return launch_fast_k<7>(p, ncl, st);
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

static aldp_status validate(const aldp_ldp_args* a, int* grid_r, int* grid_c) {
    if (!a) return fail(ALDP_EINVAL, "null args");
    if (a->k < 1 || a->k > 7) return fail(ALDP_EINVAL, "k must be in [1, 7]");
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

static aldp_status run_batch(const aldp_ldp_args* a, int kernel, cudaStream_t st) {
    int grid_r = 1, grid_c = 1;
    aldp_status s = validate(a, &grid_r, &grid_c);
    if (s != ALDP_OK) return s;
    const int nbins = aldp_n_bins(a->k);
    const int64_t cells = a->cell_rows ? int64_t(grid_r) * grid_c : 1;
    if (a->d_hist)
        ALDP_CUDA_TRY(cudaMemsetAsync(a->d_hist, 0,
                                      sizeof(uint32_t) * size_t(a->n_images) * cells * nbins, st));
    if (a->n_images == 0 || (!a->d_codes && !a->d_hist)) return ALDP_OK;

    const bool aligned =
        a->cols % 4 == 0 && a->pitch % 4 == 0 && (a->n_images <= 1 || a->img_stride % 4 == 0) &&
        (reinterpret_cast<uintptr_t>(a->d_pixels) & 3) == 0 &&
        (!a->d_codes || (a->codes_pitch % 4 == 0 && (reinterpret_cast<uintptr_t>(a->d_codes) & 3) == 0 &&
                         (a->n_images <= 1 || a->codes_img_stride % 4 == 0)));
    int ncl = 1;
    if (a->cell_rows) ncl = max_cells_per_tile(a->cols, a->cell_cols, grid_c);
    const bool fast_ok = aligned && a->k != 4 && ncl <= 3;
    if (kernel == ALDP_KERNEL_FAST && !fast_ok)
        return fail(ALDP_EINVAL, "fast kernel needs cols/pitch/strides multiple of 4, k != 4 "
                                 "and at most 3 cells per 128 columns");
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
        p.cell_mode = a->cell_rows ? 1 : 0;
        p.cell_rows = a->cell_rows;
        p.cell_cols = a->cell_cols;
        p.grid_r = grid_r;
        p.grid_c = grid_c;
        p.band_rows = a->cell_rows ? a->cell_rows : 64;
        p.bands = (a->rows + p.band_rows - 1) / p.band_rows;
        p.blocks = (a->cols + kTileCols - 1) / kTileCols;
        p.n_tiles = int64_t(a->n_images) * p.bands * p.blocks;
        return launch_fast(p, a->k, ncl, st);
    }
    GenericParams g{};
    g.px = a->d_pixels;
    g.img_stride = a->img_stride;
    g.pitch = a->pitch;
    g.rows = a->rows;
    g.cols = a->cols;
    g.n_images = a->n_images;
    g.k = a->k;
    g.codes = a->d_codes;
    g.codes_img_stride = a->codes_img_stride;
    g.codes_pitch = a->codes_pitch;
    g.hist = a->d_hist;
    g.nbins = nbins;
    g.cell_rows = a->cell_rows;
    g.cell_cols = a->cell_cols;
    g.grid_r = grid_r;
    g.grid_c = grid_c;
    const int64_t total = int64_t(a->rows) * a->cols * a->n_images;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 32LL * n_sms())));
    ldp_generic_kernel<<<grid, 256, 0, st>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "ldp_generic_kernel launch");
    return ALDP_OK;
}

}  // namespace aldp_b200

using namespace aldp_b200;

extern "C" {

aldp_status aldp_ldp_batch(const aldp_ldp_args* args, void* stream) {
    return run_batch(args, ALDP_KERNEL_AUTO, static_cast<cudaStream_t>(stream));
}

aldp_status aldp_ldp_batch_ex(const aldp_ldp_args* args, int kernel, void* stream) {
    if (kernel < ALDP_KERNEL_AUTO || kernel > ALDP_KERNEL_GENERIC)
        return fail(ALDP_EINVAL, "unknown kernel selector");
    return run_batch(args, kernel, static_cast<cudaStream_t>(stream));
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

const char* aldp_version(void) { return "aldp_b200 0.1.0 sm_100a"; }

}  // extern "C"
