// ldp_fast.cuh -- the packed sm_100a LDP kernel (product hot path).
//
// Work unit: a "tile" = one image band (band_rows rows; in cell mode one cell
// row) x 128 columns. A warp runs two tiles at once, one per 16-lane
// segment; each lane owns 8 adjacent columns (one 8-byte load per row) and
// slides down the band with three unpacked rows in registers and three raw
// rows in flight (software prefetch, distance 3).
//
// Per lane and row, the 8 columns become four u16x2 pixel pairs with
// stride-2 packing: word j (columns y+4j .. y+4j+3) gives A = (y+4j, y+4j+2)
// and B = (y+4j+1, y+4j+3); the pair "P_A" has left/centre/right columns
// (L, A, B) and "P_B" has (A, B, R), where L/R are A/B shifted by one column
// (built with one byte permute from the neighbouring register; the segment
// edges get their neighbour through a rotating shuffle and one halo load).
// Pixel values are pre-scaled by 64 so every key K_i = 64*S_i + W[i] is one
// 3-input add (ldp_common.cuh).
//
// Histograms: per warp, per segment, one 64-entry u32 table per cell the
// tile touches, counted by RED.shared.add (B200 serves same-address and
// random-address shared reductions at ~1 warp-op/clk/SM -- measured, see
// tools/microbench/atoms.cu -- so no replication is needed). Each table sits
// 256 B after a private copy of the id->code table, so one address gives
// both the code lookup (LDS [a-256]) and the count (RED [a]).
//
// Cell mode (windowed_features semantics, every cell clamped as its own
// image): the map always uses the whole-image clamp. Histogram counts differ
// only on cell borders: the band's first/last row is recounted in the main
// loop with the outside row replaced by the row itself; border columns are
// masked out of the main count and recounted afterwards from clamped loads.
#pragma once

namespace aldp_b200 {

constexpr int kFastWarps = 8;
constexpr int kSegLanes = 16;
constexpr int kLaneCols = 8;
constexpr int kTileCols = kSegLanes * kLaneCols;  // 128
constexpr int kMaxTileCells = 3;
constexpr uint32_t kScaleMask = 0x3FC03FC0u;  // bytes 0 and 2 of a word, scaled by 64
// Per-warp shared layout: for each segment kMaxTileCells regions + 1 trash
// region; a region is [id->code table copy (256 B) | counts (256 B)].
constexpr int kRegion = 512;
constexpr int kSegRegions = kMaxTileCells + 1;
constexpr int kWarpSmem = 2 * kSegRegions * kRegion;  // 4 KB
constexpr int kFixList = 16;                           // fix columns per segment (max)
constexpr int kL2Ahead = 12;                           // rows of L2 prefetch ahead of the load

struct FastParams {
    const uint8_t* px;
    int64_t img_stride;
    int pitch, rows, cols, n_images;
    uint8_t* codes;
    int64_t codes_img_stride;
    int codes_pitch;
    uint32_t* hist;
    int nbins;
    int cell_rows, cell_cols, grid_r, grid_c;  // cell mode only
    int band_rows, bands, blocks;
    int64_t n_tiles;
    uint8_t id_code[64];  // XOR id -> code (0 where no code has that id)
    uint8_t id_bin[64];   // XOR id -> histogram bin (colex rank of the code)
};

struct Raw {
    uint2 w;     // columns y..y+7
    uint32_t h;  // halo word (segment lane 15: left, lane 0: right)
};

// Unpacked row: pairs and their horizontal pair sums.
struct Row8 {
    uint32_t L0, A0, B0, R0, L1, A1, B1, R1;
    uint32_t la0, ab0, br0, la1, ab1, br1;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    return __byte_perm(a, b, s);
}

// Keys of one pixel pair from its left/centre/right column registers of rows
// a (above), b, c (below) and the pair sums lc = l + c, cr = c + r. Ring:
// TL=a.l T=a.c TR=a.r R=b.r BR=c.r B=c.c BL=c.l L=b.l (kirsch.cpp:11-12);
// S_i = r[(2-i)&7] + r[(3-i)&7] + r[(4-i)&7].
struct Col {
    uint32_t l, c, r, lc, cr;
};

template <int K>
__device__ __forceinline__ uint32_t pair_id(const Col& a, const Col& b, const Col& c) {
    constexpr uint32_t T0 = kTag(0) * 0x10001u, T1 = kTag(1) * 0x10001u, T2 = kTag(2) * 0x10001u,
                       T3 = kTag(3) * 0x10001u, T4 = kTag(4) * 0x10001u, T5 = kTag(5) * 0x10001u,
                       T6 = kTag(6) * 0x10001u, T7 = kTag(7) * 0x10001u;
    uint32_t k[8];
    k[0] = a.r + b.r + c.r + T0;  // TR + R + BR
    k[1] = a.cr + b.r + T1;       // T + TR + R
    k[2] = a.lc + a.r + T2;       // TL + T + TR
    k[3] = a.lc + b.l + T3;       // L + TL + T
    k[4] = a.l + b.l + c.l + T4;  // BL + L + TL
    k[5] = c.lc + b.l + T5;       // B + BL + L
    k[6] = c.lc + c.r + T6;       // BR + B + BL
    k[7] = c.cr + b.r + T7;       // R + BR + B
    return topk_id<K>(k);
}

__device__ __forceinline__ Col colA(const Row8& r, int j) {  // pair P_A of word j
    return j == 0 ? Col{r.L0, r.A0, r.B0, r.la0, r.ab0} : Col{r.L1, r.A1, r.B1, r.la1, r.ab1};
}
__device__ __forceinline__ Col colB(const Row8& r, int j) {  // pair P_B of word j
    return j == 0 ? Col{r.A0, r.B0, r.R0, r.ab0, r.br0} : Col{r.A1, r.B1, r.R1, r.ab1, r.br1};
}

// ids of the lane's 8 pixels for output row b: X[0..3] = P_A(0), P_B(0),
// P_A(1), P_B(1); each holds two 6-bit ids (bits 0-5 and 16-21).
template <int K>
__device__ __forceinline__ void row_ids(const Row8& a, const Row8& b, const Row8& c, uint32_t (&X)[4]) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        X[2 * j] = pair_id<K>(colA(a, j), colA(b, j), colA(c, j));
        X[2 * j + 1] = pair_id<K>(colB(a, j), colB(b, j), colB(c, j));
    }
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void red_shared(uint32_t addr) {
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr));
}

template <int K, bool CELLS>
__global__ void __launch_bounds__(kFastWarps * 32, 2) ldp_fast_kernel(FastParams p) {
    extern __shared__ __align__(512) uint8_t smem[];
    __shared__ uint8_t id_bin[64];
    __shared__ int fix_cols[kFastWarps][2][kFixList];
    __shared__ int fix_n[kFastWarps][2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int seg = lane >> 4, sl = lane & 15;
    const uint32_t smem_base = uint32_t(__cvta_generic_to_shared(smem));
    const uint32_t warp_base = smem_base + warp * kWarpSmem;
    const uint32_t seg_base = warp_base + seg * kSegRegions * kRegion;

    // id -> code table copies (one per region) and zeroed counts.
    {
        uint32_t* w = reinterpret_cast<uint32_t*>(smem);
        const int words = kFastWarps * kWarpSmem / 4;
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
            const int in_region = i & (kRegion / 4 - 1);
            w[i] = in_region < 64 ? uint32_t(p.id_code[in_region]) : 0u;
        }
        if (threadIdx.x < 64) id_bin[threadIdx.x] = p.id_bin[threadIdx.x];
    }
    __syncthreads();

    const int64_t tiles_per_image = int64_t(p.bands) * p.blocks;
    const int64_t warp_global = int64_t(blockIdx.x) * kFastWarps + warp;
    const int64_t warp_stride = int64_t(gridDim.x) * kFastWarps;
    const uint32_t src_prev = uint32_t((lane & 16) | ((lane + 15) & 15));
    const uint32_t src_next = uint32_t((lane & 16) | ((lane + 1) & 15));
    const uint32_t trash = seg_base + kMaxTileCells * kRegion + 256;

    for (int64_t pair = warp_global; 2 * pair < p.n_tiles; pair += warp_stride) {
        const int64_t tile = 2 * pair + seg;
        const bool seg_live = tile < p.n_tiles;
        const int64_t t = seg_live ? tile : p.n_tiles - 1;
        const int img = int(t / tiles_per_image);
        const int rem = int(t - int64_t(img) * tiles_per_image);
        const int band = rem / p.blocks, blk = rem - band * p.blocks;
        const int r0 = band * p.band_rows;
        const int seg_rows = seg_live ? min(p.rows, r0 + p.band_rows) - r0 : 0;
        const int n_rows = max(seg_rows, __shfl_xor_sync(0xffffffffu, seg_rows, 16));
        const int c0 = blk * kTileCols;
        const int y = c0 + sl * kLaneCols;
        const uint8_t* img_px = p.px + int64_t(img) * p.img_stride;
        const bool grid_band = !CELLS || band < p.grid_r;
        const bool do_hist = p.hist != nullptr && seg_live && grid_band;

        // ---- column clamp (image.cpp:36-40) as aligned offsets + selectors ----
        const int last = p.cols - 1;
        int halo_off;
        uint32_t halo_sel;
        {
            const int col = sl == 15 ? c0 - 4 : c0 + kTileCols;
            const int a = min(max(col, 0), last & ~3);
            halo_off = a;
            halo_sel = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) halo_sel |= uint32_t(min(max(col + j, 0), last) - a) << (4 * j);
        }
        const bool halo_lane = sl == 0 || sl == 15;
        const uint32_t halo_rot = sl == 15 ? 30u : 6u;  // B form (bytes 1,3) / A form (bytes 0,2)
        // Own 8 columns come from one aligned 8-byte window; a tile crossing
        // the right image edge selects bytes so columns past it repeat the
        // last pixel (warp-uniform branch; never taken for widths % 128 == 0).
        const bool any_edge = __any_sync(0xffffffffu, c0 + kTileCols > p.cols);
        const int own_off = min(y, last & ~7);
        uint32_t sel0 = 0x3210u, sel1 = 0x7654u;
        if (any_edge) {
            sel0 = sel1 = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sel0 |= uint32_t(min(y + j, last) - own_off) << (4 * j);
                sel1 |= uint32_t(min(y + 4 + j, last) - own_off) << (4 * j);
            }
        }

        auto load_raw = [&](int r) -> Raw {
            const uint8_t* rowp = img_px + int64_t(min(max(r, 0), p.rows - 1)) * p.pitch;
            // pull a row further ahead into L2 so the register prefetch hits L2
            if (sl == 1) {
                const uint8_t* ahead = img_px + int64_t(min(max(r + kL2Ahead, 0), p.rows - 1)) * p.pitch + c0;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ahead));
            }
            Raw q;
            q.w = __ldg(reinterpret_cast<const uint2*>(rowp + own_off));
            q.h = halo_lane ? __ldg(reinterpret_cast<const uint32_t*>(rowp + halo_off)) : 0u;
            return q;
        };
        auto unpack = [&](const Raw& q) -> Row8 {
            uint32_t w0 = q.w.x, w1 = q.w.y;
            if (any_edge) {
                w0 = prmt(q.w.x, q.w.y, sel0);
                w1 = prmt(q.w.x, q.w.y, sel1);
            }
            const uint32_t hv = prmt(q.h, q.h, halo_sel);
            const uint32_t h = __funnelshift_l(hv, hv, halo_rot) & kScaleMask;
            Row8 r;
            r.A0 = (w0 << 6) & kScaleMask;
            r.B0 = (w0 >> 2) & kScaleMask;
            r.A1 = (w1 << 6) & kScaleMask;
            r.B1 = (w1 >> 2) & kScaleMask;
            const uint32_t xb = sl == 15 ? h : r.B1;
            const uint32_t ya = sl == 0 ? h : r.A0;
            const uint32_t prevB = __shfl_sync(0xffffffffu, xb, src_prev);
            const uint32_t nextA = __shfl_sync(0xffffffffu, ya, src_next);
            r.L0 = prmt(r.B0, prevB, 0x1076);  // (y-1, y+1)
            r.R0 = prmt(r.A0, r.A1, 0x5432);   // (y+2, y+4)
            r.L1 = prmt(r.B1, r.B0, 0x1076);   // (y+3, y+5)
            r.R1 = prmt(r.A1, nextA, 0x5432);  // (y+6, y+8)
            r.la0 = r.L0 + r.A0;
            r.ab0 = r.A0 + r.B0;
            r.br0 = r.B0 + r.R0;
            r.la1 = r.L1 + r.A1;
            r.ab1 = r.A1 + r.B1;
            r.br1 = r.B1 + r.R1;
            return r;
        };

        // ---- histogram slots: region address per pixel (or trash) ----
        const int cell_c0 = CELLS ? c0 / p.cell_cols : 0;
        uint32_t slot[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int col = y + s;
            bool on = do_hist && col < p.cols;
            int lc = 0;
            if (CELLS) {
                const int cc = col / p.cell_cols, in = col - cc * p.cell_cols;
                on = on && cc < p.grid_c && !(in == 0 && col > 0) && !(in == p.cell_cols - 1 && col < last);
                lc = cc - cell_c0;
            }
            slot[s] = on ? seg_base + uint32_t(lc) * kRegion + 256 : trash;
        }
        // map slots of the four pairs: P_A(0) lo/hi = 0/2, P_B(0) = 1/3, P_A(1) = 4/6, P_B(1) = 5/7
        uint8_t* dst = p.codes ? p.codes + int64_t(img) * p.codes_img_stride : nullptr;
        const bool any_hist = __any_sync(0xffffffffu, do_hist);
        const bool lane_out = seg_live && y < p.cols;

        // Slot addresses of the 8 pixel ids: pair q covers slots (lo, hi) =
        // (q/2*4 + q%2, +2). The id sits in bits 0-5 (lo) and 16-21 (hi):
        // lo offset = (X*4) & 0xFC, hi offset = (X >> 14) & 0xFC (the shift
        // as a multiply-high so it issues on the FMA pipe, not the ALU).
        auto addrs = [&](const uint32_t (&X)[4], uint32_t (&ad)[8]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int s_lo = (q >> 1) * 4 + (q & 1), s_hi = s_lo + 2;
                ad[s_lo] = ((X[q] * 4u) & 0xFCu) | slot[s_lo];
                ad[s_hi] = (__umulhi(X[q], 1u << 18) & 0xFCu) | slot[s_hi];
            }
        };

        auto step = [&](const Row8& a, const Row8& b, const Row8& c, int i) {
            uint32_t X[4], ad[8];
            row_ids<K>(a, b, c, X);
            addrs(X, ad);
            const bool live = i < seg_rows;
            if (dst) {
                uint32_t e[8];
#pragma unroll
                for (int s = 0; s < 8; ++s) e[s] = lds32(ad[s] - 256);
                // bytes -> words with multiply-adds (FMA pipe): code < 256
                const uint32_t w0 = e[0] + e[1] * 0x100u + e[2] * 0x10000u + e[3] * 0x1000000u;
                const uint32_t w1 = e[4] + e[5] * 0x100u + e[6] * 0x10000u + e[7] * 0x1000000u;
                if (live && lane_out)
                    *reinterpret_cast<uint2*>(dst + int64_t(r0 + i) * p.codes_pitch + y) = make_uint2(w0, w1);
            }
            if (any_hist) {
                if (CELLS && (i == 0 || i == p.cell_rows - 1)) {
                    // cell border row: count with the outside row clamped to the cell
                    uint32_t Y[4], bd[8];
                    row_ids<K>(i == 0 ? b : a, b, i == p.cell_rows - 1 ? b : c, Y);
                    addrs(Y, bd);
                    if (live)
#pragma unroll
                        for (int s = 0; s < 8; ++s) red_shared(bd[s]);
                } else if (live) {
#pragma unroll
                    for (int s = 0; s < 8; ++s) red_shared(ad[s]);
                }
            }
        };

        // ---- main loop: rows r0 .. r0+n_rows-1, unrolled by 3 ----
        Row8 ra = unpack(load_raw(r0 - 1));
        Row8 rb = unpack(load_raw(r0));
        Row8 rc = unpack(load_raw(r0 + 1));
        Raw q0 = load_raw(r0 + 2), q1 = load_raw(r0 + 3), q2 = load_raw(r0 + 4);
        for (int i = 0; i < n_rows; i += 3) {
            step(ra, rb, rc, i);
            if (i + 1 >= n_rows) break;
            ra = unpack(q0);
            q0 = load_raw(r0 + i + 5);
            step(rb, rc, ra, i + 1);
            if (i + 2 >= n_rows) break;
            rb = unpack(q1);
            q1 = load_raw(r0 + i + 6);
            step(rc, ra, rb, i + 2);
            if (i + 3 >= n_rows) break;
            rc = unpack(q2);
            q2 = load_raw(r0 + i + 7);
        }

        // ---- cell border columns: recount with the cell clamp ----
        if (CELLS && __any_sync(0xffffffffu, do_hist)) {
            int* fl = fix_cols[warp][seg];
            if (sl == 0) {
                int n = 0;
                if (do_hist) {
                    const int c_end = min(c0 + kTileCols, p.grid_c * p.cell_cols);
                    for (int cc = cell_c0; cc * p.cell_cols < c_end; ++cc) {
                        const int left = cc * p.cell_cols, right = left + p.cell_cols - 1;
                        if (left >= c0 && left > 0 && n < kFixList) fl[n++] = left;
                        if (right >= c0 && right < c_end && right < last && n < kFixList) fl[n++] = right;
                    }
                }
                fix_n[warp][seg] = n;
            }
            __syncwarp();
            const int items = fix_n[warp][seg] * seg_rows;
            const int max_items = max(items, __shfl_xor_sync(0xffffffffu, items, 16));
            const int x_lo = r0, x_hi = r0 + p.cell_rows - 1;
            for (int base = 0; base < max_items; base += 2 * kSegLanes) {
                // two border pixels per lane, one per u16x2 half
                uint32_t rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                uint32_t addr[2] = {trash, trash};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int it = base + sl + kSegLanes * h;
                    if (it >= items) continue;
                    const int col = fl[it / seg_rows];
                    const int x = r0 + it % seg_rows;
                    const int cc = col / p.cell_cols;
                    const int y_lo = cc * p.cell_cols, y_hi = y_lo + p.cell_cols - 1;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int xx = min(max(x + ring_dx(q), x_lo), x_hi);
                        const int yy = min(max(col + ring_dy(q), y_lo), y_hi);
                        rv[q] |= uint32_t(__ldg(img_px + int64_t(xx) * p.pitch + yy)) << (16 * h + 6);
                    }
                    addr[h] = seg_base + uint32_t(cc - cell_c0) * kRegion + 256;
                }
                // ring slots: 0 TL, 1 T, 2 TR, 3 R, 4 BR, 5 B, 6 BL, 7 L
                const Col a{rv[0], rv[1], rv[2], rv[0] + rv[1], rv[1] + rv[2]};
                const Col b{rv[7], 0u, rv[3], 0u, 0u};
                const Col c{rv[6], rv[5], rv[4], rv[6] + rv[5], rv[5] + rv[4]};
                const uint32_t X = pair_id<K>(a, b, c);
                red_shared(((X << 2) & 0xFCu) | addr[0]);
                red_shared(((X >> 14) & 0xFCu) | addr[1]);
            }
        }
        __syncwarp();

        // ---- flush: one global atomic per (cell, bin) seen, then re-zero ----
        if (p.hist != nullptr) {
            const int ntab = !do_hist ? 0 : CELLS ? min(c0 + kTileCols, min(p.cols, p.grid_c * p.cell_cols)) > c0
                                                       ? (min(c0 + kTileCols, min(p.cols, p.grid_c * p.cell_cols)) - 1) / p.cell_cols - cell_c0 + 1
                                                       : 0
                                                 : 1;
            const int64_t cells_per_image = CELLS ? int64_t(p.grid_r) * p.grid_c : 1;
            for (int j = sl; j < ntab * 64; j += kSegLanes) {
                const int lc = j >> 6, id = j & 63;
                uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + (seg_base - smem_base) + lc * kRegion + 256);
                const uint32_t v = cnt[id];
                if (v) {
                    const int64_t cell = CELLS ? int64_t(band) * p.grid_c + cell_c0 + lc : 0;
                    atomicAdd(p.hist + (int64_t(img) * cells_per_image + cell) * p.nbins + id_bin[id], v);
                    cnt[id] = 0;
                }
            }
            // the trash region may have collected counts: clear it too
            uint32_t* tr = reinterpret_cast<uint32_t*>(smem + (trash - smem_base));
            for (int j = sl; j < 64; j += kSegLanes) tr[j] = 0;
        }
        __syncwarp();
    }
}

}  // namespace aldp_b200
