// ldp_fast.cuh -- the packed sm_100a LDP kernel (product hot path).
//
// Work unit: a "tile" = one image band (band_rows rows; in cell mode one cell
// row) x 128 columns. A tile is processed by a segment of 128/(4*NW) lanes;
// each lane owns NW 4-byte words (4*NW adjacent columns) and slides down the
// band with three unpacked rows in registers and three raw rows in flight
// (software prefetch, distance 3) plus an L2 prefetch further ahead. The
// library instantiates NW = 2 (16-lane segments, two tiles per warp); NW = 1
// (32-lane segments, one tile per warp) compiles but measured slower.
//
// Per lane and row, each word becomes two u16x2 pixel pairs with stride-2
// packing: word j (columns y+4j .. y+4j+3) gives A = (y+4j, y+4j+2) and
// B = (y+4j+1, y+4j+3); pair "P_A" has left/centre/right columns (L, A, B),
// pair "P_B" has (A, B, R), where L/R are A/B shifted by one column (one byte
// permute from the neighbouring register; segment edges get their neighbour
// through a rotating shuffle and one halo load). Pixel values are pre-scaled
// by 64, so a key K_i = 64*S_i + W[i] (ldp_common.cuh) is a sum of three
// pixel registers and its tag; pair_id never forms the eight keys: the first
// comparator layer compares the one pixel in which two neighbouring
// directions differ and adds the two they share afterwards.
//
// Histograms: per warp, per segment, one 64-entry u32 table per cell the
// tile touches, counted by RED.shared.add (B200 serves same-address shared
// reductions without serialisation -- measured, tools/microbench/atoms.cu).
// Each table sits 256 B after a private copy of the id->code table, so one
// address serves both the code lookup (LDS [a-256]) and the count (RED [a]).
//
// Cell mode (windowed_features semantics, every cell clamped as its own
// image): the map always uses the whole-image clamp; histogram counts differ
// only on cell borders. The band's first/last row is recounted in the main
// loop with the outside row replaced by the row itself; border columns are
// masked out of the main count and recounted afterwards from clamped loads.
#pragma once
#include <type_traits>

#ifndef ALDP_SIMPLE
#define ALDP_SIMPLE 1
#endif


namespace aldp_b200 {

constexpr int kFastWarps = 8;
constexpr int kTileCols = 128;
constexpr int kMaxTileCells = 5;
constexpr uint32_t kScaleMask = 0x3FC03FC0u;  // bytes 0 and 2 of a word, scaled by 64
constexpr int kNarrowTileCells = 16;  // narrow cells (>= 9 columns): up to 16 per 128-column tile
constexpr int kFixList = 16;          // border columns per segment (max), regular tiles
// Shared-memory layout of one fast-kernel CTA (the launcher sizes the
// dynamic allocation from it): per (warp, segment) NC + 1 regions, one per
// cell a tile can touch plus a trash region. Regular tiles (NC =
// kMaxTileCells): an LDP region holds a copy of the id -> code table, then
// the counts (CNT bytes in), so one slot address serves the code lookup
// (LDS [a - CNT]) and the count (RED [a]); LBP: 256 counts. Narrow tiles (NC
// = kNarrowTileCells, LDP k != 4 only): count-only regions and one code table
// per segment after them (one more LOP3 per pixel for its address). Each
// region's table and counts are stored XOR-permuted by a bank skew
// (slot_skew) so that lanes of different segments or cells that hold the
// same id hit different banks.
template <int K, int NW, int NC = kMaxTileCells>
struct FastLayout {
    static constexpr bool NARROW = NC > kMaxTileCells;
    static_assert(!NARROW || (K != 0 && K != 4), "narrow tiles: LDP with 64 ids only");
    static constexpr int NT = K == 0 ? 256 : (K == 4 ? 128 : 64);  // table entries (codes / ids)
    static constexpr int CNT = (K == 0 || NARROW) ? 0 : NT * 4;     // offset of the counts in a region
    static constexpr int REGION = K == 0 ? 1024 : (NARROW ? NT * 4 : 2 * NT * 4);
    static constexpr int NSEG = 32 / (kTileCols / (4 * NW));
    static constexpr int REGIONS = NC + 1 + (NARROW ? 1 : 0);  // cells, trash (, code table)
    static constexpr int SEG_SMEM = REGIONS * REGION;
    static constexpr int BYTES = kFastWarps * NSEG * SEG_SMEM + REGION;  // + alignment slack
    static constexpr int FIX = NARROW ? 2 * NC + 2 : kFixList;          // border columns per segment
};

#ifndef ALDP_PIXEL_LAYER
#define ALDP_PIXEL_LAYER 1  // first comparator layer on single pixels (pair_id); 0 = keys formed first (round 1)
#endif
#ifndef ALDP_PROBE
#define ALDP_PROBE 0  // 1: drop the row loop's code lookup and count (wrong output; ceiling probe)
#endif
#ifndef ALDP_MINB
#define ALDP_MINB 2  // CTAs per SM the register allocation targets (NW = 2)
#endif
#ifndef ALDP_KEYS
#define ALDP_KEYS 2  // odd keys of tag set 0 formed on the FMA pipe: 0 = none, 2 = K1/K7, 3 = all four (A/B: DESIGN 6)
#endif
// Bank skew (word XOR, < 32) of segment `seg`'s region `lc`.
__host__ __device__ constexpr uint32_t slot_skew(int seg, int lc) { return uint32_t(seg * 16 + lc * 8) & 31u; }

constexpr int kL2Ahead = 12;                      // rows of L2 prefetch ahead of the load

struct FastParams {
    const uint8_t* px;
    int64_t img_stride;
    int pitch, rows, cols, n_images;
    uint8_t* codes;
    int64_t codes_img_stride;
    int codes_pitch;
    uint32_t* hist;
    int nbins;
    int hist16;  // 1: hist holds uint16 counts (two bins per 32-bit word)
    int cell_rows, cell_cols, grid_r, grid_c;  // cell mode only
    int cell_clamp;                            // cell mode: 1 = per-cell clamp, 0 = cut from the code map
    int edge_lo, edge_hi;                      // band rows recounted with the cell clamp (-1: none)
    int row_lo, row_hi;                        // rows readable as neighbours (-1 / rows with halos)
    // exact division by per-launch constants, n < 2^31: q = (n * m) >> sh
    // (m = floor(2^sh / d) + 1, sh = 32 + ceil(log2 d); host: magic_div)
    uint64_t mg_group, mg_bandG, mg_band1, mg_blocks, mg_cell;
    int sh_group, sh_bandG, sh_band1, sh_blocks, sh_cell;
    int band_rows, bands, blocks;
    int uniform_bands;  // rows is a multiple of band_rows: no band is shorter
    int64_t n_tiles;
    // narrow cells: store the cells wholly inside a tile, add the ones that
    // straddle a tile edge (zeroed beforehand by zero_straddling_cells)
    int store_whole;
    uint32_t one;         // 1 at run time: multiplier that keeps integer adds on the FMA pipe
    uint8_t id_code[128];  // id -> code (0 where no code has that id); 7-bit ids for k == 4
    uint8_t id_bin[128];   // id -> histogram bin (colex rank of the code)
    uint8_t bin_id[64];    // histogram bin -> id (narrow cells stored whole)
};

// Tag set of a fast-kernel instantiation (ldp_common.cuh kTagT): the cell
// kernel keeps set 0, the whole-image kernel takes set 1.
__host__ __device__ constexpr int fast_tag_set(bool cells) { return cells ? 0 : 1; }

// hist[idx] += v on uint32 counts, or on uint16 counts packed two per word
// (a count never reaches 65536 there, so the add cannot carry across bins)
__device__ __forceinline__ void hist_add(uint32_t* hist, int hist16, int64_t idx, uint32_t v) {
    atomicAdd(hist + (idx >> hist16), v << ((uint32_t(idx) & uint32_t(hist16)) << 4));  // branch-free
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint64_t m, int sh) {
    return uint32_t((uint64_t(n) * m) >> sh);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    return __byte_perm(a, b, s);
}

// Integer add issued as IMAD (FMA pipe) instead of IADD3 (ALU pipe): B200's
// ALU pipe also runs every min/max of the selection network, so moving adds
// off it raises throughput (tools/microbench/viadd.cu + ncu pipe counts:
// IADD3 -> ALU, IMAD/VIADD -> FMA). `one` is 1 but unknown to the compiler.
__device__ __forceinline__ uint32_t fadd(uint32_t a, uint32_t b, uint32_t one) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
    return r;
}

// a + IMM on the FMA pipe (IMAD with the unknown-to-the-compiler `one`)
template <uint32_t IMM>
__device__ __forceinline__ uint32_t faddc(uint32_t a, uint32_t one) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "n"(IMM));
    return r;
}
// Column registers of one pixel pair: left/centre/right and the pair sums
// lc = l + c, cr = c + r (all scaled by 64).
struct Col {
    uint32_t l, c, r, lc, cr;
};

// Keys of one pixel pair from rows a (above), b, c (below). Ring: TL=a.l
// T=a.c TR=a.r R=b.r BR=c.r B=c.c BL=c.l L=b.l (kirsch.cpp:11-12);
// S_i = r[(2-i)&7] + r[(3-i)&7] + r[(4-i)&7].
template <int K, int TS = 0>
__device__ __forceinline__ uint32_t pair_id(const Col& a, const Col& b, const Col& c, uint32_t one) {
    constexpr uint32_t T0 = kTagT<TS>(0) * 0x10001u, T1 = kTagT<TS>(1) * 0x10001u, T2 = kTagT<TS>(2) * 0x10001u,
                       T3 = kTagT<TS>(3) * 0x10001u, T4 = kTagT<TS>(4) * 0x10001u, T5 = kTagT<TS>(5) * 0x10001u,
                       T6 = kTagT<TS>(6) * 0x10001u, T7 = kTagT<TS>(7) * 0x10001u;
#if ALDP_PIXEL_LAYER
    if constexpr (K != 4) {
        // First comparator layer on single pixels (round 2, the kept key
        // scheme). The paired keys share two ring pixels (K0/K1: TR+R, K2/K3:
        // TL+T, K4/K5: BL+L, K6/K7: BR+B) and differ in one, so
        //   max/min(K_2i, K_2i+1) = C_i + max/min(u + D_i, v),
        // D_i = W[2i] - W[2i+1] > 0, C_i = the shared pair + W[2i+1]. No key
        // is formed before the layer: its eight VIADDMNMX take pixel operands
        // and the tag difference as the immediate add. The shared sums and the
        // adds that complete the maxima run on the FMA pipe (IMAD); for k == 3
        // each half's minima meet only in max(q, s), so one of them rides that
        // comparator's add. The row loop's ALU-pipe instructions drop from
        // 324 to 300 per 24 pixels at the same total (the ALU pipe, which runs
        // every min/max, is what the kernel waits on: an ALU instruction costs
        // ~2.8 FMA-pipe ones in the A/B series,
        // profiles/r02m_pixel_layer_ab.txt). The cell kernel (sums on use)
        // forms the horizontal sums on the FMA pipe too; the whole-image
        // kernel adds the tag to its stored row sums. k == 4 keeps the keys
        // formed first (top4_id needs K0 itself; this layer measured 1 %
        // slower there).
        constexpr uint32_t D01 = T0 - T1, D23 = T2 - T3, D45 = T4 - T5, D67 = T6 - T7;
        const uint32_t C01 = fadd(faddc<T1>(a.r, one), b.r, one), C45 = fadd(faddc<T5>(c.l, one), b.l, one);
        uint32_t C23, C67;
        if constexpr (TS == 0) {
            C23 = fadd(faddc<T3>(a.l, one), a.c, one);
            C67 = fadd(faddc<T7>(c.r, one), c.c, one);
        } else {
            C23 = a.lc + T3;
            C67 = c.cr + T7;
        }
        const uint32_t M01 = vaddmax(c.r, D01, a.c), m01 = vaddmin(c.r, D01, a.c);
        const uint32_t M23 = vaddmax(a.r, D23, b.l), m23 = vaddmin(a.r, D23, b.l);
        const uint32_t M45 = vaddmax(a.l, D45, c.c), m45 = vaddmin(a.l, D45, c.c);
        const uint32_t M67 = vaddmax(c.l, D67, b.r), m67 = vaddmin(c.l, D67, b.r);
        const uint32_t pA = fadd(M01, C01, one), rA = fadd(M23, C23, one);
        const uint32_t pB = fadd(M45, C45, one), rB = fadd(M67, C67, one);
        const uint32_t sA = fadd(m23, C23, one), sB = fadd(m67, C67, one);
        if constexpr (K == 3) {
            const uint32_t yA = vaddmax(m01, C01, sA), yB = vaddmax(m45, C45, sB);  // max(q, s)
            const uint32_t xA = vmin(pA, rA), xB = vmin(pB, rB);
            const uint32_t a3 = vmin(xA, yA), b3 = vmin(xB, yB);
            const uint32_t c1 = vmax3(pA, rA, b3);
            const uint32_t c2 = vmax3(xA, yA, vmax(xB, yB));
            const uint32_t c3 = vmax3(a3, pB, rB);
            return c1 ^ c2 ^ c3;
        } else {
            return topk_from_pairs<K, TS>(pA, fadd(m01, C01, one), rA, sA, pB, fadd(m45, C45, one), rB, sB);
        }
    } else
#endif
    if constexpr (TS == 1) {
        // Tag set 1 (the whole-image kernel; A/B: +6 % on C3, -5.9 % if used
        // by the cell kernel): the first-layer pairs share a two-input
        // partial each (P = TR+R, Q = TL+T, R = BL+L, U = B+BR), the even
        // keys' last add is fused into the comparator, K7 (tag 0) is a
        // two-input add, and only K1/K3/K5 take a three-input IADD3.
        static_assert(K < 0 || kTagT<TS>(7) == 0, "tag set 1 has K7's tag 0");
        const uint32_t P = a.r + b.r, R = b.l + c.l;
        const uint32_t x0 = P + T0, x2 = a.lc + T2, x4 = R + T4, x6 = c.cr + T6;
        const uint32_t k1 = P + a.c + T1, k3 = a.lc + b.l + T3, k5 = R + c.c + T5;
        const uint32_t k7 = c.cr + b.r;
        if constexpr (K == 4)
            return top4_id(vaddmax(x0, c.r, k1), vaddmin(x0, c.r, k1), vaddmax(x2, a.r, k3), vaddmin(x2, a.r, k3),
                           vaddmax(x4, a.l, k5), vaddmin(x4, a.l, k5), vaddmax(x6, c.l, k7), vaddmin(x6, c.l, k7),
                           fadd(x0, c.r, one));
        else
            return topk_from_pairs<K, TS>(vaddmax(x0, c.r, k1), vaddmin(x0, c.r, k1), vaddmax(x2, a.r, k3),
                                          vaddmin(x2, a.r, k3), vaddmax(x4, a.l, k5), vaddmin(x4, a.l, k5),
                                          vaddmax(x6, c.l, k7), vaddmin(x6, c.l, k7));
    } else {
        // Tag set 0 (the cell kernel): odd keys materialised by one IADD3
        // each, the even keys' last add fused into the first comparator layer
        // (one pre-add + VIADDMNMX): 16 instructions per pair. Measured and
        // rejected for this kernel: sums on the FMA pipe
        // (IMAD), the tag-set-1 scheme above, FMA-pipe slot addresses.
#if ALDP_KEYS >= 2
        const uint32_t k1 = fadd(faddc<T1>(a.cr, one), b.r, one), k7 = fadd(faddc<T7>(c.cr, one), b.r, one);
#else
        const uint32_t k1 = a.cr + b.r + T1, k7 = c.cr + b.r + T7;
#endif
#if ALDP_KEYS >= 3
        const uint32_t k3 = fadd(faddc<T3>(a.lc, one), b.l, one), k5 = fadd(faddc<T5>(c.lc, one), b.l, one);
#else
        const uint32_t k3 = a.lc + b.l + T3, k5 = c.lc + b.l + T5;
#endif
#if ALDP_KEYS >= 1
        const uint32_t x0 = fadd(faddc<T0>(a.r, one), b.r, one), x4 = fadd(faddc<T4>(a.l, one), b.l, one);
#else
        const uint32_t x0 = a.r + b.r + T0, x4 = a.l + b.l + T4;   // + c.r / + c.l fused
#endif
        const uint32_t x2 = a.lc + T2, x6 = c.lc + T6;             // + a.r / + c.r fused
        if constexpr (K == 4)
            return top4_id(vaddmax(x0, c.r, k1), vaddmin(x0, c.r, k1), vaddmax(x2, a.r, k3), vaddmin(x2, a.r, k3),
                           vaddmax(x4, c.l, k5), vaddmin(x4, c.l, k5), vaddmax(x6, c.r, k7), vaddmin(x6, c.r, k7),
                           fadd(x0, c.r, one));
        else
            return topk_from_pairs<K>(vaddmax(x0, c.r, k1), vaddmin(x0, c.r, k1), vaddmax(x2, a.r, k3),
                                      vaddmin(x2, a.r, k3), vaddmax(x4, c.l, k5), vaddmin(x4, c.l, k5),
                                      vaddmax(x6, c.r, k7), vaddmin(x6, c.r, k7));
    }
}

// LBP codes of one pixel pair (descriptors.cpp:141-157): bit i set when ring
// neighbour i >= the centre, ring clockwise from the top-left. Each compare is
// one borrow-free add (values < 2^15, so bit 15/31 of r + 0x8000 - c is the
// result); four byte permutes in sign-replicate mode turn the eight result
// bits per lane into 0x00/0xFF bytes, a select chain + fold packs them.
// Returns the low pixel's code in byte 0 and the high pixel's in byte 1.
__device__ __forceinline__ uint32_t pair_lbp(const Col& a, const Col& b, const Col& c, uint32_t one) {
    // 0x8000 - ctr per lane, once; the eight compares are then 2-input adds
    // kept on the FMA pipe (the LBP kernel is ALU-bound)
    const uint32_t nctr = 0x80008000u - b.c;
    const uint32_t r[8] = {a.l, a.c, a.r, b.r, c.r, c.c, c.l, b.l};
    uint32_t d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = fadd(r[i], nctr, one);
    // m = [lo bit i, hi bit i, lo bit i+1, hi bit i+1] as 0x00 / 0xFF bytes:
    // PTX prmt with selector nibbles 8|byte replicates the selected byte's
    // sign bit (__byte_perm masks that bit off, hence the inline PTX)
    auto sgn = [](uint32_t x, uint32_t y) {
        uint32_t r;
        asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(r) : "r"(x), "r"(y));
        return r;
    };
    const uint32_t m01 = sgn(d[0], d[1]), m23 = sgn(d[2], d[3]);
    const uint32_t m45 = sgn(d[4], d[5]), m67 = sgn(d[6], d[7]);
    // bytes 0/1: bits 0,2,4,6 of lo/hi; bytes 2/3: bits 1,3,5,7
    constexpr uint32_t C01 = 0x02020101u, C23 = 0x08080404u, C45 = 0x20201010u;
    uint32_t t = (m45 & C45) | (m67 & ~C45);
    t = (m23 & C23) | (t & ~C23);
    t = (m01 & C01) | (t & ~C01);
    t &= 0xAAAA5555u;
    return t + (t >> 16);  // disjoint bits: add == or
}

// One unpacked row of a lane: per word j, A/B/L/R and the three pair sums.
template <int NW>
struct RowN {
    uint32_t A[NW], B[NW], L[NW], R[NW];
    uint32_t la[NW], ab[NW], br[NW];  // filled only when the kernel keeps row sums
};

// SUMS: 2 = take the row's three stored pair sums; 1 = store only ab (shared
// by both pairs of a word) and add la/br on use; 0 = add all on use (fewest
// live registers for the register-tight cell-mode kernel, a few more adds).
template <int SUMS, int NW>
__device__ __forceinline__ Col colA(const RowN<NW>& r, int j) {  // pair P_A of word j
    if constexpr (SUMS == 2) return Col{r.L[j], r.A[j], r.B[j], r.la[j], r.ab[j]};
    else if constexpr (SUMS == 1) return Col{r.L[j], r.A[j], r.B[j], r.L[j] + r.A[j], r.ab[j]};
    else return Col{r.L[j], r.A[j], r.B[j], r.L[j] + r.A[j], r.A[j] + r.B[j]};
}
template <int SUMS, int NW>
__device__ __forceinline__ Col colB(const RowN<NW>& r, int j) {  // pair P_B of word j
    if constexpr (SUMS == 2) return Col{r.A[j], r.B[j], r.R[j], r.ab[j], r.br[j]};
    else if constexpr (SUMS == 1) return Col{r.A[j], r.B[j], r.R[j], r.ab[j], r.B[j] + r.R[j]};
    else return Col{r.A[j], r.B[j], r.R[j], r.A[j] + r.B[j], r.B[j] + r.R[j]};
}

template <int NW>
struct RawN {
    uint32_t w[NW];  // columns y .. y+4NW-1
    uint32_t h;      // halo word (segment's last lane: left halo, lane 0: right halo)
};

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void red_shared(uint32_t addr) {
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr));
}


template <int NW>
__device__ __forceinline__ void load_words(const uint8_t* p, uint32_t (&w)[NW]) {
    if constexpr (NW == 1) {
        w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
    } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        w[0] = v.x;
        w[1] = v.y;
    }
}

// K = 1..7 (not 4): LDP with top-K codes; K = 0: LBP (descriptors.cpp:141-168).
// HALO: the view is a band of a taller resident frame (rows -1 / rows are
// real neighbours); a separate instantiation keeps the common path's row
// clamp a compile-time [0, rows) (a runtime bound measured 1.8 % slower).
template <int K, int NW, bool CELLS, bool CODES, bool HIST, bool HALO = false, int NC = kMaxTileCells>
__global__ void __launch_bounds__(kFastWarps * 32, NW == 1 ? 3 : ALDP_MINB) ldp_fast_kernel(FastParams p) {
    constexpr bool LBP = K == 0;
    constexpr int TS = fast_tag_set(CELLS);  // the host builds the id tables for the same set
    using Lay = FastLayout<K, NW, NC>;
    constexpr bool NARROW = Lay::NARROW;
    constexpr int REGION = Lay::REGION, CNT = Lay::CNT, NT = Lay::NT, SEG_SMEM = Lay::SEG_SMEM;
    constexpr int LC = 4 * NW;              // columns per lane
    constexpr int SEG = kTileCols / LC;     // lanes per segment (tile)
    constexpr int NSEG = 32 / SEG;          // tiles per warp
    constexpr int NPAIR = 2 * NW;           // u16x2 pixel pairs per lane
    constexpr unsigned FULL = 0xffffffffu;
#ifndef ALDP_CELL_SUMS
#define ALDP_CELL_SUMS 0
#endif
    constexpr int SUMS = CELLS ? ALDP_CELL_SUMS : 2;  // measured: all stored sums win only without cells
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(4) uint8_t id_bin[128];
    __shared__ __align__(4) uint8_t bin_id[NARROW ? 64 : 4];
    __shared__ int fix_cols[kFastWarps][NSEG][Lay::FIX];
    __shared__ int fix_n[kFastWarps][NSEG];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int seg = lane / SEG, sl = lane % SEG;
    // Regions must be REGION-aligned in the shared window: a slot address is
    // formed as (id * 4) ^ (region | skew * 4), so the region's low bits must
    // be zero. The host allocates REGION extra bytes for this alignment.
    const uint32_t raw_base = uint32_t(__cvta_generic_to_shared(smem));
    const uint32_t smem_base = (raw_base + REGION - 1) & ~uint32_t(REGION - 1);
    uint8_t* const smem_al = smem + (smem_base - raw_base);
    const uint32_t seg_base = smem_base + (warp * NSEG + seg) * SEG_SMEM;

    // LDP: id -> code table copies (one per region, in the region's skewed
    // order); zeroed counts.
    {
        uint32_t* w = reinterpret_cast<uint32_t*>(smem_al);
        const int words = kFastWarps * NSEG * SEG_SMEM / 4;
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
            const int in_region = i & (REGION / 4 - 1);
            const int region = (i / (REGION / 4)) % Lay::REGIONS, sg = (i / (SEG_SMEM / 4)) % NSEG;
            const bool table = !LBP && (NARROW ? region == NC + 1 : in_region < NT);
            w[i] = table ? uint32_t(p.id_code[NARROW ? in_region : in_region ^ slot_skew(sg, region)]) : 0u;
        }
        if (!LBP && threadIdx.x < NT) id_bin[threadIdx.x] = p.id_bin[threadIdx.x];
        if (NARROW && threadIdx.x < 64) bin_id[threadIdx.x] = p.bin_id[threadIdx.x];
    }
    __syncthreads();

    const int64_t tiles_per_image = int64_t(p.bands) * p.blocks;
    // Tile order: groups of G images (G = 2 when an image row has an odd
    // number of 128-column blocks), band-major inside a group, so the two
    // tiles a warp runs together always share a band (same height) -- the
    // warp then takes the predicate-free path. Neighbouring bands of an image
    // stay close in time, so band halos hit L2.
    const int G = (p.blocks & 1) ? 2 : 1;
    // 32-bit index math whenever the tile count allows it (a 64-bit divide
    // is a ~100-instruction software routine; this runs 3x per tile)
    const bool small_t = p.n_tiles < (int64_t(1) << 30);
    const uint32_t group_tiles = uint32_t(G * tiles_per_image);
    auto tile_coords = [&](int64_t tt, int& img_, int& band_, int& blk_) {
        int64_t grp;
        uint32_t t_in;
        if (small_t) {
            const uint32_t q = fdiv(uint32_t(tt), p.mg_group, p.sh_group);
            grp = q;
            t_in = uint32_t(tt) - q * group_tiles;
        } else {
            grp = tt / (G * tiles_per_image);
            t_in = uint32_t(tt - grp * G * tiles_per_image);
        }
        const int64_t left_ = p.n_images - grp * G;
        const int gi = left_ < G ? int(left_) : G;  // images in this group
        const uint32_t per_band = uint32_t(gi * p.blocks);
        band_ = int(gi == G ? fdiv(t_in, p.mg_bandG, p.sh_bandG) : fdiv(t_in, p.mg_band1, p.sh_band1));
        const int rem_ = int(t_in - uint32_t(band_) * per_band);
        const int q_ = int(fdiv(uint32_t(rem_), p.mg_blocks, p.sh_blocks));
        img_ = int(grp * G) + q_;
        blk_ = rem_ - q_ * p.blocks;
    };
    const int64_t warp_global = int64_t(blockIdx.x) * kFastWarps + warp;
    const int64_t warp_stride = int64_t(gridDim.x) * kFastWarps;
    const uint32_t seg_lane0 = uint32_t(seg * SEG);
    const uint32_t src_prev = seg_lane0 + uint32_t((sl + SEG - 1) % SEG);
    const uint32_t src_next = seg_lane0 + uint32_t((sl + 1) % SEG);
    // masked pixels count here; codes-only launches look codes up here too
    const uint32_t trash = seg_base + NC * REGION + CNT + slot_skew(seg, NC) * 4;
    const uint32_t code_tab = seg_base + (NC + 1) * REGION;  // narrow tiles: the segment's id -> code table
    const uint32_t one = p.one;
    // Band b of an image -> first row, height, cell row (cell mode: bands
    // are cell rows, then the rows below the grid, crow == grid_r).
    auto band_geom = [&](int b, int& r0_, int& h_, int& crow_) {
        r0_ = b * p.band_rows;
        h_ = min(p.band_rows, p.rows - r0_);
        crow_ = CELLS ? b : 0;
    };

    for (int64_t wt = warp_global; NSEG * wt < p.n_tiles; wt += warp_stride) {
        const int64_t tile = NSEG * wt + seg;
        const bool seg_live = tile < p.n_tiles;
        const int64_t t = seg_live ? tile : p.n_tiles - 1;
        int img, band, blk;
        tile_coords(t, img, band, blk);
        int r0, band_h, crow;
        band_geom(band, r0, band_h, crow);
        const int seg_rows = seg_live ? band_h : 0;
        // warp-wide row count from warp-uniform quantities only (no shuffle),
        // so the row loop's trip count is known uniform
        // (every band band_rows tall -- the cell grid's launch -- needs no
        // look at the other segment's tile: A/B C5 +0.9 %, window 10 / 25 +2 %)
        int n_rows = p.band_rows;
        if (!p.uniform_bands) {
        n_rows = 0;
#pragma unroll
        for (int sg = 0; sg < NSEG; ++sg) {
            const int64_t tt = NSEG * wt + sg;
            if (tt < p.n_tiles) {
                int im_, bnd, bk_, r0_, h_, cr_;
                tile_coords(tt, im_, bnd, bk_);
                band_geom(bnd, r0_, h_, cr_);
                n_rows = max(n_rows, h_);
            }
        }
        }
        const int c0 = blk * kTileCols;
        const int y = c0 + sl * LC;
        const uint8_t* img_px = p.px + int64_t(img) * p.img_stride;
        const bool grid_band = !CELLS || crow < p.grid_r;
        const int cell_r0 = crow * p.cell_rows;  // cell mode: the cell row's first image row
        const bool do_hist = HIST && seg_live && grid_band;

        // ---- column clamp (image.cpp:36-40) as aligned offsets + selectors ----
        // Halo word of the segment's edge lanes (last lane: the 4 columns left
        // of the tile, lane 0: the 4 right of it), loaded from an aligned
        // window clamped into the row. One byte permute per row turns it into
        // the u16x2 form the neighbour lane needs -- B form (columns c0-3,
        // c0-1) on the left, A form (c0+128, c0+130) on the right -- with the
        // clamp folded into the selector (byte 4 = a zero byte).
        const int last = p.cols - 1;
        int halo_off;
        uint32_t halo_sel;
        {
            const int col = sl == SEG - 1 ? c0 - 4 : c0 + kTileCols;
            const int a = min(max(col, 0), last & ~3);
            halo_off = a;
            const int j0 = sl == SEG - 1 ? 1 : 0;  // B form: columns col+1, col+3; A form: col, col+2
            const uint32_t s0 = uint32_t(min(max(col + j0, 0), last) - a);
            const uint32_t s1 = uint32_t(min(max(col + j0 + 2, 0), last) - a);
            halo_sel = s0 | 0x40u | (s1 << 8) | 0x4000u;
        }
        const bool halo_lane = sl == 0 || sl == SEG - 1;
        // Own columns come from one aligned window of 4*NW bytes; a tile
        // crossing the right image edge selects bytes so columns past it
        // repeat the last pixel (warp-uniform; such a tile is never SIMPLE,
        // and never occurs when the width is a multiple of 128).
        const bool any_edge = __any_sync(FULL, c0 + kTileCols > p.cols);
        const int own_off = min(y, last & ~(LC - 1));
        uint32_t sel[NW];
#pragma unroll
        for (int j = 0; j < NW; ++j) sel[j] = 0x3210u + 0x4444u * j;
        if (any_edge) {
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                sel[j] = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) sel[j] |= uint32_t(min(y + 4 * j + b, last) - own_off) << (4 * b);
            }
        }

        // Row loads: a per-lane row pointer that the row loop advances by one
        // pitch per step (one IADD3 + IMAD.X); the halo word sits at a fixed
        // distance from it. Rows outside [row_lo, row_hi] are clamped only
        // where they can occur: the band's first row and the rows past the
        // image's last one (row loop tail).
        const int row_lo = HALO ? p.row_lo : 0, row_hi = HALO ? p.row_hi : p.rows - 1;
        const int64_t pitch = p.pitch;
        const uint8_t* const own_p = img_px + own_off;
        const int64_t halo_d = int64_t(halo_off) - own_off;
        const uint8_t* const pf_p = img_px + c0;
        auto row_ptr = [&](int r) { return own_p + int64_t(min(max(r, row_lo), row_hi)) * pitch; };
        // r: the row's index (for the L2 prefetch of the whole-image kernel)
        auto load_ptr = [&](const uint8_t* ptr, int r, RawN<NW>& q) {
            if (!CELLS && sl == 1) {  // pull a row further ahead into L2 (measured: pays only without cells)
                const int ra_ = min(r + kL2Ahead, p.rows - 1);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pf_p + (long long)ra_ * p.pitch));
            }
            load_words<NW>(ptr, q.w);
            const uint32_t* hp = reinterpret_cast<const uint32_t*>(ptr + halo_d);  // every lane: no predicated moves
            if (halo_lane) q.h = __ldg(hp);
        };
        // raw row -> A/B/L/R u16x2 forms, scaled by 64 (byte permutes with a
        // zero byte, then IMAD shifts on the FMA pipe)
        auto unpack = [&](auto simple_tag, const RawN<NW>& q) -> RowN<NW> {
            constexpr bool SIMPLE = decltype(simple_tag)::value;
            uint32_t w[NW];
#pragma unroll
            for (int j = 0; j < NW; ++j) w[j] = q.w[j];
            if (!SIMPLE && any_edge) {
#pragma unroll
                for (int j = 0; j < NW; ++j) w[j] = prmt(q.w[0], q.w[NW - 1], NW == 1 ? sel[j] & 0x3333u : sel[j]);
            }
            const uint32_t h = prmt(q.h, 0u, halo_sel) * 64u;
            RowN<NW> r;
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                r.A[j] = prmt(w[j], 0u, 0x4240u) * 64u;  // columns y+4j, y+4j+2
                r.B[j] = prmt(w[j], 0u, 0x4341u) * 64u;  // columns y+4j+1, y+4j+3
            }
            const uint32_t xb = sl == SEG - 1 ? h : r.B[NW - 1];
            const uint32_t ya = sl == 0 ? h : r.A[0];
            const uint32_t prevB = __shfl_sync(FULL, xb, src_prev);
            const uint32_t nextA = __shfl_sync(FULL, ya, src_next);
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                r.L[j] = prmt(r.B[j], j == 0 ? prevB : r.B[j - 1], 0x1076);       // (y+4j-1, y+4j+1)
                r.R[j] = prmt(r.A[j], j == NW - 1 ? nextA : r.A[j + 1], 0x5432);  // (y+4j+2, y+4j+4)
                if constexpr (SUMS >= 1) r.ab[j] = fadd(r.A[j], r.B[j], one);
                if constexpr (SUMS == 2) {
                    r.la[j] = fadd(r.L[j], r.A[j], one);
                    r.br[j] = fadd(r.B[j], r.R[j], one);
                }
            }
            return r;
        };

        // ---- histogram slots: region address | skew per pixel (or trash) ----
        const int cell_c0 = CELLS ? int(fdiv(uint32_t(c0), p.mg_cell, p.sh_cell)) : 0;
        uint32_t slot[LC];
        // one divide per lane: the lane's columns are consecutive, so the
        // cell index / in-cell offset advance by carries (cell_cols >= 3)
        int cc = CELLS ? int(fdiv(uint32_t(y), p.mg_cell, p.sh_cell)) : 0, in = CELLS ? y - cc * p.cell_cols : 0;
#pragma unroll
        for (int s = 0; s < LC; ++s) {
            const int col = y + s;
            bool on = do_hist && col < p.cols;
            int lc = 0;
            if (CELLS) {
                if (s > 0 && ++in == p.cell_cols) in = 0, ++cc;
                on = on && cc < p.grid_c &&
                     (!p.cell_clamp || (!(in == 0 && col > 0) && !(in == p.cell_cols - 1 && col < last)));
                lc = cc - cell_c0;
            }
            slot[s] = on ? seg_base + uint32_t(lc) * REGION + CNT + slot_skew(seg, lc) * 4 : trash;
        }
        // per-lane code-map pointer at row r0; a row's store adds one IMAD.WIDE
        // (advanced one row per step, so the row loop carries no row index)
        const int64_t cpitch = p.codes_pitch;
        uint8_t* st =
            CODES ? p.codes + int64_t(img) * p.codes_img_stride + int64_t(r0) * p.codes_pitch + y : nullptr;
        const bool lane_out = seg_live && y < p.cols;
        // widths that are not a multiple of the lane's 4*NW columns: the lane
        // holding the last column stores its valid bytes one by one
        const bool lane_full = lane_out && y + LC <= p.cols;
        // Common case: every lane of the warp is inside the image and on a
        // live row of equal-height tiles -> no per-lane predication at all.
        const bool simple = __all_sync(FULL, lane_full && seg_rows == n_rows);

        // Slot addresses of the lane's pixel ids. Pair q = 2j (P_A of word
        // j) covers columns y+4j (lo) / y+4j+2 (hi); q = 2j+1 (P_B) covers
        // y+4j+1 / y+4j+3. The id sits in bits 0-5 (lo) and 16-21 (hi).
        // LBP: the pair's two codes sit in bytes 0 and 1 instead.
        auto addrs = [&](const uint32_t (&X)[NPAIR], uint32_t (&ad)[LC]) {
#pragma unroll
            for (int q = 0; q < NPAIR; ++q) {
                const int s_lo = (q >> 1) * 4 + (q & 1), s_hi = s_lo + 2;
                constexpr uint32_t M = (NT - 1) * 4;
                ad[s_lo] = ((X[q] * 4u) & M) ^ slot[s_lo];
                ad[s_hi] = (LBP ? (X[q] >> 6) & M : __umulhi(X[q], 1u << 18) & M) ^ slot[s_hi];
            }
        };
        // narrow tiles: code-table addresses of the same ids
        auto code_addrs = [&](const uint32_t (&X)[NPAIR], uint32_t (&cd)[LC]) {
#pragma unroll
            for (int q = 0; q < NPAIR; ++q) {
                const int s_lo = (q >> 1) * 4 + (q & 1), s_hi = s_lo + 2;
                constexpr uint32_t M = (NT - 1) * 4;
                cd[s_lo] = ((X[q] * 4u) & M) | code_tab;
                cd[s_hi] = (__umulhi(X[q], 1u << 18) & M) | code_tab;
            }
        };
        // count the lane's pixels at slot addresses ad
        auto count = [&](const uint32_t (&ad)[LC]) {
#pragma unroll
            for (int s = 0; s < LC; ++s) red_shared(ad[s]);
        };
        auto row_ids = [&](const RowN<NW>& a, const RowN<NW>& b, const RowN<NW>& c, uint32_t (&X)[NPAIR]) {
#pragma unroll
            for (int j = 0; j < NW; ++j) {
                if constexpr (LBP) {
                    X[2 * j] = pair_lbp(colA<SUMS>(a, j), colA<SUMS>(b, j), colA<SUMS>(c, j), one);
                    X[2 * j + 1] = pair_lbp(colB<SUMS>(a, j), colB<SUMS>(b, j), colB<SUMS>(c, j), one);
                } else {
                    X[2 * j] = pair_id<K, TS>(colA<SUMS>(a, j), colA<SUMS>(b, j), colA<SUMS>(c, j), one);
                    X[2 * j + 1] = pair_id<K, TS>(colB<SUMS>(a, j), colB<SUMS>(b, j), colB<SUMS>(c, j), one);
                }
            }
        };

        // Cell border rows (windowing.cpp:42 crops every cell): with the
        // per-cell clamp the band's first / last row counts its histogram with
        // the outside row replaced by the row itself; the map keeps the
        // whole-image code. Those two rows are peeled out of the row loop.
        const bool clamp_top = HIST && CELLS && grid_band && p.edge_lo == 0 && r0 == cell_r0;
        const bool clamp_bot = HIST && CELLS && grid_band && p.edge_hi >= 0 && r0 + n_rows == cell_r0 + p.cell_rows;

        // One output row. SIMPLE (a std::integral_constant) drops the per-lane
        // live/in-image predicates for warps that need none; EDGE: 0 = a row
        // inside the band, 1 / 2 = the band's first / last row, counted with
        // the cell clamp when `clamp` is set.
        auto step = [&](auto simple_tag, auto edge_tag, const RowN<NW>& a, const RowN<NW>& b, const RowN<NW>& c,
                        int i, bool clamp) {
            constexpr bool SIMPLE = decltype(simple_tag)::value;
            constexpr int EDGE = decltype(edge_tag)::value;
            uint32_t X[NPAIR], ad[LC];
            row_ids(a, b, c, X);
            addrs(X, ad);
            const bool live = SIMPLE || i < seg_rows;
            if (CODES) {
                uint32_t wd[NW];
                if constexpr (LBP) {
#pragma unroll
                    for (int j = 0; j < NW; ++j)  // [A.lo, B.lo, A.hi, B.hi]
                        wd[j] = prmt(X[2 * j], X[2 * j + 1], 0x5140);
                } else {
                    uint32_t e[LC];
                    if constexpr (NARROW) {
                        uint32_t cd[LC];
                        code_addrs(X, cd);
#pragma unroll
                        for (int s = 0; s < LC; ++s) e[s] = lds32(cd[s]);
                    } else {
#pragma unroll
                        for (int s = 0; s < LC; ++s) e[s] = ALDP_PROBE ? ad[s] & 0xFFu : lds32(ad[s] - CNT);
                    }
#pragma unroll
                    for (int j = 0; j < NW; ++j)  // bytes -> word with multiply-adds (FMA pipe)
                        wd[j] = e[4 * j] + e[4 * j + 1] * 0x100u + e[4 * j + 2] * 0x10000u + e[4 * j + 3] * 0x1000000u;
                }
                if (SIMPLE || (live && lane_full)) {
                    if constexpr (NW == 1) *reinterpret_cast<uint32_t*>(st) = wd[0];
                    else *reinterpret_cast<uint2*>(st) = make_uint2(wd[0], wd[1]);
                } else if (live && lane_out) {
                    for (int b = 0; b < p.cols - y; ++b) st[b] = uint8_t(wd[b >> 2] >> (8 * (b & 3)));
                }
                st += cpitch;
            }
            if (HIST) {
                if (EDGE != 0 && clamp) {
                    uint32_t Y[NPAIR], bd[LC];
                    row_ids(EDGE == 1 ? b : a, b, EDGE == 2 ? b : c, Y);
                    addrs(Y, bd);
                    if (live) count(bd);
                } else if (live) {
                    if (!ALDP_PROBE) count(ad);
                }
            }
        };

        // ---- rows r0 .. r0+n_rows-1: first row, 3-way unrolled middle, last row ----
        // Three unpacked rows in registers, three raw rows in flight.
        auto run_rows = [&](auto simple_tag) {
            using E0 = std::integral_constant<int, 0>;
            using E1 = std::integral_constant<int, 1>;
            using E2 = std::integral_constant<int, 2>;
            RawN<NW> q0, q1, q2;
            q0.h = q1.h = q2.h = 0u;
            load_ptr(row_ptr(r0 - 1), r0 - 1, q0);
            load_ptr(row_ptr(r0), r0, q1);
            load_ptr(row_ptr(r0 + 1), r0 + 1, q2);
            RowN<NW> ra = unpack(simple_tag, q0), rb = unpack(simple_tag, q1), rc = unpack(simple_tag, q2);
            load_ptr(row_ptr(r0 + 2), r0 + 2, q0);
            load_ptr(row_ptr(r0 + 3), r0 + 3, q1);
            load_ptr(row_ptr(r0 + 4), r0 + 4, q2);
            if (n_rows == 1) {  // a one-row band (image remainder): never a cell row
                step(simple_tag, E0{}, ra, rb, rc, 0, false);
                return;
            }
            step(simple_tag, E1{}, ra, rb, rc, 0, clamp_top);
            ra = unpack(simple_tag, q0);
            load_ptr(row_ptr(r0 + 5), r0 + 5, q0);
            // rows in registers: rb = i-1, rc = i, ra = i+1; in flight q1, q2, q0 = i+2, i+3, i+4.
            // The unrolled loop loads rows i+5 .. i+7 unclamped, so it stops
            // before they pass row_hi; the tail clamps.
            const uint8_t* ld = row_ptr(r0 + 5);
            const int i_end = min(n_rows - 1, row_hi - r0 - 4);
            int i = 1;
            for (; i + 3 <= i_end; i += 3) {
                step(simple_tag, E0{}, rb, rc, ra, i, false);
                rb = unpack(simple_tag, q1);
                ld += pitch;
                load_ptr(ld, r0 + i + 5, q1);
                step(simple_tag, E0{}, rc, ra, rb, i + 1, false);
                rc = unpack(simple_tag, q2);
                ld += pitch;
                load_ptr(ld, r0 + i + 6, q2);
                step(simple_tag, E0{}, ra, rb, rc, i + 2, false);
                ra = unpack(simple_tag, q0);
                ld += pitch;
                load_ptr(ld, r0 + i + 7, q0);
            }
            for (; i < n_rows - 1; ++i) {  // the rows before the last the loop left
                step(simple_tag, E0{}, rb, rc, ra, i, false);
                rb = rc;
                rc = ra;
                ra = unpack(simple_tag, q1);
                q1 = q2;
                q2 = q0;
                load_ptr(row_ptr(r0 + i + 5), r0 + i + 5, q0);
            }
            step(simple_tag, E2{}, rb, rc, ra, n_rows - 1, clamp_bot);
        };
        if (ALDP_SIMPLE && simple) run_rows(std::integral_constant<bool, true>{});
        else run_rows(std::integral_constant<bool, false>{});

        // ---- cell border columns: recount with the cell clamp ----
        if (HIST && CELLS && p.cell_clamp && __any_sync(FULL, do_hist)) {
            // The segment's border columns, one cell per lane (a tile touches
            // at most SEG cells), compacted in cell order with ballots.
            int* fl = fix_cols[warp][seg];
            {
                const int c_end = min(c0 + kTileCols, p.grid_c * p.cell_cols);
                const int left = (cell_c0 + sl) * p.cell_cols, right = left + p.cell_cols - 1;
                const bool in_tile = do_hist && left < c_end;
                const bool okl = in_tile && left >= c0 && left > 0;
                const bool okr = in_tile && right >= c0 && right < c_end && right < last;
                const unsigned seg_mask = (SEG == 32 ? FULL : ((1u << SEG) - 1u)) << (seg * SEG);
                const unsigned bl = __ballot_sync(FULL, okl) & seg_mask, br = __ballot_sync(FULL, okr) & seg_mask;
                const unsigned below = (1u << lane) - 1u;
                const int pos = __popc(bl & below) + __popc(br & below);
                if (okl) fl[pos] = left;
                if (okr) fl[pos + (okl ? 1 : 0)] = right;
                if (sl == 0) fix_n[warp][seg] = __popc(bl) + __popc(br);
            }
            __syncwarp();
            // Vertical runs: the segment's 2*SEG u16 half-slots split the
            // border columns x rows; each slot slides down one column with a
            // 3-row window of the bytes (col-1, col, col+1), clamped to the cell
            // (rows to the band = cell row, the outside column to the column).
            const int nb = fix_n[warp][seg];
            const int runs_per_col = nb ? max(1, (2 * SEG) / nb) : 1;
            const int run_len = nb ? (seg_rows + runs_per_col - 1) / runs_per_col : 0;
            const int x_lo = cell_r0, x_hi = cell_r0 + p.cell_rows - 1;
            int xs[2], len[2];
            uint32_t wsel[2], addr[2];
            const uint8_t* colp[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int sidx = sl + SEG * h;
                const int ci = sidx / runs_per_col, ri = sidx - ci * runs_per_col;
                const bool act = ci < nb && ri * run_len < seg_rows;
                const int col = act ? fl[ci] : y;
                const int cc = col / max(p.cell_cols, 1);
                const bool left = col == cc * p.cell_cols;
                xs[h] = r0 + ri * run_len;
                len[h] = act ? min(run_len, seg_rows - ri * run_len) : 0;
                const int wo = max(col - 1, 0) & ~3;
                colp[h] = img_px + wo;
                // byte offset of column col-1 inside the 8-byte window at wo;
                // left border: (c, c, r); right border: (l, c, c)
                const uint32_t o = uint32_t(col - 1 - wo);
                wsel[h] = left ? (o + 1) | ((o + 1) << 4) | ((o + 2) << 8) : o | ((o + 1) << 4) | ((o + 1) << 8);
                addr[h] = act ? seg_base + uint32_t(cc - cell_c0) * REGION + CNT + slot_skew(seg, cc - cell_c0) * 4 : trash;
            }
            int n_it = max(len[0], len[1]);
            for (int o = 16; o > 0; o >>= 1) n_it = max(n_it, __shfl_xor_sync(FULL, n_it, o));
            // raw 8-byte windows of one row for both halves (the second word
            // only when it holds column col+1 -- it never leaves the row)
            bool need_hi[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) need_hi[h] = ((wsel[h] >> 8) & 0xFu) >= 4u;
            auto fetch = [&](int rh0, int rh1, uint32_t (&q)[4]) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rr = min(max(h == 0 ? rh0 : rh1, x_lo), x_hi);
                    const uint8_t* ptr = colp[h] + int64_t(rr) * p.pitch;
                    q[2 * h] = __ldg(reinterpret_cast<const uint32_t*>(ptr));
                    q[2 * h + 1] = need_hi[h] ? __ldg(reinterpret_cast<const uint32_t*>(ptr + 4)) : 0u;
                }
            };
            // packed u16x2 (l, c, r) x64 of one row from its raw windows
            auto make_col = [&](const uint32_t (&q)[4]) -> Col {
                const uint32_t w0 = prmt(q[0], q[1], wsel[0]) & 0x00FFFFFFu;
                const uint32_t w1 = prmt(q[2], q[3], wsel[1]) & 0x00FFFFFFu;
                Col c;
                c.l = prmt(w0, w1, 0x7430) << 6;
                c.c = prmt(w0, w1, 0x7531) << 6;
                c.r = prmt(w0, w1, 0x7632) << 6;
                c.lc = fadd(c.l, c.c, one);
                c.cr = fadd(c.c, c.r, one);
                return c;
            };
            uint32_t qa[4], qb[4], qn[4];
            fetch(xs[0] - 1, xs[1] - 1, qa);
            fetch(xs[0], xs[1], qb);
            fetch(xs[0] + 1, xs[1] + 1, qn);
            Col wa = make_col(qa), wb = make_col(qb);
            for (int it = 0; it < n_it; ++it) {
                const Col wc = make_col(qn);
                fetch(xs[0] + it + 2, xs[1] + it + 2, qn);  // next row in flight
                constexpr uint32_t M = (NT - 1) * 4;
                uint32_t X;
                if constexpr (LBP) X = pair_lbp(wa, wb, wc, one);
                else X = pair_id<K, TS>(wa, wb, wc, one);
                red_shared(((X * 4u) & M) ^ (it < len[0] ? addr[0] : trash));
                red_shared(((LBP ? X >> 6 : __umulhi(X, 1u << 18)) & M) ^ (it < len[1] ? addr[1] : trash));
                wa = wb;
                wb = wc;
            }
        }
        __syncwarp();

        // ---- flush: one global atomic per (cell, bin) seen, then re-zero ----
        if (HIST && NARROW && p.store_whole) {
            // Narrow cells: a cell that lies wholly inside this tile is
            // stored -- all its bins, zeros included, four per lane (lanes
            // sl < NB / 4) -- so its histogram needs no memset and no global
            // atomics; a cell that straddles the tile's edge adds its non-zero
            // bins to the histogram zeroed beforehand. Then the tables are
            // re-zeroed.
            constexpr int NB = (K == 1 || K == 7) ? 8 : (K == 2 || K == 6) ? 28 : 56;
            constexpr int G4 = NB / 4;
            const uint8_t* seg_ptr = smem_al + (seg_base - smem_base);
            const int c_end = min(c0 + kTileCols, min(p.cols, p.grid_c * p.cell_cols));
            const int n_c = c_end > c0 ? (c_end - 1) / p.cell_cols - cell_c0 + 1 : 0;
            if (do_hist && sl < G4) {
                const uint32_t ids = reinterpret_cast<const uint32_t*>(bin_id)[sl];  // bins 4 sl .. 4 sl + 3
                const int64_t at0 = ((int64_t(img) * p.grid_r + crow) * p.grid_c + cell_c0) * NB + 4 * sl;
                for (int lc = 0; lc < n_c; ++lc) {
                    const uint32_t* cnt = reinterpret_cast<const uint32_t*>(seg_ptr + lc * REGION + CNT);
                    const uint32_t sk = slot_skew(seg, lc);
                    uint32_t c4[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) c4[j] = cnt[((ids >> (8 * j)) & 0xFFu) ^ sk];
                    const int cf = (cell_c0 + lc) * p.cell_cols;
                    const bool whole = cf >= c0 && cf + p.cell_cols <= c0 + kTileCols;
                    const int64_t at = at0 + int64_t(lc) * NB;  // bins; a multiple of 4
                    if (whole) {
                        if (!p.hist16)
                            *reinterpret_cast<uint4*>(p.hist + at) = make_uint4(c4[0], c4[1], c4[2], c4[3]);
                        else
                            *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(p.hist) + at) =
                                make_uint2(c4[0] | (c4[1] << 16), c4[2] | (c4[3] << 16));
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (c4[j]) hist_add(p.hist, p.hist16, at + j, c4[j]);
                    }
                }
            }
            __syncwarp();
            uint4* tb = reinterpret_cast<uint4*>(smem_al + (seg_base - smem_base));
            for (int j = sl; j < n_c * (REGION / 16); j += SEG) tb[j] = make_uint4(0u, 0u, 0u, 0u);
            uint4* tr = reinterpret_cast<uint4*>(smem_al + (seg_base - smem_base) + NC * REGION + CNT);
            for (int j = sl; j < NT / 4; j += SEG) tr[j] = make_uint4(0u, 0u, 0u, 0u);
        } else if (HIST) {
            int ntab = 0;
            if (do_hist) {
                if (CELLS) {
                    const int c_end = min(c0 + kTileCols, min(p.cols, p.grid_c * p.cell_cols));
                    ntab = c_end > c0 ? (c_end - 1) / p.cell_cols - cell_c0 + 1 : 0;
                } else {
                    ntab = 1;
                }
            }
            const int64_t cells_per_image = CELLS ? int64_t(p.grid_r) * p.grid_c : 1;
            uint8_t* seg_ptr = smem_al + (seg_base - smem_base);
            // four counts per 128-bit load: the bank skew is a multiple of 8
            // words, so words 4g .. 4g+3 hold ids (4g ^ skew) .. + 3
            constexpr int G4 = NT / 4;
            for (int g = sl; g < ntab * G4; g += SEG) {
                const int lc = g / G4, w4 = (g % G4) * 4;
                uint4* q = reinterpret_cast<uint4*>(seg_ptr + lc * REGION + CNT) + (w4 >> 2);
                const uint4 v = *q;
                if (v.x | v.y | v.z | v.w) {
                    const int id0 = w4 ^ int(slot_skew(seg, lc));
                    // bins of ids id0 .. id0+3: one word of the byte table
                    const uint32_t b4 = LBP ? 0u : reinterpret_cast<const uint32_t*>(id_bin)[id0 >> 2];
                    const int64_t base =
                        (int64_t(img) * cells_per_image + (CELLS ? int64_t(crow) * p.grid_c + cell_c0 + lc : 0)) *
                        p.nbins;  // even (every bin count is even)
                    const uint32_t c4[4] = {v.x, v.y, v.z, v.w};
                    if (!p.hist16) {
                        uint32_t* hp = p.hist + base;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (c4[j]) atomicAdd(hp + (LBP ? id0 + j : (b4 >> (8 * j)) & 0xFFu), c4[j]);
                    } else {  // uint16 counts, two bins per word
                        uint32_t* hp = p.hist + (base >> 1);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t bin = LBP ? uint32_t(id0 + j) : (b4 >> (8 * j)) & 0xFFu;
                            if (c4[j]) atomicAdd(hp + (bin >> 1), c4[j] << ((bin & 1u) << 4));
                        }
                    }
                    *q = make_uint4(0u, 0u, 0u, 0u);
                }
            }
            // the trash region collects masked counts: clear it too
            uint4* tr = reinterpret_cast<uint4*>(seg_ptr + NC * REGION + CNT);
            for (int j = sl; j < G4; j += SEG) tr[j] = make_uint4(0u, 0u, 0u, 0u);
        }
        __syncwarp();
    }
}

}  // namespace aldp_b200
