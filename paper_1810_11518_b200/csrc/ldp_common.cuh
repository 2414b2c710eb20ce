// ldp_common.cuh -- shared device helpers for the B200 LDP kernels.
//
// Semantics (reference paths relative to the reference tree):
//   ring order, clockwise from top-left            proj/src/kirsch.cpp:11-12
//   mask i = base ring {-3,-3,5,5,5,-3,-3,-3}
//            rotated by i                          proj/src/kirsch.cpp:15,25
//   code: top-k by (response desc, index asc)      proj/src/descriptors.cpp:83-102
//   bins: ascending rank among popcount-k codes    proj/src/descriptors.cpp:25-45
//
// Kirsch redundancy identity (verified against the reference by the parity
// tests): with r_j the eight ring pixels and S_i the sum of mask i's three
// "+5" pixels, r[(2-i)&7] + r[(3-i)&7] + r[(4-i)&7], and T the ring sum,
//     m_i = 5*S_i - 3*(T - S_i) = 8*S_i - 3*T.
// T is common to all eight responses, so ordering m equals ordering S, ties
// included, and the code depends on S alone (10-bit values, 0..765).
//
// Unique keys: K_i = 64*S_i + W[i] with W strictly decreasing, so a larger
// key means a larger response, or an equal response and a lower index --
// exactly the reference's selection order. K fits in 16 bits (<= 49023), so
// two pixels share one 32-bit register as u16x2 lanes, and the whole
// selection runs on the full-rate VIMNMX/VIMNMX3.U16x2 min/max instructions.
//
// The six-bit tags W are chosen so that the XOR of the tags of any k-subset
// (k != 4) is distinct: XOR-ing the k selected keys' low six bits yields a
// 6-bit id that names the code. A 64-entry table maps id -> code; the
// histogram is counted per id and remapped to bins at flush time.
#pragma once
#include <cstdint>

namespace aldp_b200 {

// Two tag sets. TS 0: W[0..7] = 53, 48, 43, 37, 25, 19, 17, 16; TS 1: the
// same set XOR-ed with 16 and re-sorted, 59, 53, 37, 32, 9, 3, 1, 0 (a
// uniform XOR keeps every k-subset XOR distinct). Both strictly decreasing,
// triple-XOR distinct and k == 4 (XOR, direction-0) distinct; see
// tests/test_host.py::test_tag_set_properties. TS 1's zero tag lets the fast
// kernel form K7 as a plain two-input add (measured faster on the whole-image
// kernel, slower on the cell kernel: DESIGN.md section 6).
template <int TS>
__host__ __device__ constexpr uint32_t kTagT(int i) {
    if constexpr (TS == 0)
        return i == 0 ? 53u : i == 1 ? 48u : i == 2 ? 43u : i == 3 ? 37u
             : i == 4 ? 25u : i == 5 ? 19u : i == 6 ? 17u : 16u;
    else
        return i == 0 ? 59u : i == 1 ? 53u : i == 2 ? 37u : i == 3 ? 32u
             : i == 4 ? 9u : i == 5 ? 3u : i == 6 ? 1u : 0u;
}
__host__ __device__ constexpr uint32_t kTag(int i) { return kTagT<0>(i); }
template <int TS>
constexpr uint32_t kTagAllXorT =
    kTagT<TS>(0) ^ kTagT<TS>(1) ^ kTagT<TS>(2) ^ kTagT<TS>(3) ^ kTagT<TS>(4) ^ kTagT<TS>(5) ^ kTagT<TS>(6) ^ kTagT<TS>(7);
constexpr uint32_t kTagAllXor = kTagAllXorT<0>;
constexpr int kKeyShift = 6;

__host__ __device__ inline int popcount8(unsigned c) {
    int n = 0;
    for (int b = 0; b < 8; ++b) n += (c >> b) & 1u;
    return n;
}

__host__ __device__ inline int binom(int n, int r) {
    if (r < 0 || r > n) return 0;
    int v = 1;
    for (int i = 1; i <= r; ++i) v = v * (n - r + i) / i;
    return v;
}

// Rank of `code` among popcount(code)-bit codes in ascending numeric order:
// ascending value is colex order of the bit sets, rank = sum_j C(p_j, j) over
// the set bit positions p_1 < p_2 < ... (descriptors.cpp:25-45 enumerates
// the same order by scanning c = 0..255).
__host__ __device__ inline int colex_rank(unsigned code) {
    int rank = 0, j = 0;
    for (int p = 0; p < 8; ++p)
        if ((code >> p) & 1u) rank += binom(p, ++j);
    return rank;
}

__host__ __device__ inline uint32_t tag_xor(unsigned code, int ts = 0) {
    uint32_t x = 0;
    for (int i = 0; i < 8; ++i)
        if ((code >> i) & 1u) x ^= ts ? kTagT<1>(i) : kTagT<0>(i);
    return x;
}

// ---- packed u16x2 min/max (VIMNMX / VIMNMX3 on sm_100a) ----
__device__ __forceinline__ uint32_t vmax(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t vmin(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t vmax3(uint32_t a, uint32_t b, uint32_t c) {
    return vmax(vmax(a, b), c);  // ptxas fuses into VIMNMX3.U16x2
}
__device__ __forceinline__ uint32_t vmin3(uint32_t a, uint32_t b, uint32_t c) {
    return vmin(vmin(a, b), c);
}

// max/min(a + b, c) on u16x2 lanes as one VIADDMNMX.U16x2 (b may be an
// immediate): fuses a key's last add into its first comparator.
__device__ __forceinline__ uint32_t vaddmax(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("{.reg .b32 t; add.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t vaddmin(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("{.reg .b32 t; add.u16x2 t, %1, %2; min.u16x2 %0, t, %3;}" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// XOR of the low-six-bit tags of the top-k keys of K[0..7] (u16x2 lanes,
// keys unique per lane). Returns the per-lane id in bits 0-5 / 16-21 plus
// garbage in the other bits (callers mask).
//
// Top-3 set: split into halves {K0..K3}, {K4..K7}; a partial 4-sorter gives
// each half's three largest a1>=a2>=a3 (a1 = max(p,r), {a2,a3} = {x,y} with
// p/q = max/min(K0,K1), r/s = max/min(K2,K3), x = min(p,r), y = max(q,s));
// the top three of the union are then the half-cleaner maxima
// {max(a1,b3), max(a2,b2), max(a3,b1)}. 18 min/max per two pixels.
//
// topk_from_pairs takes the network after its first comparator layer:
// p/q = max/min(K0,K1), r/s = max/min(K2,K3) (half A), same for K4..K7.
template <int K, int TS = 0>
__device__ __forceinline__ uint32_t topk_from_pairs(uint32_t pA, uint32_t qA, uint32_t rA, uint32_t sA,
                                                    uint32_t pB, uint32_t qB, uint32_t rB, uint32_t sB) {
    static_assert(K >= 1 && K <= 7 && K != 4, "k == 4 selects through top4_id");
    if constexpr (K == 1) {
        return vmax(vmax3(pA, rA, pB), rB);
    } else if constexpr (K == 7) {  // complement of the single smallest key
        return kTagAllXorT<TS> * 0x10001u ^ vmin(vmin3(qA, sA, qB), sB);
    } else {
        const uint32_t xA = vmin(pA, rA), yA = vmax(qA, sA);
        const uint32_t xB = vmin(pB, rB), yB = vmax(qB, sB);
        if constexpr (K == 3) {
            const uint32_t a3 = vmin(xA, yA), b3 = vmin(xB, yB);
            const uint32_t c1 = vmax3(pA, rA, b3);
            const uint32_t c2 = vmax3(xA, yA, vmax(xB, yB));
            const uint32_t c3 = vmax3(a3, pB, rB);
            return c1 ^ c2 ^ c3;
        } else if constexpr (K == 2) {  // {max(a1,b2), max(a2,b1)}
            const uint32_t a2 = vmax(xA, yA), b2 = vmax(xB, yB);
            return vmax3(pA, rA, b2) ^ vmax3(a2, pB, rB);
        } else if constexpr (K == 6) {  // complement of the two smallest
            const uint32_t s2A = vmin(xA, yA), s2B = vmin(xB, yB);
            return kTagAllXorT<TS> * 0x10001u ^ vmin3(qA, sA, s2B) ^ vmin3(s2A, qB, sB);
        } else {  // K == 5: complement of the three smallest (dual network)
            const uint32_t s3A = vmax(xA, yA), s3B = vmax(xB, yB);
            const uint32_t e1 = vmin3(qA, sA, s3B);
            const uint32_t e2 = vmin3(xA, yA, vmin(xB, yB));
            const uint32_t e3 = vmin3(s3A, qB, sB);
            return kTagAllXorT<TS> * 0x10001u ^ e1 ^ e2 ^ e3;
        }
    }
}

// k == 4: 70 four-subsets do not fit the 6-bit XOR id, but the tag set keeps
// (XOR of the subset's tags, whether direction 0 is in it) unique (checked on
// the host). Both halves are sorted fully, the bitonic half-cleaner keeps the
// top four {max(a1,b4), max(a2,b3), max(a3,b2), max(a4,b1)}, and bit 6 of
// each lane's id is set when K0 >= the fourth largest. ~33 ops per pair.
__device__ __forceinline__ uint32_t top4_id(uint32_t pA, uint32_t qA, uint32_t rA, uint32_t sA, uint32_t pB,
                                            uint32_t qB, uint32_t rB, uint32_t sB, uint32_t k0) {
    const uint32_t a1 = vmax(pA, rA), a4 = vmin(qA, sA), xA = vmin(pA, rA), yA = vmax(qA, sA);
    const uint32_t a2 = vmax(xA, yA), a3 = vmin(xA, yA);
    const uint32_t b1 = vmax(pB, rB), b4 = vmin(qB, sB), xB = vmin(pB, rB), yB = vmax(qB, sB);
    const uint32_t b2 = vmax(xB, yB), b3 = vmin(xB, yB);
    const uint32_t c1 = vmax(a1, b4), c2 = vmax(a2, b3), c3 = vmax(a3, b2), c4 = vmax(a4, b1);
    const uint32_t t4 = vmin(vmin3(c1, c2, c3), c4);
    // lane of e is 0 iff K0 >= t4 (keys unique): min(e, 1) ^ 1 is the flag
    const uint32_t in0 = (vmin(vmax(k0, t4) ^ k0, 0x00010001u) ^ 0x00010001u) << 6;
    return ((c1 ^ c2 ^ c3 ^ c4) & 0xFFBFFFBFu) | in0;
}

template <int K>
__device__ __forceinline__ uint32_t topk_id(const uint32_t (&k)[8]) {
    return topk_from_pairs<K>(vmax(k[0], k[1]), vmin(k[0], k[1]), vmax(k[2], k[3]), vmin(k[2], k[3]),
                              vmax(k[4], k[5]), vmin(k[4], k[5]), vmax(k[6], k[7]), vmin(k[6], k[7]));
}

// Scalar ring -> code for arbitrary k (1..7), the reference's rule stated as
// "bit i set iff fewer than k keys beat K_i" (keys unique).
__device__ __forceinline__ unsigned ring_code(const int (&r)[8], int k) {
    uint32_t key[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int s = r[(2 - i) & 7] + r[(3 - i) & 7] + r[(4 - i) & 7];
        key[i] = (uint32_t(s) << kKeyShift) | kTag(i);
    }
    unsigned code = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        int beaten = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) beaten += key[j] > key[i];
        code |= unsigned(beaten < k) << i;
    }
    return code;
}

// Ring offsets (dx = row, dy = col), clockwise from the top-left
// (kirsch.cpp:11-12).
__device__ __forceinline__ int ring_dx(int j) { return j <= 2 ? -1 : (j == 3 || j == 7) ? 0 : 1; }
__device__ __forceinline__ int ring_dy(int j) {
    return (j == 0 || j == 6 || j == 7) ? -1 : (j == 1 || j == 5) ? 0 : 1;
}

// Code at (x, y) with every neighbour clamped into [x_lo, x_hi] x [y_lo, y_hi]
// (image.cpp:36-40 applied to the image, or to a cell as windowing.cpp:42
// does by cropping).
__device__ __forceinline__ unsigned clamped_code(const uint8_t* img, int pitch, int x, int y,
                                                 int x_lo, int x_hi, int y_lo, int y_hi, int k) {
    int r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int xx = min(max(x + ring_dx(j), x_lo), x_hi);
        const int yy = min(max(y + ring_dy(j), y_lo), y_hi);
        r[j] = __ldg(img + int64_t(xx) * pitch + yy);  // xx may be -1 (halo row of a band view)
    }
    return ring_code(r, k);
}

// LBP code at (x, y) with clamped neighbours (descriptors.cpp:141-157): bit i
// set when ring neighbour i >= the centre.
__device__ __forceinline__ unsigned clamped_lbp(const uint8_t* img, int pitch, int x, int y,
                                                int x_lo, int x_hi, int y_lo, int y_hi) {
    const int ctr = __ldg(img + size_t(x) * size_t(pitch) + size_t(y));
    unsigned code = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int xx = min(max(x + ring_dx(j), x_lo), x_hi);
        const int yy = min(max(y + ring_dy(j), y_lo), y_hi);
        code |= unsigned(__ldg(img + int64_t(xx) * pitch + yy) >= ctr) << j;
    }
    return code;
}

}  // namespace aldp_b200
