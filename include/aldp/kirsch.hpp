// B200 build of the reference's Kirsch-response API (reference header
// proj/include/aldp/kirsch.hpp, implementation kirsch.cpp:10-208).
// The per-pixel routines below are single-pixel API surface evaluated on the
// host (csrc/aldp_api.cpp); response_field, and every whole-image code or
// histogram, runs on the B200.
#ifndef ALDP_B200_KIRSCH_HPP
#define ALDP_B200_KIRSCH_HPP

#include <array>
#include <cstdint>
#include <vector>

#include "aldp/image.hpp"

namespace aldp {

// A 3x3 compass mask; weights[k][l] applies to pixel (x + k - 1, y + l - 1).
// Mask i is mask 0 (5s on the right column) with its outer ring turned i
// steps (kirsch.cpp:10-29).
struct KirschMask {
    int index = 0;
    std::array<std::array<int, 3>, 3> weights{};
};
const std::array<KirschMask, 8>& standard_masks();

// m_0..m_7, signed, each within [-3825, 3825].
struct ResponseVector {
    std::array<int, 8> m{};
    bool operator==(const ResponseVector&) const = default;
};

// a0..a14: the column partial sums the accelerated path shares between masks.
struct ColumnTerms {
    std::array<int, 15> a{};
    bool operator==(const ColumnTerms&) const = default;
};

// Multiplications / additions performed, accumulated over calls.
struct OpCounter {
    std::uint64_t multiplications = 0, additions = 0;
};

// Nine-tap dot product per mask (72 mul / 64 add per pixel).
ResponseVector responses_naive(const GrayImage& img, int x, int y, BorderPolicy policy = BorderPolicy::Clamp,
                               OpCounter* counter = nullptr);
// The accelerated scheme: fifteen column terms, then three adds per mask.
ColumnTerms column_terms(const GrayImage& img, int x, int y, BorderPolicy policy = BorderPolicy::Clamp,
                         OpCounter* counter = nullptr);
ResponseVector responses_accelerated(const ColumnTerms& terms, OpCounter* counter = nullptr);

enum class ResponsePath { Naive, Accelerated };

// Every pixel's responses in raster order (B200 kernel; both paths agree).
std::vector<ResponseVector> response_field(const GrayImage& img, ResponsePath path,
                                           BorderPolicy policy = BorderPolicy::Clamp);

}  // namespace aldp

#endif  // ALDP_B200_KIRSCH_HPP
