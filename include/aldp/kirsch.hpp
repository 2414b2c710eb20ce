// aldp/kirsch.hpp -- drop-in for the reference's proj/include/aldp/kirsch.hpp.
// These per-pixel helpers are API surface, evaluated on the host; the hot
// path (whole-image codes and histograms) runs on the B200 kernels.
#ifndef ALDP_KIRSCH_HPP
#define ALDP_KIRSCH_HPP

#include <array>
#include <cstdint>
#include <vector>

#include "aldp/image.hpp"

namespace aldp {

/// One 3x3 compass mask: weights[k][l] multiplies pixel (x+k-1, y+l-1).
struct KirschMask {
    int index = 0;
    std::array<std::array<int, 3>, 3> weights{};
};

/// Mask 0 has its +5 column on the right; mask i rotates the outer ring by i
/// steps (reference kirsch.hpp:15-24, kirsch.cpp:10-29).
const std::array<KirschMask, 8>& standard_masks();

/// The eight signed responses m_0..m_7, each in [-3825, 3825].
struct ResponseVector {
    std::array<int, 8> m{};
    bool operator==(const ResponseVector&) const = default;
};

/// The fifteen shared column dot products a0..a14 (reference kirsch.hpp:33-57).
struct ColumnTerms {
    std::array<int, 15> a{};
    bool operator==(const ColumnTerms&) const = default;
};

/// Scalar arithmetic executed by a response routine (accrues across calls).
struct OpCounter {
    std::uint64_t multiplications = 0;
    std::uint64_t additions = 0;
};

ResponseVector responses_naive(const GrayImage& img, int x, int y,
                               BorderPolicy policy = BorderPolicy::Clamp,
                               OpCounter* counter = nullptr);
ColumnTerms column_terms(const GrayImage& img, int x, int y,
                         BorderPolicy policy = BorderPolicy::Clamp,
                         OpCounter* counter = nullptr);
ResponseVector responses_accelerated(const ColumnTerms& terms, OpCounter* counter = nullptr);

enum class ResponsePath { Naive, Accelerated };

std::vector<ResponseVector> response_field(const GrayImage& img, ResponsePath path,
                                           BorderPolicy policy = BorderPolicy::Clamp);

}  // namespace aldp

#endif  // ALDP_KIRSCH_HPP
