// aldp/descriptors.hpp -- drop-in for the reference's
// proj/include/aldp/descriptors.hpp (LDP part) plus the new code-map entry.
// ldp_histogram and ldp_code_map run on the B200 through the C-ABI.
#ifndef ALDP_B200_DESCRIPTORS_HPP
#define ALDP_B200_DESCRIPTORS_HPP

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "aldp/image.hpp"
#include "aldp/kirsch.hpp"

namespace aldp {

enum class Descriptor { Lbp, Ldp, Aldp };

std::string descriptor_name(Descriptor d);            // "LBP" / "LDP" / "ALDP"
Descriptor parse_descriptor(const std::string& name);  // case-insensitive

/// Top-k directions by (response desc, index asc): exactly k bits. 1 <= k <= 7.
std::uint8_t ldp_code(const ResponseVector& responses, int k = 3);

/// Rank of a three-bit code among the 56 in ascending order (7 -> 0); -1
/// for other popcounts.
int ldp_bin_index(std::uint8_t code);
std::uint8_t ldp_bin_code(int index);  // inverse; index in [0, 56)

struct LdpHistogram {
    std::array<std::uint64_t, 56> bins{};
    std::uint64_t total() const;
    bool operator==(const LdpHistogram&) const = default;
};

/// 56-bin code histogram over every pixel, clamped borders; k must be 3.
/// Runs on the B200 (both paths: outputs identical by contract).
LdpHistogram ldp_histogram(const GrayImage& img, int k, ResponsePath path);

struct LbpHistogram {
    std::array<std::uint64_t, 256> bins{};
    std::uint64_t total() const;
    bool operator==(const LbpHistogram&) const = default;
};

/// Binary pattern of the 3x3 neighbourhood: ring neighbour i (clockwise
/// from the top-left) contributes 2^i when >= the centre. Host helper.
std::uint8_t lbp_code(const GrayImage& img, int x, int y, BorderPolicy policy = BorderPolicy::Clamp,
                      OpCounter* counter = nullptr);

/// 256-bin pattern histogram over every pixel (clamped borders), on the B200.
LbpHistogram lbp_histogram(const GrayImage& img, BorderPolicy policy = BorderPolicy::Clamp);

/// NEW: the whole-image code map, codes[x*cols+y] = ldp_code(responses(x,y), k),
/// on the B200. Any k in [1, 7].
std::vector<std::uint8_t> ldp_code_map(const GrayImage& img, int k = 3,
                                       ResponsePath path = ResponsePath::Accelerated);

}  // namespace aldp

#endif  // ALDP_B200_DESCRIPTORS_HPP
