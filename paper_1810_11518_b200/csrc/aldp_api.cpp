// aldp_api.cpp -- the C++ drop-in for the reference's public API
// (include/aldp/*.hpp, namespace aldp), built into libaldp_b200.so.
//
// Hot entry points go to the B200 through the C-ABI (include/aldp_cuda.h):
//   ldp_histogram      -> aldp_ldp_histogram      (ref descriptors.cpp:123-139)
//   windowed_features  -> aldp_windowed_features  (ref windowing.cpp:35-63)
//   ldp_code_map       -> aldp_ldp_code_map       (new)
//   lbp_histogram      -> aldp_lbp_histogram      (ref descriptors.cpp:159-168)
//   windowed_features(Lbp) -> aldp_windowed_features (ALDP_DESC_LBP)
//   response_field     -> aldp_response_field     (ref kirsch.cpp:193-208)
//   verify_equivalence -> aldp_verify_equivalence (ref verify.cpp:63-111)
//   verify_image       -> aldp_verify_image       (ref verify.cpp:37-61)
// Status codes become the reference's exceptions: EINVAL ->
// std::invalid_argument, ERANGE -> std::out_of_range, ECUDA/ENOMEM ->
// std::runtime_error.
//
// Per-pixel helpers (responses, column terms, ldp_code, bins, generators)
// are API surface evaluated on the host, written from the reference's
// documented semantics.
#include <cstring>
#include <algorithm>
#include <bit>
#include <cctype>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#include "aldp/descriptors.hpp"
#include "aldp/image.hpp"
#include "aldp/kirsch.hpp"
#include "aldp/verify.hpp"
#include "aldp/windowing.hpp"
#include "aldp_cuda.h"

namespace aldp {

namespace {

void throw_status(aldp_status s) {
    const std::string msg = aldp_last_error();
    switch (s) {
    case ALDP_OK: return;
    case ALDP_EINVAL: throw std::invalid_argument(msg);
    case ALDP_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
    }
}

void need_3x3(const GrayImage& img) {
    if (img.rows() < 3 || img.cols() < 3)
        throw std::invalid_argument("descriptor extraction needs at least a 3x3 image, got " +
                                    std::to_string(img.rows()) + "x" + std::to_string(img.cols()));
}

void need_inside(const GrayImage& img, int x, int y) {
    if (x < 0 || y < 0 || x >= img.rows() || y >= img.cols())
        throw std::out_of_range("pixel (" + std::to_string(x) + "," + std::to_string(y) +
                                ") outside " + std::to_string(img.rows()) + "x" +
                                std::to_string(img.cols()) + " image");
}

void need_dims(int rows, int cols, int minimum) {
    if (rows < minimum || cols < minimum)
        throw std::invalid_argument("image dimensions must be at least " + std::to_string(minimum) +
                                    "x" + std::to_string(minimum));
}

// Ring slots clockwise from the top-left neighbour, as (row, col) offsets.
constexpr int kRing[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, 1}, {1, 1}, {1, 0}, {1, -1}, {0, -1}};

// Column-term table (reference kirsch.hpp:33-52): column offset and the
// (top, middle, bottom) weights of each term, and which three terms form
// each response (reference kirsch.cpp:142-144).
struct TermSpec {
    int dy;
    int w[3];
};
constexpr TermSpec kTerms[15] = {
    {-1, {-3, -3, -3}}, {0, {-3, 0, -3}},  {1, {5, 5, 5}},    {0, {5, 0, -3}},  {1, {5, 5, -3}},
    {-1, {5, -3, -3}},  {1, {5, -3, -3}},  {-1, {5, 5, -3}},  {1, {-3, -3, -3}}, {-1, {5, 5, 5}},
    {-1, {-3, 5, 5}},   {0, {-3, 0, 5}},   {-1, {-3, -3, 5}}, {1, {-3, -3, 5}},  {1, {-3, 5, 5}},
};
constexpr int kUse[8][3] = {{0, 1, 2}, {0, 3, 4},  {5, 3, 6},   {7, 3, 8},
                            {9, 1, 8}, {10, 11, 8}, {12, 11, 13}, {0, 11, 14}};

struct Bins {
    std::array<int, 256> rank{};
    std::array<std::uint8_t, 56> code{};
    Bins() {
        rank.fill(-1);
        int n = 0;
        for (int c = 0; c < 256; ++c)
            if (std::popcount(static_cast<unsigned>(c)) == 3) {
                rank[c] = n;
                code[n++] = static_cast<std::uint8_t>(c);
            }
    }
};
const Bins& bins() {
    static const Bins b;
    return b;
}

}  // namespace

// ---------------------------------------------------------------- image
GrayImage::GrayImage(int rows, int cols) : rows_(rows), cols_(cols) {
    need_dims(rows, cols, 1);
    pixels_.assign(static_cast<std::size_t>(rows) * cols, 0);
}

GrayImage::GrayImage(int rows, int cols, std::vector<std::uint8_t> pixels)
    : rows_(rows), cols_(cols), pixels_(std::move(pixels)) {
    need_dims(rows, cols, 1);
    if (pixels_.size() != static_cast<std::size_t>(rows) * cols)
        throw std::invalid_argument("pixel buffer size does not match dimensions");
}

std::uint8_t GrayImage::sample(int x, int y, BorderPolicy) const {
    return at(std::clamp(x, 0, rows_ - 1), std::clamp(y, 0, cols_ - 1));
}

GrayImage make_constant(int rows, int cols, std::uint8_t value) {
    need_dims(rows, cols, 3);
    return {rows, cols, std::vector<std::uint8_t>(static_cast<std::size_t>(rows) * cols, value)};
}

GrayImage make_gradient(int rows, int cols) {
    need_dims(rows, cols, 3);
    std::vector<std::uint8_t> px(static_cast<std::size_t>(rows) * cols);
    for (int x = 0; x < rows; ++x)
        for (int y = 0; y < cols; ++y)
            px[static_cast<std::size_t>(x) * cols + y] = static_cast<std::uint8_t>(std::min(x + y, 255));
    return {rows, cols, std::move(px)};
}

GrayImage make_checker(int rows, int cols, int cell) {
    need_dims(rows, cols, 3);
    if (cell < 1) throw std::invalid_argument("checker cell must be >= 1");
    std::vector<std::uint8_t> px(static_cast<std::size_t>(rows) * cols);
    for (int x = 0; x < rows; ++x)
        for (int y = 0; y < cols; ++y)
            px[static_cast<std::size_t>(x) * cols + y] = ((x / cell) + (y / cell)) % 2 ? 0 : 255;
    return {rows, cols, std::move(px)};
}

GrayImage make_random(int rows, int cols, std::uint32_t seed) {
    need_dims(rows, cols, 3);
    std::mt19937 engine(seed);
    std::vector<std::uint8_t> px(static_cast<std::size_t>(rows) * cols);
    for (auto& v : px) v = static_cast<std::uint8_t>(engine() & 0xFFu);
    return {rows, cols, std::move(px)};
}

// ---------------------------------------------------------------- kirsch
const std::array<KirschMask, 8>& standard_masks() {
    static const std::array<KirschMask, 8> masks = [] {
        constexpr int base[8] = {-3, -3, 5, 5, 5, -3, -3, -3};
        std::array<KirschMask, 8> m{};
        for (int i = 0; i < 8; ++i) {
            m[i].index = i;
            for (int j = 0; j < 8; ++j)
                m[i].weights[kRing[j][0] + 1][kRing[j][1] + 1] = base[(i + j) % 8];
        }
        return m;
    }();
    return masks;
}

ResponseVector responses_naive(const GrayImage& img, int x, int y, BorderPolicy policy,
                               OpCounter* counter) {
    need_3x3(img);
    need_inside(img, x, y);
    const auto& masks = standard_masks();
    ResponseVector out;
    for (int i = 0; i < 8; ++i) {
        int acc = 0;
        for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l)
                acc += masks[i].weights[k][l] * img.sample(x + k - 1, y + l - 1, policy);
        out.m[i] = acc;
    }
    if (counter) {  // nine products and eight sums per mask, centre zero included
        counter->multiplications += 72;
        counter->additions += 64;
    }
    return out;
}

ColumnTerms column_terms(const GrayImage& img, int x, int y, BorderPolicy policy,
                         OpCounter* counter) {
    need_3x3(img);
    need_inside(img, x, y);
    ColumnTerms t;
    for (int n = 0; n < 15; ++n) {
        const TermSpec& s = kTerms[n];
        int plus = 0, minus = 0, n_plus = 0, n_minus = 0;
        for (int k = 0; k < 3; ++k) {
            const int v = img.sample(x + k - 1, y + s.dy, policy);
            if (s.w[k] == 5) plus += v, ++n_plus;
            if (s.w[k] == -3) minus += v, ++n_minus;
        }
        t.a[n] = 5 * plus - 3 * minus;
        if (counter) {  // factored form as executed: one product per weight group
            counter->multiplications += (n_plus > 0) + (n_minus > 0);
            counter->additions += std::max(n_plus - 1, 0) + std::max(n_minus - 1, 0) +
                                  ((n_plus > 0 && n_minus > 0) ? 1 : 0);
        }
    }
    return t;
}

ResponseVector responses_accelerated(const ColumnTerms& terms, OpCounter* counter) {
    ResponseVector out;
    for (int i = 0; i < 8; ++i) out.m[i] = terms.a[kUse[i][0]] + terms.a[kUse[i][1]] + terms.a[kUse[i][2]];
    if (counter) counter->additions += 16;
    return out;
}

std::vector<ResponseVector> response_field(const GrayImage& img, ResponsePath path, BorderPolicy) {
    need_3x3(img);
    std::vector<ResponseVector> f(img.pixel_count());
    static_assert(sizeof(ResponseVector) == 8 * sizeof(std::int32_t), "ResponseVector is int m[8]");
    throw_status(aldp_response_field(img.pixels().data(), img.rows(), img.cols(),
                                     path == ResponsePath::Naive ? ALDP_PATH_NAIVE : ALDP_PATH_ACCELERATED,
                                     reinterpret_cast<std::int32_t*>(f.data())));
    return f;
}

// ---------------------------------------------------------------- descriptors
std::string descriptor_name(Descriptor d) {
    switch (d) {
    case Descriptor::Lbp: return "LBP";
    case Descriptor::Ldp: return "LDP";
    case Descriptor::Aldp: return "ALDP";
    }
    throw std::invalid_argument("unknown descriptor");
}

Descriptor parse_descriptor(const std::string& name) {
    std::string s(name);
    std::transform(s.begin(), s.end(), s.begin(),
                   [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    if (s == "lbp") return Descriptor::Lbp;
    if (s == "ldp") return Descriptor::Ldp;
    if (s == "aldp") return Descriptor::Aldp;
    throw std::invalid_argument("unknown descriptor '" + name + "' (expected lbp, ldp or aldp)");
}

std::uint8_t ldp_code(const ResponseVector& r, int k) {
    if (k < 1 || k > 7) throw std::invalid_argument("k must be in [1, 7]");
    // bit i iff fewer than k directions beat i under (response desc, index asc)
    unsigned code = 0;
    for (int i = 0; i < 8; ++i) {
        int beaten = 0;
        for (int j = 0; j < 8; ++j) beaten += r.m[j] > r.m[i] || (r.m[j] == r.m[i] && j < i);
        if (beaten < k) code |= 1u << i;
    }
    return static_cast<std::uint8_t>(code);
}

int ldp_bin_index(std::uint8_t code) { return bins().rank[code]; }

std::uint8_t ldp_bin_code(int index) {
    if (index < 0 || index >= 56) throw std::out_of_range("bin index must be in [0, 56)");
    return bins().code[static_cast<std::size_t>(index)];
}

std::uint64_t LdpHistogram::total() const {
    return std::accumulate(bins.begin(), bins.end(), std::uint64_t{0});
}

LdpHistogram ldp_histogram(const GrayImage& img, int k, ResponsePath path) {
    if (k != 3) throw std::invalid_argument("the 56-bin histogram layout requires k == 3");
    need_3x3(img);
    LdpHistogram h;
    throw_status(aldp_ldp_histogram(img.pixels().data(), img.rows(), img.cols(), k,
                                    path == ResponsePath::Naive ? ALDP_PATH_NAIVE
                                                                : ALDP_PATH_ACCELERATED,
                                    h.bins.data()));
    return h;
}

std::uint64_t LbpHistogram::total() const {
    return std::accumulate(bins.begin(), bins.end(), std::uint64_t{0});
}

std::uint8_t lbp_code(const GrayImage& img, int x, int y, BorderPolicy policy, OpCounter* counter) {
    need_3x3(img);
    need_inside(img, x, y);
    const int centre = img.sample(x, y, policy);
    unsigned code = 0;
    for (int i = 0; i < 8; ++i)
        code |= unsigned(img.sample(x + kRing[i][0], y + kRing[i][1], policy) >= centre) << i;
    if (counter) counter->additions += 8;  // one threshold compare per neighbour
    return static_cast<std::uint8_t>(code);
}

LbpHistogram lbp_histogram(const GrayImage& img, BorderPolicy) {
    need_3x3(img);
    LbpHistogram h;
    throw_status(aldp_lbp_histogram(img.pixels().data(), img.rows(), img.cols(), h.bins.data()));
    return h;
}

std::vector<std::uint8_t> ldp_code_map(const GrayImage& img, int k, ResponsePath path) {
    if (k < 1 || k > 7) throw std::invalid_argument("k must be in [1, 7]");
    need_3x3(img);
    std::vector<std::uint8_t> codes(img.pixel_count());
    throw_status(aldp_ldp_code_map(img.pixels().data(), img.rows(), img.cols(), k,
                                   path == ResponsePath::Naive ? ALDP_PATH_NAIVE
                                                               : ALDP_PATH_ACCELERATED,
                                   codes.data()));
    return codes;
}

// ---------------------------------------------------------------- windowing
WindowGrid make_grid(const GrayImage& img, int window) {
    if (window < 3) throw std::invalid_argument("window side must be >= 3, got " + std::to_string(window));
    if (window > img.rows() || window > img.cols())
        throw std::invalid_argument("window side " + std::to_string(window) + " exceeds image " +
                                    std::to_string(img.rows()) + "x" + std::to_string(img.cols()));
    return WindowGrid{window, img.rows() / window, img.cols() / window};
}

GrayImage crop(const GrayImage& img, int x0, int y0, int rows, int cols) {
    if (x0 < 0 || y0 < 0 || rows < 1 || cols < 1 || x0 + rows > img.rows() || y0 + cols > img.cols())
        throw std::out_of_range("crop region outside image");
    std::vector<std::uint8_t> px;
    px.reserve(static_cast<std::size_t>(rows) * cols);
    for (int x = 0; x < rows; ++x) {
        const auto row = img.pixels().begin() + static_cast<std::ptrdiff_t>(x0 + x) * img.cols() + y0;
        px.insert(px.end(), row, row + cols);
    }
    return {rows, cols, std::move(px)};
}

std::vector<std::vector<std::uint64_t>> windowed_features(const GrayImage& img, int window,
                                                          Descriptor descriptor) {
    const WindowGrid grid = make_grid(img, window);
    const std::size_t nb = descriptor == Descriptor::Lbp ? 256 : 56;
    const int sel = descriptor == Descriptor::Lbp   ? ALDP_DESC_LBP
                    : descriptor == Descriptor::Ldp ? ALDP_PATH_NAIVE
                                                    : ALDP_PATH_ACCELERATED;
    std::vector<std::uint64_t> flat(static_cast<std::size_t>(grid.total()) * nb);
    throw_status(aldp_windowed_features(img.pixels().data(), img.rows(), img.cols(), window, sel,
                                        flat.data(), flat.size()));
    std::vector<std::vector<std::uint64_t>> out;
    out.reserve(static_cast<std::size_t>(grid.total()));
    for (int w = 0; w < grid.total(); ++w)
        out.emplace_back(flat.begin() + static_cast<std::ptrdiff_t>(w) * nb,
                         flat.begin() + static_cast<std::ptrdiff_t>(w + 1) * nb);
    return out;
}

// ---------------------------------------------------------------- verify
namespace {
VerifyResult from_c(const aldp_verify_result& r) {
    VerifyResult v;
    v.images_checked = r.images_checked;
    v.pixels_checked = r.pixels_checked;
    if (r.has_mismatch)
        v.mismatch = Mismatch{r.image_index, r.x, r.y, r.direction, r.naive_value, r.accelerated_value};
    return v;
}
aldp_fault to_c(const FaultInjection& f) { return aldp_fault{f.image_index, f.x, f.y, f.term_index, f.delta}; }
}  // namespace

VerifyResult verify_equivalence(int images, std::uint32_t seed, std::optional<FaultInjection> fault,
                                int threads) {
    aldp_verify_result r{};
    const aldp_fault f = fault ? to_c(*fault) : aldp_fault{};
    throw_status(aldp_verify_equivalence(images, seed, fault ? &f : nullptr, threads, &r));
    return from_c(r);
}

VerifyResult verify_image(const GrayImage& img, std::optional<FaultInjection> fault, int image_index) {
    need_3x3(img);
    aldp_verify_result r{};
    const aldp_fault f = fault ? to_c(*fault) : aldp_fault{};
    throw_status(aldp_verify_image(img.pixels().data(), img.rows(), img.cols(), fault ? &f : nullptr,
                                   image_index, &r));
    return from_c(r);
}

}  // namespace aldp

extern "C" aldp_status aldp_make_random(uint8_t* out, int rows, int cols, uint32_t seed) {
    if (!out || rows < 3 || cols < 3) return ALDP_EINVAL;
    const aldp::GrayImage img = aldp::make_random(rows, cols, seed);
    std::memcpy(out, img.pixels().data(), img.pixels().size());
    return ALDP_OK;
}
