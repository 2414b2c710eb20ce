// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libaldp_ref.so).
//
// TEST INFRASTRUCTURE ONLY: the reference's own CPU implementation, used to
// pin oracle/ldp_oracle.c and as the CPU baseline arm of bench.py
// (`--impl reference`, cpu_baseline.kind = "reference"). Nothing in the
// product path links it.
//
// Every function is a composition of reference calls only:
//   ref_make_random      aldp::make_random                (src/image.cpp:75-83)
//   ref_code_map         aldp::ldp_code(responses_*(...))  (src/descriptors.cpp:83-102,
//                        src/kirsch.cpp:63-84,86-157) -- the reference has no
//                        code-map entry point; this is its per-pixel loop body
//                        (src/descriptors.cpp:129-136)
//   ref_ldp_histogram    aldp::ldp_histogram              (src/descriptors.cpp:123-139)
//   ref_windowed         aldp::windowed_features          (src/windowing.cpp:35-63)
//   ref_cell_histograms  aldp::crop + aldp::ldp_histogram (rectangular cells,
//                        the composition windowed_features performs per window)
//   k == 0 selects LBP: aldp::lbp_code / aldp::lbp_histogram
//                        (src/descriptors.cpp:141-168), windowed_features(Lbp)
//   ref_response_field   aldp::response_field             (src/kirsch.cpp:193-208)
//   ref_verify_*         aldp::verify_equivalence / verify_image (src/verify.cpp:37-111)
//   ref_load_pgm         aldp::load_pgm                   (src/pgm.cpp:59-125)
//   ref_save_pgm         aldp::save_pgm                   (src/pgm.cpp:127-149)
//   ref_op_counts        aldp::measured_ops               (src/bench.cpp:97-116)
//   ref_batch            the above over a batch, std::thread sharded by image
//                        (the reference functions are pure)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <stdexcept>
#include <thread>
#include <vector>

#include "aldp/bench.hpp"
#include "aldp/descriptors.hpp"
#include "aldp/image.hpp"
#include "aldp/kirsch.hpp"
#include "aldp/pgm.hpp"
#include "aldp/verify.hpp"
#include "aldp/windowing.hpp"

namespace {

// 0 ok, 1 invalid_argument, 2 out_of_range, 3 other
template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

aldp::GrayImage wrap(const uint8_t* px, int rows, int cols) {
    return aldp::GrayImage(rows, cols,
                           std::vector<std::uint8_t>(px, px + static_cast<size_t>(rows) * cols));
}

aldp::ResponsePath path_of(int path) {
    return path == 0 ? aldp::ResponsePath::Naive : aldp::ResponsePath::Accelerated;
}

void code_map(const aldp::GrayImage& img, int k, aldp::ResponsePath path, uint8_t* out) {
    if (k == 0) {
        for (int x = 0; x < img.rows(); ++x)
            for (int y = 0; y < img.cols(); ++y)
                out[static_cast<size_t>(x) * img.cols() + y] = aldp::lbp_code(img, x, y);
        return;
    }
    for (int x = 0; x < img.rows(); ++x)
        for (int y = 0; y < img.cols(); ++y) {
            const aldp::ResponseVector r =
                path == aldp::ResponsePath::Naive
                    ? aldp::responses_naive(img, x, y)
                    : aldp::responses_accelerated(aldp::column_terms(img, x, y));
            out[static_cast<size_t>(x) * img.cols() + y] = aldp::ldp_code(r, k);
        }
}

// k == 3 goes through ldp_histogram itself; the reference throws for other k
// (descriptors.cpp:124-126), so for k != 3 the codes are counted into C(8,k)
// ascending bins -- the repo's documented extension.
void histogram(const aldp::GrayImage& img, int k, aldp::ResponsePath path, uint64_t* out) {
    if (k == 0) {
        const aldp::LbpHistogram h = aldp::lbp_histogram(img);
        std::memcpy(out, h.bins.data(), sizeof(uint64_t) * 256);
        return;
    }
    if (k == 3) {
        const aldp::LdpHistogram h = aldp::ldp_histogram(img, 3, path);
        std::memcpy(out, h.bins.data(), sizeof(uint64_t) * 56);
        return;
    }
    int rank[256];
    int nb = 0;
    for (int c = 0; c < 256; ++c) rank[c] = __builtin_popcount(c) == k ? nb++ : -1;
    std::memset(out, 0, sizeof(uint64_t) * nb);
    std::vector<uint8_t> codes(img.pixel_count());
    code_map(img, k, path, codes.data());
    for (uint8_t c : codes) ++out[rank[c]];
}

int n_bins(int k) {
    if (k == 0) return 256;
    int nb = 0;
    for (int c = 0; c < 256; ++c) nb += __builtin_popcount(c) == k;
    return nb;
}

void cell_histograms(const aldp::GrayImage& img, int cr, int cc, int k, aldp::ResponsePath path,
                     uint64_t* out) {
    if (cr == cc && (k == 3 || k == 0)) {  // square windows: the reference entry point itself
        const auto d = k == 0 ? aldp::Descriptor::Lbp
                              : path == aldp::ResponsePath::Naive ? aldp::Descriptor::Ldp : aldp::Descriptor::Aldp;
        const auto feats = aldp::windowed_features(img, cr, d);
        const size_t nb = k == 0 ? 256 : 56;
        for (size_t w = 0; w < feats.size(); ++w)
            std::memcpy(out + w * nb, feats[w].data(), sizeof(uint64_t) * nb);
        return;
    }
    if (cr < 3 || cc < 3 || cr > img.rows() || cc > img.cols())
        throw std::invalid_argument("bad cell size");
    const int gr = img.rows() / cr, gc = img.cols() / cc, nb = n_bins(k);
    for (int r = 0; r < gr; ++r)
        for (int c = 0; c < gc; ++c)
            histogram(aldp::crop(img, r * cr, c * cc, cr, cc), k, path,
                      out + (static_cast<size_t>(r) * gc + c) * nb);
}

}  // namespace

extern "C" {

int ref_make_random(int rows, int cols, uint32_t seed, uint8_t* out) {
    return guarded([&] {
        const aldp::GrayImage img = aldp::make_random(rows, cols, seed);
        std::memcpy(out, img.pixels().data(), img.pixel_count());
    });
}

int ref_responses(const uint8_t* px, int rows, int cols, int x, int y, int path, int32_t* out8) {
    return guarded([&] {
        const aldp::GrayImage img = wrap(px, rows, cols);
        const aldp::ResponseVector r =
            path == 0 ? aldp::responses_naive(img, x, y)
                      : aldp::responses_accelerated(aldp::column_terms(img, x, y));
        for (int i = 0; i < 8; ++i) out8[i] = r.m[i];
    });
}

int ref_ldp_code(const int32_t* m8, int k, uint8_t* out) {
    return guarded([&] {
        aldp::ResponseVector r;
        for (int i = 0; i < 8; ++i) r.m[i] = m8[i];
        *out = aldp::ldp_code(r, k);
    });
}

int ref_ldp_bin_index(int code) { return aldp::ldp_bin_index(static_cast<uint8_t>(code)); }

int ref_code_map(const uint8_t* px, int rows, int cols, int k, int path, uint8_t* out) {
    return guarded([&] {
        const aldp::GrayImage img = wrap(px, rows, cols);
        if (img.rows() < 3 || img.cols() < 3) throw std::invalid_argument("image < 3x3");
        code_map(img, k, path_of(path), out);
    });
}

int ref_ldp_histogram(const uint8_t* px, int rows, int cols, int k, int path, uint64_t* out) {
    return guarded([&] {
        const aldp::LdpHistogram h = aldp::ldp_histogram(wrap(px, rows, cols), k, path_of(path));
        std::memcpy(out, h.bins.data(), sizeof(uint64_t) * 56);
    });
}

// windowed_features(img, window, Ldp|Aldp) flattened to [cells][56].
int ref_windowed(const uint8_t* px, int rows, int cols, int window, int path, uint64_t* out,
                 int64_t* n_cells) {
    return guarded([&] {
        const auto feats = aldp::windowed_features(
            wrap(px, rows, cols), window, path == 0 ? aldp::Descriptor::Ldp : aldp::Descriptor::Aldp);
        for (size_t w = 0; w < feats.size(); ++w)
            std::memcpy(out + w * 56, feats[w].data(), sizeof(uint64_t) * 56);
        *n_cells = static_cast<int64_t>(feats.size());
    });
}

// Batch over n contiguous rows x cols images, sharded by image over `threads`
// std::threads. cell_rows == 0: one whole-image histogram per image.
int ref_batch(const uint8_t* px, int64_t n, int rows, int cols, int k, int cell_rows,
              int cell_cols, int path, uint8_t* codes, uint64_t* hist, int threads) {
    if (threads < 1) threads = 1;
    const size_t plane = static_cast<size_t>(rows) * cols;
    const int nb = n_bins(k);
    const int cells = cell_rows == 0 ? 1 : (rows / cell_rows) * (cols / cell_cols);
    std::vector<int> status(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
            status[t] = guarded([&] {
                for (int64_t i = lo; i < hi; ++i) {
                    const aldp::GrayImage img = wrap(px + i * plane, rows, cols);
                    if (codes) code_map(img, k, path_of(path), codes + i * plane);
                    if (hist) {
                        uint64_t* h = hist + static_cast<size_t>(i) * cells * nb;
                        if (cell_rows == 0) histogram(img, k, path_of(path), h);
                        else cell_histograms(img, cell_rows, cell_cols, k, path_of(path), h);
                    }
                }
            });
        });
    }
    for (auto& th : pool) th.join();
    for (int s : status)
        if (s) return s;
    return 0;
}

// aldp::response_field flattened to int32 [rows*cols][8].
int ref_response_field(const uint8_t* px, int rows, int cols, int path, int32_t* out) {
    return guarded([&] {
        const auto f = aldp::response_field(wrap(px, rows, cols), path_of(path));
        for (size_t i = 0; i < f.size(); ++i)
            for (int d = 0; d < 8; ++d) out[i * 8 + d] = f[i].m[d];
    });
}

namespace {
void flatten(const aldp::VerifyResult& v, uint64_t* counts2, int* mm7) {
    counts2[0] = v.images_checked;
    counts2[1] = v.pixels_checked;
    mm7[0] = v.mismatch.has_value();
    if (v.mismatch) {
        const aldp::Mismatch& m = *v.mismatch;
        mm7[1] = m.image_index, mm7[2] = m.x, mm7[3] = m.y, mm7[4] = m.direction;
        mm7[5] = m.naive_value, mm7[6] = m.accelerated_value;
    }
}
std::optional<aldp::FaultInjection> fault_of(const int* f5) {
    if (!f5) return std::nullopt;
    aldp::FaultInjection f;
    f.image_index = f5[0], f.x = f5[1], f.y = f5[2], f.term_index = f5[3], f.delta = f5[4];
    return f;
}
}  // namespace

// aldp::verify_equivalence; fault5 = {image_index, x, y, term_index, delta} or NULL.
int ref_verify_equivalence(int images, uint32_t seed, const int* fault5, int threads, uint64_t* counts2,
                           int* mm7) {
    return guarded([&] { flatten(aldp::verify_equivalence(images, seed, fault_of(fault5), threads), counts2, mm7); });
}

int ref_verify_image(const uint8_t* px, int rows, int cols, const int* fault5, int image_index,
                     uint64_t* counts2, int* mm7) {
    return guarded([&] {
        flatten(aldp::verify_image(wrap(px, rows, cols), fault_of(fault5), image_index), counts2, mm7);
    });
}

// aldp::load_pgm: 0 ok (rows/cols/pixels), 4 std::runtime_error (message in
// err), other codes as guarded(). out == NULL: dimensions only.
int ref_load_pgm(const char* path, uint8_t* out, size_t cap, int* rows, int* cols, char* err, int err_len) {
    try {
        const aldp::GrayImage img = aldp::load_pgm(path);
        *rows = img.rows(), *cols = img.cols();
        if (out) {
            if (cap < img.pixel_count()) return 1;
            std::memcpy(out, img.pixels().data(), img.pixel_count());
        }
        return 0;
    } catch (const std::runtime_error& e) {
        if (err && err_len > 0) {
            std::strncpy(err, e.what(), size_t(err_len) - 1);
            err[err_len - 1] = 0;
        }
        return 4;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

int ref_save_pgm(const char* path, const uint8_t* px, int rows, int cols, int ascii) {
    return guarded([&] {
        aldp::save_pgm(path, wrap(px, rows, cols), ascii ? aldp::PgmFormat::Ascii : aldp::PgmFormat::Binary);
    });
}

// descriptor: 0 LDP, 1 ALDP, 2 LBP
int ref_op_counts(int descriptor, int* mults, int* adds) {
    return guarded([&] {
        const auto d = descriptor == 2 ? aldp::Descriptor::Lbp
                                       : descriptor == 0 ? aldp::Descriptor::Ldp : aldp::Descriptor::Aldp;
        const aldp::OpCountRow r = aldp::measured_ops(d);
        *mults = r.multiplications;
        *adds = r.additions;
    });
}

// The reference CLI's `bench` body (tools/aldp_main.cpp:128-165) over the
// reference library: run_time_series / run_window_series + write_csv into
// `out` (NUL-terminated, truncated to cap).
int ref_bench_csv(const char* series, int size, const int* counts, int n_counts, const int* windows,
                  int n_windows, int repeats, uint32_t seed, int descriptor, char* out, size_t cap) {
    return guarded([&] {
        std::vector<aldp::Descriptor> ds = {aldp::Descriptor::Lbp, aldp::Descriptor::Ldp, aldp::Descriptor::Aldp};
        if (descriptor >= 0)
            ds = {descriptor == 2 ? aldp::Descriptor::Lbp
                                  : descriptor == 0 ? aldp::Descriptor::Ldp : aldp::Descriptor::Aldp};
        std::vector<aldp::BenchRecord> records;
        if (std::string(series) == "images") {
            const int side = size > 0 ? size : 260;
            std::vector<int> cs(counts, counts + n_counts);
            int corpus_size = 1;
            for (int c : cs) corpus_size = std::max(corpus_size, c);
            std::vector<aldp::GrayImage> corpus;
            for (int i = 0; i < corpus_size; ++i)
                corpus.push_back(aldp::make_random(side, side, seed + static_cast<uint32_t>(i)));
            for (auto d : ds) {
                const auto rows = aldp::run_time_series(corpus, d, repeats, cs);
                records.insert(records.end(), rows.begin(), rows.end());
            }
        } else {
            const int side = size > 0 ? size : 300;
            const aldp::GrayImage img = aldp::make_random(side, side, seed);
            std::vector<int> ws(windows, windows + n_windows);
            for (auto d : ds) {
                const auto rows = aldp::run_window_series(img, ws, d, repeats);
                records.insert(records.end(), rows.begin(), rows.end());
            }
        }
        std::ostringstream os;
        aldp::write_csv(os, records);
        const std::string s = os.str();
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    });
}

// The reference's own timer (src/bench.cpp:51-78): warm-up pass, batches to
// >= 5 ms, median of `repeats` samples.
double ref_median_seconds_batch(const uint8_t* px, int64_t n, int rows, int cols, int k,
                                int cell_rows, int cell_cols, int path, uint8_t* codes,
                                uint64_t* hist, int threads, int repeats) {
    return aldp::median_seconds(
        [&] { ref_batch(px, n, rows, cols, k, cell_rows, cell_cols, path, codes, hist, threads); },
        repeats);
}

}  // extern "C"
