// Drop-in probe: one C++ program written only against the reference's public
// API (proj/include/aldp/*.hpp). tests/golden/make_dropin.sh compiles it
// against the reference headers + sources and records its output
// (tests/golden/dropin_reference.txt); tests/test_dropin_gpu.py compiles the
// same file against this repo's include/aldp + libaldp_b200.so and requires
// byte-identical output. Large results are printed as FNV-1a hashes.
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "aldp/bench.hpp"
#include "aldp/descriptors.hpp"
#include "aldp/image.hpp"
#include "aldp/kirsch.hpp"
#include "aldp/pgm.hpp"
#include "aldp/verify.hpp"
#include "aldp/windowing.hpp"

namespace {

struct Fnv {
    std::uint64_t h = 1469598103934665603ull;
    void add(std::uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xFF;
            h *= 1099511628211ull;
        }
    }
};

template <typename F>
std::string throws(F&& f) {
    try {
        f();
        return "none";
    } catch (const std::invalid_argument&) {
        return "invalid_argument";
    } catch (const std::out_of_range&) {
        return "out_of_range";
    } catch (const std::runtime_error&) {
        return "runtime_error";
    } catch (const std::logic_error&) {
        return "logic_error";
    }
}

}  // namespace

int main(int argc, char** argv) {
    using namespace aldp;
    const std::string tmp = argc > 1 ? argv[1] : "/tmp";

    // histograms, both paths, several sizes (descriptors.cpp:123-139)
    const int sizes[][2] = {{3, 3}, {5, 9}, {16, 16}, {37, 53}, {64, 130}, {490, 640}};
    for (const auto& s : sizes) {
        const GrayImage img = make_random(s[0], s[1], 1000u + s[0] * 7u + s[1]);
        const LdpHistogram a = ldp_histogram(img, 3, ResponsePath::Naive);
        const LdpHistogram b = ldp_histogram(img, 3, ResponsePath::Accelerated);
        Fnv f;
        for (auto v : a.bins) f.add(v);
        std::cout << "ldp_histogram " << s[0] << "x" << s[1] << " total " << a.total() << " equal "
                  << (a == b) << " fnv " << f.h << "\n";
        const LbpHistogram l = lbp_histogram(img);
        Fnv g;
        for (auto v : l.bins) g.add(v);
        std::cout << "lbp_histogram " << s[0] << "x" << s[1] << " fnv " << g.h << "\n";
    }
    // windows (windowing.cpp:35-63)
    const GrayImage big = make_random(300, 300, 42);
    for (int w : {3, 25, 50, 100, 300})
        for (Descriptor d : {Descriptor::Lbp, Descriptor::Ldp, Descriptor::Aldp}) {
            const auto feats = windowed_features(big, w, d);
            Fnv f;
            for (const auto& h : feats)
                for (auto v : h) f.add(v);
            std::cout << "windowed " << w << " " << descriptor_name(d) << " n " << feats.size() << " grid "
                      << make_grid(big, w).total() << " fnv " << f.h << "\n";
        }
    // per-pixel API and the op model (kirsch.cpp:63-191, bench.cpp:97-131)
    const GrayImage small = make_gradient(7, 9);
    for (int x = 0; x < 7; x += 3)
        for (int y = 0; y < 9; y += 4) {
            OpCounter c1, c2;
            const ResponseVector n = responses_naive(small, x, y, BorderPolicy::Clamp, &c1);
            const ResponseVector a = responses_accelerated(column_terms(small, x, y, BorderPolicy::Clamp, &c2), &c2);
            std::cout << "responses " << x << "," << y << ":";
            for (int v : n.m) std::cout << " " << v;
            std::cout << " equal " << (n == a) << " ops " << c1.multiplications << "/" << c1.additions << " "
                      << c2.multiplications << "/" << c2.additions << " code3 " << int(ldp_code(n, 3))
                      << " bin " << ldp_bin_index(ldp_code(n, 3)) << " lbp " << int(lbp_code(small, x, y)) << "\n";
        }
    for (const auto& row : op_count_report())
        std::cout << "ops " << row.descriptor << " " << row.multiplications << " " << row.additions << "\n";
    std::cout << "bin_code 0 " << int(ldp_bin_code(0)) << " 55 " << int(ldp_bin_code(55)) << "\n";
    // the whole response field (kirsch.cpp:193-208)
    {
        const GrayImage img = make_random(41, 67, 5);
        for (ResponsePath p : {ResponsePath::Naive, ResponsePath::Accelerated}) {
            Fnv f;
            for (const auto& r : response_field(img, p))
                for (int v : r.m) f.add(std::uint64_t(std::int64_t(v)));
            std::cout << "response_field " << int(p) << " fnv " << f.h << "\n";
        }
    }
    // equivalence sweep (verify.cpp:37-111)
    {
        const VerifyResult ok = verify_equivalence(200, 7);
        std::cout << "verify ok " << ok.ok() << " " << ok.images_checked << " " << ok.pixels_checked << "\n";
        for (int t : {1, 4}) {
            const VerifyResult bad = verify_equivalence(120, 9, FaultInjection{33, 2, 1, 8, -4}, t);
            const Mismatch& m = *bad.mismatch;
            std::cout << "verify fault threads " << t << " " << bad.images_checked << " " << bad.pixels_checked
                      << " at " << m.image_index << " " << m.x << " " << m.y << " " << m.direction << " "
                      << m.naive_value << " " << m.accelerated_value << "\n";
        }
        const VerifyResult one = verify_image(make_random(20, 30, 3), FaultInjection{0, 5, 6, 11, 2});
        std::cout << "verify_image " << one.pixels_checked << " " << one.mismatch->direction << "\n";
    }
    // PGM round trip (pgm.cpp)
    {
        const std::filesystem::path p5 = std::filesystem::path(tmp) / "dropin_probe.pgm";
        const GrayImage img = make_random(13, 21, 77);
        save_pgm(p5, img);
        std::cout << "pgm p5 roundtrip " << (load_pgm(p5) == img) << "\n";
        save_pgm(p5, img, PgmFormat::Ascii);
        std::cout << "pgm p2 roundtrip " << (load_pgm(p5) == img) << "\n";
        std::filesystem::remove(p5);
        std::cout << "pgm missing " << throws([&] { load_pgm(std::filesystem::path(tmp) / "no_such.pgm"); }) << "\n";
    }
    // bench CSV formatting (bench.cpp:161-178) on fixed records
    {
        std::ostringstream os;
        write_csv(os, {BenchRecord{"ALDP", 4, 0, 1, 0.0123456, 25, 43}, BenchRecord{"LBP", 1, 25, 144, 2.5, 0, 8}});
        std::cout << os.str();
    }
    // error behaviour (descriptors.cpp:84-86,124-126; windowing.cpp:9-17)
    std::cout << "err k2 " << throws([&] { ldp_histogram(big, 2, ResponsePath::Naive); }) << "\n";
    std::cout << "err 2x3 " << throws([&] { ldp_histogram(GrayImage(2, 3), 3, ResponsePath::Naive); }) << "\n";
    std::cout << "err window2 " << throws([&] { windowed_features(big, 2, Descriptor::Aldp); }) << "\n";
    std::cout << "err window301 " << throws([&] { make_grid(big, 301); }) << "\n";
    std::cout << "err code k8 " << throws([&] { ldp_code(ResponseVector{}, 8); }) << "\n";
    std::cout << "err pixel " << throws([&] { responses_naive(small, 7, 0); }) << "\n";
    std::cout << "err descriptor " << throws([&] { parse_descriptor("hog"); }) << "\n";
    std::cout << "parse " << descriptor_name(parse_descriptor("aLdP")) << "\n";
    return 0;
}
