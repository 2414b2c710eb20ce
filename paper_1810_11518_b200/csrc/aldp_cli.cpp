// aldp_cli.cpp -- the reference's command-line front end (tools/aldp_main.cpp)
// over the B200 library: same subcommands, options, output text and exit
// codes (0 success, 1 verification failure, 2 usage/input error), with the
// heavy lifting in libaldp_b200.so:
//
//   extract  -> aldp_extract_files  (pipelined PGM decode + B200 histograms)
//   verify   -> aldp::verify_equivalence (device sweep) + op_count_report
//   bench    -> aldp_bench_csv      (the reference's CSV schema, B200 rows)
//   compare  -> aldp::verify_image + ldp_histogram on both response paths
//
// Options accept "--opt value" and "--opt=value"; list options are
// comma-separated (CLI11 ->delimiter(',') in the reference).
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "aldp/bench.hpp"
#include "aldp/descriptors.hpp"
#include "aldp/pgm.hpp"
#include "aldp/verify.hpp"
#include "aldp_cuda.h"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitFailure = 1;
constexpr int kExitUsage = 2;

const char* kUsage =
    "LBP/LDP/ALDP texture descriptor extraction and benchmarking (B200)\n"
    "Usage: aldp_b200 SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  extract INPUTS... [--descriptor lbp|ldp|aldp] [--window N] [--out PATH] [--threads N]\n"
    "  verify [--images N] [--seed S] [--parallel]\n"
    "  bench [--series images|window] [--size N] [--counts a,b,..] [--windows a,b,..]\n"
    "        [--repeats N] [--seed S] [--descriptor D] [--out PATH]\n"
    "  compare [INPUTS...] [--seed S]\n";

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Splits argv into positionals and --name[=value] options.
struct Args {
    std::vector<std::string> positional;
    std::vector<std::pair<std::string, std::optional<std::string>>> options;

    bool help() const {
        for (const auto& o : options)
            if (o.first == "--help") return true;
        return false;
    }

    Args(int argc, char** argv, int first, const std::vector<std::string>& flags) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) {
                positional.push_back(a);
                continue;
            }
            const size_t eq = a.find('=');
            if (eq != std::string::npos) {
                options.emplace_back(a.substr(0, eq), a.substr(eq + 1));
                continue;
            }
            bool is_flag = false;  // value-less options
            for (const auto& f : flags) is_flag |= f == a;
            if (is_flag || a == "--help") {
                options.emplace_back(a, std::nullopt);
            } else {
                if (i + 1 >= argc) throw UsageError(a + " requires an argument");
                options.emplace_back(a, std::string(argv[++i]));
            }
        }
    }
};

int to_int(const std::string& opt, const std::string& v) {
    try {
        size_t used = 0;
        const long long x = std::stoll(v, &used);
        if (used != v.size() || x < INT32_MIN || x > INT32_MAX) throw std::invalid_argument(v);
        return static_cast<int>(x);
    } catch (const std::logic_error&) {
        throw UsageError(opt + ": value " + v + " is not an integer");
    }
}

uint32_t to_u32(const std::string& opt, const std::string& v) {
    try {
        size_t used = 0;
        const long long x = std::stoll(v, &used);
        if (used != v.size() || x < 0 || x > 0xFFFFFFFFLL) throw std::invalid_argument(v);
        return static_cast<uint32_t>(x);
    } catch (const std::logic_error&) {
        throw UsageError(opt + ": value " + v + " is not an unsigned 32-bit integer");
    }
}

std::vector<int> to_list(const std::string& opt, const std::string& v) {
    std::vector<int> out;
    size_t start = 0;
    while (start <= v.size()) {
        const size_t comma = v.find(',', start);
        out.push_back(to_int(opt, v.substr(start, comma == std::string::npos ? std::string::npos : comma - start)));
        if (comma == std::string::npos) break;
        start = comma + 1;
    }
    return out;
}

void check_status(aldp_status s) {
    if (s == ALDP_OK) return;
    const std::string msg = aldp_last_error();
    if (s == ALDP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

int cmd_extract(const Args& a) {
    std::string descriptor = "aldp", out;
    int window = 0, threads = 0;
    for (const auto& [k, v] : a.options) {
        if (k == "--descriptor") descriptor = *v;
        else if (k == "--window") window = to_int(k, *v);
        else if (k == "--out") out = *v;
        else if (k == "--threads") threads = to_int(k, *v);
        else throw UsageError("The following argument was not expected: " + k);
    }
    if (a.positional.empty()) throw UsageError("inputs is required");
    if (window != 0 && window < 3) {
        std::cerr << "error: --window must be >= 3\n";
        return kExitUsage;
    }
    std::vector<const char*> paths;
    for (const auto& p : a.positional) paths.push_back(p.c_str());
    check_status(aldp_extract_files(paths.data(), int(paths.size()), descriptor.c_str(), window,
                                    out.empty() ? nullptr : out.c_str(), threads));
    return kExitOk;
}

int cmd_verify(const Args& a) {
    int images = 1000;
    uint32_t seed = 42;
    bool parallel = false, fault = false;
    for (const auto& [k, v] : a.options) {
        if (k == "--images") images = to_int(k, *v);
        else if (k == "--seed") seed = to_u32(k, *v);
        else if (k == "--parallel") parallel = true;
        else if (k == "--inject-fault") fault = true;  // test harness hook
        else throw UsageError("The following argument was not expected: " + k);
    }
    if (!a.positional.empty()) throw UsageError("The following argument was not expected: " + a.positional[0]);
    std::optional<aldp::FaultInjection> f;
    if (fault) f = aldp::FaultInjection{0, 1, 1, 0, 1};  // aldp_main.cpp:101-104
    const int threads = parallel ? int(std::max(1u, std::thread::hardware_concurrency())) : 1;
    const aldp::VerifyResult r = aldp::verify_equivalence(images, seed, f, threads);
    if (!r.ok()) {
        const aldp::Mismatch& m = *r.mismatch;
        std::cout << "MISMATCH image " << m.image_index << " pixel (" << m.x << "," << m.y << ") direction "
                  << m.direction << ": naive " << m.naive_value << " != accelerated " << m.accelerated_value
                  << '\n';
        return kExitFailure;
    }
    const auto ops = aldp::op_count_report();
    std::cout << "equivalence OK: " << r.images_checked << " images, " << r.pixels_checked
              << " pixels, 8 directions each\n";
    std::cout << "op counts per pixel:";
    for (const auto& row : ops)
        std::cout << ' ' << row.descriptor << " (" << row.multiplications << " mul, " << row.additions << " add)";
    std::cout << '\n';
    return kExitOk;
}

int cmd_bench(const Args& a) {
    std::string series = "images", descriptor, out;
    int size = 0, repeats = 5;
    uint32_t seed = 42;
    std::vector<int> counts = {1, 2, 4, 6, 8, 10}, windows = {25, 50, 100};
    for (const auto& [k, v] : a.options) {
        if (k == "--series") series = *v;
        else if (k == "--size") size = to_int(k, *v);
        else if (k == "--counts") counts = to_list(k, *v);
        else if (k == "--windows") windows = to_list(k, *v);
        else if (k == "--repeats") repeats = to_int(k, *v);
        else if (k == "--seed") seed = to_u32(k, *v);
        else if (k == "--descriptor") descriptor = *v;
        else if (k == "--out") out = *v;
        else throw UsageError("The following argument was not expected: " + k);
    }
    if (repeats < 3) {
        std::cerr << "error: --repeats must be at least 3\n";
        return kExitUsage;
    }
    check_status(aldp_bench_csv(series.c_str(), size, counts.data(), int(counts.size()), windows.data(),
                                int(windows.size()), repeats, seed, descriptor.c_str(),
                                out.empty() ? nullptr : out.c_str()));
    return kExitOk;
}

int cmd_compare(const Args& a) {
    uint32_t seed = 42;
    for (const auto& [k, v] : a.options) {
        if (k == "--seed") seed = to_u32(k, *v);
        else throw UsageError("The following argument was not expected: " + k);
    }
    bool all_ok = true;
    auto check_one = [&](const std::string& label, const aldp::GrayImage& img) {
        const aldp::VerifyResult r = aldp::verify_image(img);
        const bool hist_equal = aldp::ldp_histogram(img, 3, aldp::ResponsePath::Naive) ==
                                aldp::ldp_histogram(img, 3, aldp::ResponsePath::Accelerated);
        if (r.ok() && hist_equal) {
            std::cout << label << ": identical (" << r.pixels_checked << " pixels, 8 directions, 56 bins)\n";
            return;
        }
        all_ok = false;
        if (r.mismatch) {
            const aldp::Mismatch& m = *r.mismatch;
            std::cout << label << ": MISMATCH pixel (" << m.x << "," << m.y << ") direction " << m.direction
                      << ": naive " << m.naive_value << " != accelerated " << m.accelerated_value << '\n';
        } else {
            std::cout << label << ": MISMATCH in histogram bins\n";
        }
    };
    if (a.positional.empty()) check_one("seeded-256x256", aldp::make_random(256, 256, seed));
    else
        for (const auto& p : a.positional) check_one(p, aldp::load_pgm(p));
    return all_ok ? kExitOk : kExitFailure;
}

int help() {
    std::cout << kUsage;
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "A subcommand is required\n" << kUsage;
        return kExitUsage;
    }
    const std::string sub = argv[1];
    if (sub == "--help" || sub == "-h") {
        std::cout << kUsage;
        return kExitOk;
    }
    try {
        if (sub == "extract") {
            const Args a(argc, argv, 2, {});
            if (a.help()) return help();
            return cmd_extract(a);
        }
        if (sub == "verify") {
            const Args a(argc, argv, 2, {"--parallel", "--inject-fault"});
            if (a.help()) return help();
            return cmd_verify(a);
        }
        if (sub == "bench") {
            const Args a(argc, argv, 2, {});
            if (a.help()) return help();
            return cmd_bench(a);
        }
        if (sub == "compare") {
            const Args a(argc, argv, 2, {});
            if (a.help()) return help();
            return cmd_compare(a);
        }
        std::cerr << "The following argument was not expected: " << sub << '\n' << kUsage;
        return kExitUsage;
    } catch (const UsageError& e) {
        std::cerr << e.what() << '\n' << kUsage;
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    }
}
