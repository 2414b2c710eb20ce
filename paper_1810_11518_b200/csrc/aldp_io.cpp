// aldp_io.cpp -- SURVEY 8f ranks 3 and 4: on-disk input and the reference's
// report formats, around the B200 path.
//
//   load_pgm / save_pgm      drop-in for reference pgm.hpp (pgm.cpp:59-149),
//                            restated from its documented behaviour: same
//                            header tokenizer (comments do not end a token),
//                            same checks and messages ("<path>: <what>")
//   aldp_extract_files       the CLI `extract` command (aldp_main.cpp:59-96)
//                            as one native pipeline: a thread pool parses the
//                            next group of PGM files while the B200 extracts
//                            the current group (runs of equal-size images go
//                            through the chunked 3-stream host batch from
//                            pinned staging), and rows are written in input
//                            order in the reference's CSV layout
//   bench.hpp drop-in        median_seconds / measured_ops / op_count_report /
//                            run_time_series / run_window_series / write_csv
//                            (bench.cpp:51-178): the reference's timing rules
//                            and CSV schema; the timed calls are this
//                            library's GPU-backed extraction functions
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <future>
#include <limits>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "aldp/bench.hpp"
#include "aldp/descriptors.hpp"
#include "aldp/image.hpp"
#include "aldp/kirsch.hpp"
#include "aldp/pgm.hpp"
#include "aldp/windowing.hpp"
#include "aldp_cuda.h"

namespace aldp_b200 {
aldp_status set_error(aldp_status s, const std::string& msg);  // ldp_kernels.cu
}

namespace aldp {

namespace {

// File-level failures: std::runtime_error, as the reference throws.
struct PgmError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] void pgm_fail(const std::string& path, const std::string& what) {
    throw PgmError(path + ": " + what);
}

// Byte cursor with the reference tokenizer's rules (pgm.cpp:17-37): skip
// whitespace before a token; '#' skips to end of line without ending the
// token being built; whitespace after a token is left unread.
struct Cursor {
    const unsigned char* p;
    const unsigned char* end;
    int get() { return p < end ? *p++ : EOF; }
    void unget() { --p; }
    std::string token() {
        std::string tok;
        int c;
        while ((c = get()) != EOF) {
            if (c == '#') {
                while ((c = get()) != EOF && c != '\n') {
                }
                continue;
            }
            if (std::isspace(c)) {
                if (!tok.empty()) {
                    unget();
                    break;
                }
                continue;
            }
            tok.push_back(static_cast<char>(c));
        }
        return tok;
    }
};

// std::stoi(tok, &used) semantics on a whitespace-free token: optional sign,
// decimal digits, int range; `ok` false when stoi would throw or stop early.
int parse_int(const std::string& tok, bool& ok) {
    ok = false;
    size_t i = 0;
    bool neg = false;
    if (i < tok.size() && (tok[i] == '+' || tok[i] == '-')) neg = tok[i++] == '-';
    if (i >= tok.size()) return 0;
    long long v = 0;
    for (; i < tok.size(); ++i) {
        if (tok[i] < '0' || tok[i] > '9') return 0;
        v = v * 10 + (tok[i] - '0');
        if (v > static_cast<long long>(std::numeric_limits<int>::max()) + 1) return 0;
    }
    if (neg) v = -v;
    if (v > std::numeric_limits<int>::max() || v < std::numeric_limits<int>::min()) return 0;
    ok = true;
    return static_cast<int>(v);
}

int header_int(Cursor& in, const std::string& path, const char* field) {
    const std::string tok = in.token();
    if (tok.empty()) pgm_fail(path, std::string("missing ") + field + " in header");
    bool ok = false;
    const int v = parse_int(tok, ok);
    if (!ok || v < 0) pgm_fail(path, std::string("malformed ") + field + " '" + tok + "'");
    return v;
}

std::vector<unsigned char> read_file(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) pgm_fail(path, "cannot open file");
    std::vector<unsigned char> buf;
    long size = -1;
    if (std::fseek(f, 0, SEEK_END) == 0) size = std::ftell(f);
    if (size >= 0 && std::fseek(f, 0, SEEK_SET) == 0) {  // regular file: one sized read
        buf.resize(size_t(size));
        const size_t got = size ? std::fread(buf.data(), 1, buf.size(), f) : 0;
        buf.resize(got);
    } else {  // pipes and the like: read to EOF
        std::clearerr(f);
        unsigned char chunk[1 << 16];
        size_t n;
        while ((n = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + n);
    }
    const bool err = std::ferror(f);
    std::fclose(f);
    if (err) pgm_fail(path, "cannot open file");
    return buf;
}

struct PgmHeader {
    int rows = 0, cols = 0, maxval = 0;
    bool binary = false;
};

PgmHeader parse_header(Cursor& in, const std::string& path) {
    const std::string magic = in.token();
    if (magic != "P2" && magic != "P5") pgm_fail(path, "not a PGM file (magic '" + magic + "')");
    PgmHeader h;
    h.binary = magic == "P5";
    h.cols = header_int(in, path, "width");  // width first (pgm.cpp:69-70)
    h.rows = header_int(in, path, "height");
    h.maxval = header_int(in, path, "maxval");
    if (h.cols < 1 || h.rows < 1)
        pgm_fail(path, "invalid dimensions " + std::to_string(h.cols) + "x" + std::to_string(h.rows));
    if (h.maxval < 1) pgm_fail(path, "invalid maxval " + std::to_string(h.maxval));
    if (h.maxval > 255)
        pgm_fail(path, "unsupported bit depth (maxval " + std::to_string(h.maxval) + " > 255)");
    return h;
}

void parse_payload(Cursor& in, const PgmHeader& h, const std::string& path, uint8_t* px) {
    const size_t count = size_t(h.rows) * size_t(h.cols);
    if (h.binary) {
        const int sep = in.get();  // exactly one whitespace byte (pgm.cpp:91-95)
        if (sep == EOF || !std::isspace(sep)) pgm_fail(path, "malformed header/payload separator");
        if (size_t(in.end - in.p) < count) pgm_fail(path, "truncated pixel payload");
        std::memcpy(px, in.p, count);
        if (h.maxval < 255) {
            for (size_t i = 0; i < count; ++i)
                if (px[i] > h.maxval)
                    pgm_fail(path, "pixel value " + std::to_string(px[i]) + " exceeds maxval");
        }
        return;
    }
    for (size_t i = 0; i < count; ++i) {
        const std::string tok = in.token();
        if (tok.empty()) pgm_fail(path, "truncated pixel payload");
        bool ok = false;
        const int v = parse_int(tok, ok);
        if (!ok || v < 0 || v > h.maxval) pgm_fail(path, "malformed pixel value '" + tok + "'");
        px[i] = static_cast<uint8_t>(v);
    }
}

// One decoded file: dimensions + pixels (or the error it raised). P5 keeps
// the file buffer and points at its payload (no copy); P2 holds the parsed
// pixels at offset 0.
struct Loaded {
    int rows = 0, cols = 0;
    std::vector<uint8_t> buf;
    size_t offset = 0;
    std::string error;
    const uint8_t* pixels() const { return buf.data() + offset; }
};

Loaded load_one(const std::string& path) {
    Loaded out;
    try {
        std::vector<unsigned char> file = read_file(path);
        Cursor in{file.data(), file.data() + file.size()};
        const PgmHeader h = parse_header(in, path);
        const size_t count = size_t(h.rows) * h.cols;
        if (h.binary) {
            const int sep = in.get();  // exactly one whitespace byte (pgm.cpp:91-95)
            if (sep == EOF || !std::isspace(sep)) pgm_fail(path, "malformed header/payload separator");
            if (size_t(in.end - in.p) < count) pgm_fail(path, "truncated pixel payload");
            if (h.maxval < 255)
                for (size_t i = 0; i < count; ++i)
                    if (in.p[i] > h.maxval)
                        pgm_fail(path, "pixel value " + std::to_string(in.p[i]) + " exceeds maxval");
            out.offset = size_t(in.p - file.data());
            out.buf = std::move(file);
        } else {
            out.buf.resize(count);
            parse_payload(in, h, path, out.buf.data());
        }
        out.rows = h.rows, out.cols = h.cols;
    } catch (const std::exception& e) {
        out.error = e.what();
    }
    return out;
}

// Runs fn(i) for i in [0, n) on up to `threads` host threads.
template <typename F>
void parallel_for(size_t n, int threads, F fn) {
    const int t = int(std::max<size_t>(1, std::min<size_t>(size_t(std::max(threads, 1)), n)));
    if (t == 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < t; ++w)
        pool.emplace_back([&, w] {
            for (size_t i = size_t(w); i < n; i += size_t(t)) fn(i);
        });
    for (auto& th : pool) th.join();
}

std::vector<Loaded> load_parallel(const std::vector<std::string>& paths, size_t lo, size_t hi, int threads) {
    std::vector<Loaded> out(hi - lo);
    parallel_for(hi - lo, threads, [&](size_t i) { out[i] = load_one(paths[lo + i]); });
    return out;
}

void throw_status(aldp_status s) {
    if (s == ALDP_OK) return;
    const std::string msg = aldp_last_error();
    switch (s) {
    case ALDP_EINVAL: throw std::invalid_argument(msg);
    case ALDP_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
    }
}

// Pinned staging for one run of equal-size images (grow-only, per thread).
struct Pinned {
    uint8_t* p = nullptr;
    size_t cap = 0;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
    uint8_t* get(size_t n) {
        if (n > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            if (cudaHostAlloc(reinterpret_cast<void**>(&p), n, cudaHostAllocDefault) != cudaSuccess)
                throw std::runtime_error("pinned host allocation of " + std::to_string(n) + " bytes failed");
            cap = n;
        }
        return p;
    }
};

void append_u64(std::string& s, uint64_t v) {
    char b[24];
    const auto r = std::to_chars(b, b + sizeof b, v);
    s.append(b, r.ptr);
}

}  // namespace

GrayImage load_pgm(const std::filesystem::path& path) {
    const std::string p = path.string();
    const std::vector<unsigned char> buf = read_file(p);
    Cursor in{buf.data(), buf.data() + buf.size()};
    const PgmHeader h = parse_header(in, p);
    std::vector<std::uint8_t> px(size_t(h.rows) * h.cols);
    parse_payload(in, h, p, px.data());
    return {h.rows, h.cols, std::move(px)};
}

void save_pgm(const std::filesystem::path& path, const GrayImage& img, PgmFormat format) {
    std::ofstream out(path, std::ios::binary);
    if (!out) pgm_fail(path.string(), "cannot open file for writing");
    out << (format == PgmFormat::Binary ? "P5\n" : "P2\n") << img.cols() << ' ' << img.rows() << "\n255\n";
    if (format == PgmFormat::Binary) {
        out.write(reinterpret_cast<const char*>(img.pixels().data()), std::streamsize(img.pixel_count()));
    } else {
        for (int x = 0; x < img.rows(); ++x)
            for (int y = 0; y < img.cols(); ++y)
                out << int(img.at(x, y)) << (y + 1 == img.cols() ? '\n' : ' ');
    }
    if (!out) pgm_fail(path.string(), "write failed");
}

// ------------------------------------------------------------------ bench

namespace {
constexpr double kMinSampleSeconds = 5e-3;  // bench.cpp:21
volatile std::uint64_t g_sink = 0;
void sink(std::uint64_t v) { g_sink = g_sink + v; }

void extract_whole(const GrayImage& img, Descriptor d) {
    switch (d) {
    case Descriptor::Lbp: sink(lbp_histogram(img).bins[255]); break;
    case Descriptor::Ldp: sink(ldp_histogram(img, 3, ResponsePath::Naive).bins[0]); break;
    case Descriptor::Aldp: sink(ldp_histogram(img, 3, ResponsePath::Accelerated).bins[0]); break;
    }
}
}  // namespace

double median_seconds(const std::function<void()>& work, int repeats) {
    if (repeats < 3) throw std::invalid_argument("repeats must be >= 3");
    using Clock = std::chrono::steady_clock;
    auto once = [&] {
        const auto t0 = Clock::now();
        work();
        return std::chrono::duration<double>(Clock::now() - t0).count();
    };
    const double first = once();  // warm-up doubles as batch calibration
    int batch = 1;
    if (first < kMinSampleSeconds)
        batch = std::min(static_cast<int>(std::ceil(kMinSampleSeconds / std::max(first, 1e-9))), 1000000);
    std::vector<double> samples;
    for (int r = 0; r < repeats; ++r) {
        const auto t0 = Clock::now();
        for (int b = 0; b < batch; ++b) work();
        samples.push_back(std::chrono::duration<double>(Clock::now() - t0).count() / batch);
    }
    std::sort(samples.begin(), samples.end());
    const size_t mid = samples.size() / 2;
    return samples.size() % 2 ? samples[mid] : 0.5 * (samples[mid - 1] + samples[mid]);
}

OpCountRow measured_ops(Descriptor d) {
    const GrayImage probe = make_random(8, 8, 12345);  // any pixel: counts are constant
    OpCounter c;
    switch (d) {
    case Descriptor::Lbp: lbp_code(probe, 4, 4, BorderPolicy::Clamp, &c); break;
    case Descriptor::Ldp: responses_naive(probe, 4, 4, BorderPolicy::Clamp, &c); break;
    case Descriptor::Aldp: responses_accelerated(column_terms(probe, 4, 4, BorderPolicy::Clamp, &c), &c); break;
    }
    return {descriptor_name(d), static_cast<int>(c.multiplications), static_cast<int>(c.additions)};
}

std::array<OpCountRow, 3> op_count_report() {
    const std::array<OpCountRow, 3> rows = {measured_ops(Descriptor::Aldp), measured_ops(Descriptor::Ldp),
                                            measured_ops(Descriptor::Lbp)};
    if (rows[1].multiplications != 72 || rows[1].additions != 64)
        throw std::logic_error("naive directional kernel no longer reads (72, 64)");
    if (rows[2].multiplications != 0 || rows[2].additions != 8)
        throw std::logic_error("binary-pattern kernel no longer reads (0, 8)");
    if (rows[0].multiplications > 30 || rows[0].additions > 46)
        throw std::logic_error("accelerated kernel exceeds its (30, 46) budget");
    return rows;
}

std::vector<BenchRecord> run_time_series(const std::vector<GrayImage>& corpus, Descriptor d, int repeats,
                                         const std::vector<int>& counts) {
    if (corpus.empty()) throw std::invalid_argument("corpus must not be empty");
    const OpCountRow ops = measured_ops(d);
    std::vector<BenchRecord> out;
    for (int count : counts) {
        if (count < 1 || count > static_cast<int>(corpus.size())) continue;
        const double t = median_seconds(
            [&] {
                for (int i = 0; i < count; ++i) extract_whole(corpus[size_t(i)], d);
            },
            repeats);
        out.push_back({descriptor_name(d), count, 0, 1, t, ops.multiplications, ops.additions});
    }
    return out;
}

std::vector<BenchRecord> run_window_series(const GrayImage& img, const std::vector<int>& windows, Descriptor d,
                                           int repeats) {
    const OpCountRow ops = measured_ops(d);
    std::vector<BenchRecord> out;
    for (int w : windows) {
        const WindowGrid grid = make_grid(img, w);
        const double t = median_seconds([&] { sink(windowed_features(img, w, d).size()); }, repeats);
        out.push_back({descriptor_name(d), 1, w, grid.total(), t, ops.multiplications, ops.additions});
    }
    return out;
}

const char* const kBenchCsvHeader = "descriptor,images,window,grid_total,elapsed_s,mults_per_pixel,adds_per_pixel";

void write_csv(std::ostream& out, const std::vector<BenchRecord>& records) {
    out << kBenchCsvHeader << '\n';
    for (const BenchRecord& r : records) {
        char sec[32];
        std::snprintf(sec, sizeof sec, "%.6f", r.elapsed_s);
        out << r.descriptor << ',' << r.images << ',';
        if (r.window == 0) out << "none";
        else out << r.window;
        out << ',' << r.grid_total << ',' << sec << ',' << r.mults_per_pixel << ',' << r.adds_per_pixel << '\n';
    }
}

// ------------------------------------------------------------------ extract

namespace {

// Group = consecutive input files decoded together; the next group decodes
// on the pool while the B200 extracts this one.
constexpr size_t kGroupFiles = 256;

struct Sink {
    std::FILE* f = nullptr;
    bool own = false;
    explicit Sink(const char* path) {
        if (path && *path) {
            f = std::fopen(path, "wb");
            if (!f) throw std::runtime_error(std::string("cannot open output file ") + path);
            own = true;
        } else {
            f = stdout;
        }
    }
    ~Sink() {
        if (own) std::fclose(f);
        else std::fflush(f);
    }
    void write(const std::string& s) {
        if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size())
            throw std::runtime_error("write to output failed");
    }
};

void extract_files(const std::vector<std::string>& paths, Descriptor d, int window, const char* out_path,
                   int threads) {
    Sink out(out_path);
    const int nb = d == Descriptor::Lbp ? 256 : 56;
    {
        std::string head = "identifier,descriptor";  // aldp_main.cpp:59-66
        for (int i = 0; i < nb; ++i) head += ",bin_" + std::to_string(i);
        head += '\n';
        out.write(head);
    }
    const std::string name = descriptor_name(d);
    Pinned staging;
    std::vector<uint32_t> hist;
    std::future<std::vector<Loaded>> next;
    auto start = [&](size_t lo) {
        const size_t hi = std::min(paths.size(), lo + kGroupFiles);
        return std::async(std::launch::async, [&paths, lo, hi, threads] {
            return load_parallel(paths, lo, hi, threads);
        });
    };
    if (!paths.empty()) next = start(0);
    for (size_t lo = 0; lo < paths.size(); lo += kGroupFiles) {
        std::vector<Loaded> group = next.get();
        if (lo + kGroupFiles < paths.size()) next = start(lo + kGroupFiles);
        size_t i = 0;
        while (i < group.size()) {
            if (!group[i].error.empty()) throw PgmError(group[i].error);
            // run of equal-size, successfully decoded images
            size_t j = i + 1;
            while (j < group.size() && group[j].error.empty() && group[j].rows == group[i].rows &&
                   group[j].cols == group[i].cols)
                ++j;
            const int rows = group[i].rows, cols = group[i].cols, n = int(j - i);
            if (rows < 3 || cols < 3)
                throw std::invalid_argument("descriptor extraction needs at least a 3x3 image, got " +
                                            std::to_string(rows) + "x" + std::to_string(cols));
            int64_t cells = 1;
            if (window > 0) {
                if (window > rows || window > cols)
                    throw std::invalid_argument("window side " + std::to_string(window) + " exceeds image " +
                                                std::to_string(rows) + "x" + std::to_string(cols));
                cells = int64_t(rows / window) * (cols / window);
            }
            const size_t plane = size_t(rows) * cols;
            uint8_t* px = staging.get(plane * n);
            parallel_for(size_t(n), threads, [&](size_t k) {
                std::memcpy(px + k * plane, group[i + k].pixels(), plane);
            });
            hist.resize(size_t(n) * cells * nb);
            const int cell = window > 0 ? window : 0;
            throw_status(d == Descriptor::Lbp
                             ? aldp_lbp_batch_host(px, n, rows, cols, cell, cell, nullptr, hist.data(), nullptr)
                             : aldp_ldp_batch_host(px, n, rows, cols, 3, cell, cell, nullptr, hist.data(), nullptr));
            // rows formatted per image on the pool, written in input order
            std::vector<std::string> text(static_cast<size_t>(n));
            parallel_for(size_t(n), threads, [&](size_t k) {
                std::string& t = text[k];
                const std::string& id = paths[lo + i + k];
                t.reserve(size_t(cells) * (nb * 4 + id.size() + 16));
                for (int64_t c = 0; c < cells; ++c) {
                    t += id;
                    if (window > 0) {
                        t += "#w";
                        append_u64(t, uint64_t(c));
                    }
                    t += ',';
                    t += name;
                    const uint32_t* h = hist.data() + (k * cells + c) * nb;
                    for (int b = 0; b < nb; ++b) {
                        t += ',';
                        append_u64(t, h[b]);
                    }
                    t += '\n';
                }
            });
            for (const std::string& t : text) out.write(t);
            i = j;
        }
    }
}

template <typename F>
aldp_status guarded(F&& f) {
    try {
        f();
        return ALDP_OK;
    } catch (const PgmError& e) {
        return aldp_b200::set_error(ALDP_EIO, e.what());
    } catch (const std::invalid_argument& e) {
        return aldp_b200::set_error(ALDP_EINVAL, e.what());
    } catch (const std::out_of_range& e) {
        return aldp_b200::set_error(ALDP_ERANGE, e.what());
    } catch (const std::logic_error& e) {
        return aldp_b200::set_error(ALDP_EINVAL, e.what());
    } catch (const std::bad_alloc&) {
        return aldp_b200::set_error(ALDP_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return aldp_b200::set_error(ALDP_EIO, e.what());
    }
}

Descriptor desc_of(int d) {
    if (d == ALDP_DESC_LBP) return Descriptor::Lbp;
    if (d == ALDP_PATH_NAIVE) return Descriptor::Ldp;
    if (d == ALDP_PATH_ACCELERATED) return Descriptor::Aldp;
    throw std::invalid_argument("descriptor must be ALDP_PATH_NAIVE, ALDP_PATH_ACCELERATED or ALDP_DESC_LBP");
}

}  // namespace

}  // namespace aldp

using namespace aldp;

extern "C" {

aldp_status aldp_load_pgm(const char* path, uint8_t* out, size_t cap, int* rows, int* cols) {
    return guarded([&] {
        if (!path || !rows || !cols) throw std::invalid_argument("null argument");
        const std::vector<unsigned char> buf = read_file(path);
        Cursor in{buf.data(), buf.data() + buf.size()};
        const PgmHeader h = parse_header(in, path);
        *rows = h.rows, *cols = h.cols;
        if (!out) return;  // size query
        if (cap < size_t(h.rows) * h.cols)
            throw std::invalid_argument("output buffer holds " + std::to_string(cap) + " bytes, image needs " +
                                        std::to_string(size_t(h.rows) * h.cols));
        parse_payload(in, h, path, out);
    });
}

aldp_status aldp_save_pgm(const char* path, const uint8_t* pixels, int rows, int cols, int ascii) {
    return guarded([&] {
        if (!path || !pixels) throw std::invalid_argument("null argument");
        const GrayImage img(rows, cols, std::vector<std::uint8_t>(pixels, pixels + size_t(rows) * cols));
        save_pgm(path, img, ascii ? PgmFormat::Ascii : PgmFormat::Binary);
    });
}

aldp_status aldp_load_pgm_batch(const char* const* paths, int n, int rows, int cols, uint8_t* out, int threads) {
    return guarded([&] {
        if (n < 0 || (n > 0 && (!paths || !out))) throw std::invalid_argument("bad batch arguments");
        std::vector<std::string> p(paths, paths + n);
        const std::vector<Loaded> got = load_parallel(p, 0, p.size(), threads < 1 ? 1 : threads);
        const size_t plane = size_t(rows) * cols;
        for (int i = 0; i < n; ++i) {
            if (!got[size_t(i)].error.empty()) throw PgmError(got[size_t(i)].error);
            if (got[size_t(i)].rows != rows || got[size_t(i)].cols != cols)
                throw std::invalid_argument(p[size_t(i)] + ": expected " + std::to_string(cols) + "x" +
                                            std::to_string(rows) + " (width x height), got " +
                                            std::to_string(got[size_t(i)].cols) + "x" +
                                            std::to_string(got[size_t(i)].rows));
            std::memcpy(out + size_t(i) * plane, got[size_t(i)].pixels(), plane);
        }
    });
}

aldp_status aldp_extract_files(const char* const* paths, int n, const char* descriptor, int window,
                               const char* out_path, int threads) {
    return guarded([&] {
        if (n < 0 || (n > 0 && !paths) || !descriptor) throw std::invalid_argument("bad extract arguments");
        if (window != 0 && window < 3) throw std::invalid_argument("--window must be >= 3");
        const Descriptor d = parse_descriptor(descriptor);
        if (threads < 1) threads = int(std::max(1u, std::thread::hardware_concurrency()));
        extract_files(std::vector<std::string>(paths, paths + n), d, window, out_path, threads);
    });
}

aldp_status aldp_op_counts(int descriptor, int* mults, int* adds) {
    return guarded([&] {
        const OpCountRow r = measured_ops(desc_of(descriptor));
        *mults = r.multiplications;
        *adds = r.additions;
    });
}

aldp_status aldp_bench_csv(const char* series, int size, const int* counts, int n_counts, const int* windows,
                           int n_windows, int repeats, uint32_t seed, const char* descriptor,
                           const char* out_path) {
    return guarded([&] {
        if (repeats < 3) throw std::invalid_argument("--repeats must be at least 3");
        std::vector<Descriptor> ds = {Descriptor::Lbp, Descriptor::Ldp, Descriptor::Aldp};
        if (descriptor && *descriptor) ds = {parse_descriptor(descriptor)};
        std::vector<BenchRecord> records;
        const std::string s = series ? series : "images";
        if (s == "images") {  // aldp_main.cpp:138-152
            const int side = size > 0 ? size : 260;
            std::vector<int> cs(counts, counts + n_counts);
            if (cs.empty()) cs = {1, 2, 4, 6, 8, 10};
            int corpus_size = 1;
            for (int c : cs) corpus_size = std::max(corpus_size, c);
            std::vector<GrayImage> corpus;
            for (int i = 0; i < corpus_size; ++i)
                corpus.push_back(make_random(side, side, seed + static_cast<std::uint32_t>(i)));
            for (Descriptor d : ds) {
                const auto rows = run_time_series(corpus, d, repeats, cs);
                records.insert(records.end(), rows.begin(), rows.end());
            }
        } else if (s == "window") {  // aldp_main.cpp:153-159
            const int side = size > 0 ? size : 300;
            std::vector<int> ws(windows, windows + n_windows);
            if (ws.empty()) ws = {25, 50, 100};
            const GrayImage img = make_random(side, side, seed);
            for (Descriptor d : ds) {
                const auto rows = run_window_series(img, ws, d, repeats);
                records.insert(records.end(), rows.begin(), rows.end());
            }
        } else {
            throw std::invalid_argument("--series: must be 'images' or 'window'");
        }
        std::ostringstream os;
        write_csv(os, records);
        Sink out(out_path);
        out.write(os.str());
    });
}

}  // extern "C"
