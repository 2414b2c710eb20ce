// ldp_host.cu -- host-buffer C-ABI entry points (the reference's public
// functions as C calls) and the synthetic input generators.
//
// The host entry points copy pixels to the device, run aldp_ldp_batch on a
// per-thread stream with per-thread cached device buffers (no allocation on
// the steady-state path), and copy results back:
//   aldp_ldp_histogram      <- aldp::ldp_histogram      (descriptors.hpp:55)
//   aldp_windowed_features  <- aldp::windowed_features  (windowing.hpp:34-36)
//   aldp_ldp_code_map       <- new (descriptors.cpp:129-136 per-pixel code)
//   aldp_ldp_batch_host     <- batch of the above (end-to-end bench path)
#include <cuda_runtime.h>
#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#endif

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#include <thread>

#include "aldp_cuda.h"

namespace aldp_b200 {

aldp_status set_error(aldp_status s, const std::string& msg);  // ldp_kernels.cu

static aldp_status hfail(aldp_status s, const std::string& msg) { return set_error(s, msg); }

#define HOST_CUDA_TRY(expr)                                                                 \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return hfail(_e == cudaErrorMemoryAllocation ? ALDP_ENOMEM : ALDP_ECUDA,        \
                         std::string(#expr) + ": " + cudaGetErrorString(_e));               \
    } while (0)

// Per host thread: kSlots streams, each with grow-only device buffers for one
// chunk of images. A batch is cut into chunks that rotate over the slots, so
// chunk i+1's H2D, chunk i's kernel and chunk i-1's D2H run concurrently
// (separate copy engines per direction; stream order protects buffer reuse).
constexpr int kSlots = 3;
constexpr size_t kChunkBytes = size_t(48) << 20;  // pixel bytes per chunk (~150 640x490 frames)
// ALDP_CHUNK_BYTES overrides the chunk size (tests drive the banded and
// chunked paths with small inputs through it)
static size_t chunk_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("ALDP_CHUNK_BYTES");
        const long long x = e ? std::atoll(e) : 0;
        return x > 0 ? size_t(x) : kChunkBytes;
    }();
    return v;
}
constexpr size_t kSmallBytes = size_t(4) << 20;   // calls up to this many pixel bytes take the staged path

// Pinned host staging (grow-only).
struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

struct Slot {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;  // staged path: the slot's chunk has landed in h_codes / h_hist
    uint8_t* d_px = nullptr;
    size_t px_cap = 0;
    uint8_t* d_codes = nullptr;
    size_t codes_cap = 0;
    uint32_t* d_hist = nullptr;
    size_t hist_cap = 0;
    PinnedBuf h_px, h_codes, h_hist;  // staging for pageable caller buffers
    void release() {
        if (d_px) cudaFree(d_px);
        if (d_codes) cudaFree(d_codes);
        if (d_hist) cudaFree(d_hist);
        if (stream) cudaStreamDestroy(stream);
        if (done) cudaEventDestroy(done);
        h_px.release();
        h_codes.release();
        h_hist.release();
        *this = Slot{};
    }
};

struct HostCtx {
    int device = -1;
    Slot slot[kSlots];
    PinnedBuf h_px, h_codes, h_hist;  // small-call staging
    ~HostCtx() {
        // Process teardown: the CUDA context may already be gone; ignore errors.
        for (auto& s : slot) s.release();
        h_px.release();
        h_codes.release();
        h_hist.release();
    }
};
static thread_local HostCtx t_ctx;

static aldp_status ensure(void** p, size_t* cap, size_t need) {
    if (*cap >= need) return ALDP_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    HOST_CUDA_TRY(cudaMalloc(p, need));
    *cap = need;
    return ALDP_OK;
}

static aldp_status ensure_pinned(PinnedBuf& b, size_t need) {
    if (b.cap >= need) return ALDP_OK;
    b.release();
    HOST_CUDA_TRY(cudaHostAlloc(&b.p, need, cudaHostAllocDefault));
    b.cap = need;
    return ALDP_OK;
}

static aldp_status ctx_ready(HostCtx& c) {
    int dev = 0;
    HOST_CUDA_TRY(cudaGetDevice(&dev));
    if (c.device != dev) {  // a different device on this thread: drop the old buffers
        for (auto& s : c.slot) s.release();
        c.h_px.release();
        c.h_codes.release();
        c.h_hist.release();
        for (auto& s : c.slot) {
            HOST_CUDA_TRY(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
            HOST_CUDA_TRY(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
        }
        c.device = dev;
    }
    return ALDP_OK;
}

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

// Page-locked (or registered) host memory can be a DMA source/target as is.
static bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Large copy with non-temporal (streaming) stores: the staging and caller
// buffers it fills are read next by the DMA engine or much later by the
// caller, so write-allocating them in the host caches only costs memory
// bandwidth -- the resource the pageable path is bound by. SSE2 only (any
// x86-64 host). ALDP_NT_COPY=0 turns it off (A/B).
static bool nt_copy_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ALDP_NT_COPY");
        return !(e && e[0] == '0');
    }();
    return on;
}
static void copy_bytes(uint8_t* dst, const uint8_t* src, size_t n) {
#if defined(__x86_64__) || defined(_M_X64)
    if (n >= (size_t(1) << 16) && nt_copy_enabled()) {
        const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
        std::memcpy(dst, src, head);
        dst += head, src += head, n -= head;
        const size_t body = n & ~size_t(63);
        for (size_t i = 0; i < body; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
            const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
        }
        std::memcpy(dst + body, src + body, n - body);
        _mm_sfence();  // streaming stores drained before the buffer is handed on
        return;
    }
#endif
    std::memcpy(dst, src, n);
}

// Copies `nrows` rows of `width` bytes between strided buffers on up to
// kCopyThreads host threads (one thread moves ~8 GB/s; PCIe needs ~45).
constexpr int kCopyThreads = 16;
static int copy_threads() {
    static const int t = [] {
        const char* e = std::getenv("ALDP_COPY_THREADS");
        return e ? std::max(1, std::min(kCopyThreads, std::atoi(e))) : 8;
    }();
    return t;
}
static void copy_rows(uint8_t* dst, size_t dst_pitch, const uint8_t* src, size_t src_pitch, size_t width,
                      size_t nrows) {
    const size_t bytes = width * nrows;
    const int t = int(std::min<size_t>(copy_threads(), std::max<size_t>(1, bytes >> 22)));  // >= 4 MB per thread
    auto part = [&](size_t r0, size_t r1) {
        if (dst_pitch == width && src_pitch == width) {
            copy_bytes(dst + r0 * width, src + r0 * width, (r1 - r0) * width);
        } else {
            for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dst_pitch, src + r * src_pitch, width);
        }
    };
    if (t == 1) {
        part(0, nrows);
        return;
    }
    std::thread pool[kCopyThreads];
    for (int i = 0; i < t; ++i) pool[i] = std::thread(part, nrows * i / t, nrows * (i + 1) / t);
    for (int i = 0; i < t; ++i) pool[i].join();
}

// Tall single frame in bands (see host_batch). Band b covers rows
// [b*B, min(rows, (b+1)*B)); B is a multiple of cell_rows so every cell lies
// in one band and the band's cells are a contiguous run of the frame's grid.
// Pageable pixels and codes go through pinned staging (the copy in also
// assembles the halo rows and the device pitch); pinned ones are DMA'd.
static aldp_status host_band(HostCtx& c, const uint8_t* px, int rows, int cols, int k, int cell_rows,
                             int cell_cols, uint8_t* codes, uint32_t* hist32, bool lbp, int nbins, int64_t cells) {
    const int pitch = round_up(cols, 16);
    const int unit = cell_rows ? cell_rows : 16;
    const int B = std::max(unit, int(chunk_bytes() / size_t(pitch)) / unit * unit);
    const int n_bands = (rows + B - 1) / B;
    const int grid_c = cell_rows ? cols / cell_cols : 1;
    const size_t band_hist = cell_rows ? size_t(B / cell_rows) * grid_c * nbins : size_t(nbins);
    const bool stage_px = !is_pinned(px);
    const bool stage_codes = codes && !is_pinned(codes);
    std::vector<uint32_t> whole(hist32 && !cell_rows ? size_t(n_bands) * nbins : 0);
    aldp_status s = ALDP_OK;
    const int used = std::min(n_bands, kSlots);
    for (int i = 0; i < used; ++i) {
        Slot& sl = c.slot[i];
        s = ensure(reinterpret_cast<void**>(&sl.d_px), &sl.px_cap, size_t(B + 2) * pitch);
        if (s == ALDP_OK && codes) s = ensure(reinterpret_cast<void**>(&sl.d_codes), &sl.codes_cap, size_t(B) * pitch);
        if (s == ALDP_OK && hist32)
            s = ensure(reinterpret_cast<void**>(&sl.d_hist), &sl.hist_cap, sizeof(uint32_t) * band_hist);
        if (s == ALDP_OK && stage_px) s = ensure_pinned(sl.h_px, size_t(B + 2) * pitch);
        if (s == ALDP_OK && stage_codes) s = ensure_pinned(sl.h_codes, size_t(B) * pitch);
        if (s == ALDP_OK && hist32) s = ensure_pinned(sl.h_hist, sizeof(uint32_t) * band_hist);
        if (s != ALDP_OK) return s;
    }
    int pending[kSlots];
    for (int i = 0; i < kSlots; ++i) pending[i] = -1;
    auto band_rows = [&](int b, int& start, int& end) {
        start = b * B;
        end = std::min(rows, start + B);
    };
    auto drain = [&](int si) -> aldp_status {
        const int b = pending[si];
        if (b < 0) return ALDP_OK;
        Slot& sl = c.slot[si];
        HOST_CUDA_TRY(cudaEventSynchronize(sl.done));
        int start, end;
        band_rows(b, start, end);
        if (stage_codes)
            copy_rows(codes + size_t(start) * cols, cols, static_cast<const uint8_t*>(sl.h_codes.p), pitch, cols,
                      size_t(end - start));
        if (hist32 && (!cell_rows || end - start >= cell_rows)) {
            const uint32_t* h = static_cast<const uint32_t*>(sl.h_hist.p);
            if (cell_rows) {
                const size_t n_cell_rows = size_t(std::min(end, rows / cell_rows * cell_rows) - start) / cell_rows;
                std::memcpy(hist32 + size_t(start / cell_rows) * grid_c * nbins, h,
                            sizeof(uint32_t) * n_cell_rows * grid_c * nbins);
            } else {
                std::memcpy(whole.data() + size_t(b) * nbins, h, sizeof(uint32_t) * nbins);
            }
        }
        pending[si] = -1;
        return ALDP_OK;
    };
    for (int b = 0; b < n_bands; ++b) {
        const int si = b % kSlots;
        Slot& sl = c.slot[si];
        const cudaStream_t st = sl.stream;
        s = drain(si);
        if (s != ALDP_OK) return s;
        int start, end;
        band_rows(b, start, end);
        const int top = start > 0 ? 1 : 0, bot = end < rows ? 1 : 0;
        const int src_rows = end - start + top + bot;
        if (stage_px) {
            copy_rows(static_cast<uint8_t*>(sl.h_px.p), pitch, px + size_t(start - top) * cols, cols, cols,
                      size_t(src_rows));
            HOST_CUDA_TRY(cudaMemcpyAsync(sl.d_px, sl.h_px.p, size_t(src_rows) * pitch, cudaMemcpyHostToDevice, st));
        } else {
            HOST_CUDA_TRY(cudaMemcpy2DAsync(sl.d_px, pitch, px + size_t(start - top) * cols, cols, cols,
                                            size_t(src_rows), cudaMemcpyHostToDevice, st));
        }
        aldp_ldp_args a{};
        a.d_pixels = sl.d_px + size_t(top) * pitch;
        a.img_stride = int64_t(B + 2) * pitch;
        a.rows = end - start;
        a.cols = cols;
        a.pitch = pitch;
        a.n_images = 1;
        a.k = k;
        // a band shorter than a cell (the frame's remainder rows) has no cells
        const bool band_cells = cell_rows && a.rows >= cell_rows;
        a.cell_rows = band_cells ? cell_rows : 0;
        a.cell_cols = band_cells ? cell_cols : 0;
        a.d_codes = codes ? sl.d_codes : nullptr;
        a.codes_img_stride = int64_t(B) * pitch;
        a.codes_pitch = pitch;
        a.d_hist = hist32 && (band_cells || !cell_rows) ? sl.d_hist : nullptr;
        a.rows_above = top;
        a.rows_below = bot;
        if (a.d_codes || a.d_hist) {
            s = lbp ? aldp_lbp_batch(&a, st) : aldp_ldp_batch(&a, st);
            if (s != ALDP_OK) return hfail(s, aldp_last_error());
        }
        if (codes) {
            if (stage_codes)
                HOST_CUDA_TRY(cudaMemcpyAsync(sl.h_codes.p, sl.d_codes, size_t(a.rows) * pitch, cudaMemcpyDeviceToHost, st));
            else
                HOST_CUDA_TRY(cudaMemcpy2DAsync(codes + size_t(start) * cols, cols, sl.d_codes, pitch, cols,
                                                size_t(a.rows), cudaMemcpyDeviceToHost, st));
        }
        if (a.d_hist)
            HOST_CUDA_TRY(cudaMemcpyAsync(sl.h_hist.p, sl.d_hist,
                                          sizeof(uint32_t) * (band_cells ? size_t(a.rows / cell_rows) * grid_c * nbins
                                                                         : size_t(nbins)),
                                          cudaMemcpyDeviceToHost, st));
        HOST_CUDA_TRY(cudaEventRecord(sl.done, st));
        pending[si] = b;  // drained (and its staging freed) before the slot's next band
    }
    for (int i = 0; i < used; ++i) {
        s = drain(i);
        if (s != ALDP_OK) return s;
    }
    for (int i = 0; i < used; ++i) HOST_CUDA_TRY(cudaStreamSynchronize(c.slot[i].stream));
    if (hist32 && !cell_rows) {
        for (int bin = 0; bin < nbins; ++bin) {
            uint32_t t = 0;
            for (int b = 0; b < n_bands; ++b) t += whole[size_t(b) * nbins + bin];
            hist32[bin] = t;
        }
    }
    (void)cells;
    return ALDP_OK;
}

// Shared body: host pixels (n contiguous rows x cols images) -> optional host
// codes (contiguous) and u32 histograms `hist32` [n][cells][bins]. Pinned
// host memory gives full PCIe rate in both directions at once.
static aldp_status host_batch(const uint8_t* px, int n, int rows, int cols, int k, int cell_rows,
                              int cell_cols, uint8_t* codes, uint32_t* hist32, cudaStream_t user,
                              bool lbp = false) {
    if (!px && n > 0) return hfail(ALDP_EINVAL, "null pixels");
    if (n < 0) return hfail(ALDP_EINVAL, "negative image count");
    if (rows < 3 || cols < 3)
        return hfail(ALDP_EINVAL, "descriptor extraction needs at least a 3x3 image, got " +
                                      std::to_string(rows) + "x" + std::to_string(cols));
    const int nbins = lbp ? 256 : aldp_n_bins(k);
    if (nbins == 0) return hfail(ALDP_EINVAL, "k must be in [1, 7]");
    const int64_t cells = aldp_grid_cells(rows, cols, cell_rows, cell_cols);
    if (cells < 0) return hfail(ALDP_EINVAL, "invalid window/cell size for this image");
    HostCtx& c = t_ctx;
    aldp_status s = ctx_ready(c);
    if (s != ALDP_OK) return s;
    if (n == 0) return ALDP_OK;
    // pad the device pitch to 16 B so the packed kernel always applies
    const int pitch = round_up(cols, 16);
    const size_t img_bytes = size_t(pitch) * rows;
    const size_t plane = size_t(rows) * cols;
    const size_t hist_per_img = size_t(cells) * nbins;
    const int chunk = int(std::max<size_t>(1, std::min<size_t>(size_t(n), chunk_bytes() / img_bytes)));
    const int n_chunks = (n + chunk - 1) / chunk;
    const int used = std::min(n_chunks, kSlots);
    // Small calls (the reference's one-image-per-call pattern): stage through
    // pinned host buffers on one stream. The CPU does the pitch padding, so
    // every transfer is a single 1D DMA instead of a pageable (2D) copy.
    if (!user && img_bytes * size_t(n) <= kSmallBytes) {
        Slot& sl = c.slot[0];
        s = ensure(reinterpret_cast<void**>(&sl.d_px), &sl.px_cap, img_bytes * n);
        if (s == ALDP_OK && codes) s = ensure(reinterpret_cast<void**>(&sl.d_codes), &sl.codes_cap, img_bytes * n);
        if (s == ALDP_OK && hist32)
            s = ensure(reinterpret_cast<void**>(&sl.d_hist), &sl.hist_cap, sizeof(uint32_t) * hist_per_img * n);
        if (s == ALDP_OK) s = ensure_pinned(c.h_px, img_bytes * n);
        if (s == ALDP_OK && codes) s = ensure_pinned(c.h_codes, img_bytes * n);
        if (s == ALDP_OK && hist32) s = ensure_pinned(c.h_hist, sizeof(uint32_t) * hist_per_img * n);
        if (s != ALDP_OK) return s;
        uint8_t* hp = static_cast<uint8_t*>(c.h_px.p);
        if (pitch == cols) {
            std::memcpy(hp, px, plane * n);
        } else {
            for (size_t r = 0; r < size_t(rows) * n; ++r) std::memcpy(hp + r * pitch, px + r * cols, cols);
        }
        const cudaStream_t st = sl.stream;
        HOST_CUDA_TRY(cudaMemcpyAsync(sl.d_px, hp, img_bytes * n, cudaMemcpyHostToDevice, st));
        aldp_ldp_args a{};
        a.d_pixels = sl.d_px;
        a.img_stride = int64_t(img_bytes);
        a.rows = rows;
        a.cols = cols;
        a.pitch = pitch;
        a.n_images = n;
        a.k = k;
        a.cell_rows = cell_rows;
        a.cell_cols = cell_cols;
        a.d_codes = codes ? sl.d_codes : nullptr;
        a.codes_img_stride = int64_t(img_bytes);
        a.codes_pitch = pitch;
        a.d_hist = hist32 ? sl.d_hist : nullptr;
        s = lbp ? aldp_lbp_batch(&a, st) : aldp_ldp_batch(&a, st);
        if (s != ALDP_OK) return hfail(s, aldp_last_error());
        if (codes)
            HOST_CUDA_TRY(cudaMemcpyAsync(c.h_codes.p, sl.d_codes, img_bytes * n, cudaMemcpyDeviceToHost, st));
        if (hist32)
            HOST_CUDA_TRY(cudaMemcpyAsync(c.h_hist.p, sl.d_hist, sizeof(uint32_t) * hist_per_img * n,
                                          cudaMemcpyDeviceToHost, st));
        HOST_CUDA_TRY(cudaStreamSynchronize(st));
        if (codes) {
            const uint8_t* hc = static_cast<const uint8_t*>(c.h_codes.p);
            if (pitch == cols) {
                std::memcpy(codes, hc, plane * n);
            } else {
                for (size_t r = 0; r < size_t(rows) * n; ++r) std::memcpy(codes + r * cols, hc + r * pitch, cols);
            }
        }
        if (hist32) std::memcpy(hist32, c.h_hist.p, sizeof(uint32_t) * hist_per_img * n);
        return ALDP_OK;
    }
    // One frame taller than a chunk: stream it as bands of whole cells (or
    // of 16-row multiples), each with its real neighbour rows as halos, so
    // H2D, kernel and D2H overlap inside the frame too.
    if (n == 1 && !user && img_bytes > chunk_bytes()) return host_band(c, px, rows, cols, k, cell_rows, cell_cols,
                                                                       codes, hist32, lbp, nbins, cells);
    // order the internal streams after work already queued on the caller's stream
    cudaEvent_t start = nullptr;
    if (user) {
        HOST_CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
        HOST_CUDA_TRY(cudaEventRecord(start, user));
    }
    for (int i = 0; i < used; ++i) {
        Slot& sl = c.slot[i];
        s = ensure(reinterpret_cast<void**>(&sl.d_px), &sl.px_cap, img_bytes * chunk);
        if (s == ALDP_OK && codes) s = ensure(reinterpret_cast<void**>(&sl.d_codes), &sl.codes_cap, img_bytes * chunk);
        if (s == ALDP_OK && hist32)
            s = ensure(reinterpret_cast<void**>(&sl.d_hist), &sl.hist_cap, sizeof(uint32_t) * hist_per_img * chunk);
        if (s != ALDP_OK) return s;
        if (start) HOST_CUDA_TRY(cudaStreamWaitEvent(sl.stream, start, 0));
    }
    if (start) cudaEventDestroy(start);
    // Pageable caller buffers go through per-slot pinned staging: the CPU
    // copies chunk i+1 in and chunk i-1 out (pooled threads) while the GPU
    // works on chunk i. Pinned ones are DMA'd directly.
    const bool stage_px = !is_pinned(px);
    const bool stage_codes = codes && !is_pinned(codes);
    const bool stage_hist = hist32 && !is_pinned(hist32);
    const bool staged = stage_px || stage_codes || stage_hist;
    if (staged) {
        for (int i = 0; i < used; ++i) {
            Slot& sl = c.slot[i];
            if (stage_px) s = ensure_pinned(sl.h_px, img_bytes * chunk);
            if (s == ALDP_OK && stage_codes) s = ensure_pinned(sl.h_codes, img_bytes * chunk);
            if (s == ALDP_OK && stage_hist) s = ensure_pinned(sl.h_hist, sizeof(uint32_t) * hist_per_img * chunk);
            if (s != ALDP_OK) return s;
        }
    }
    int pending[kSlots];  // chunk whose results wait in the slot's staging, or -1
    for (int i = 0; i < kSlots; ++i) pending[i] = -1;
    auto drain = [&](int slot_i) -> aldp_status {  // staged results of the slot's chunk -> caller
        const int ch = pending[slot_i];
        if (ch < 0) return ALDP_OK;
        Slot& sl = c.slot[slot_i];
        HOST_CUDA_TRY(cudaEventSynchronize(sl.done));
        const int i0 = ch * chunk, cnt = std::min(chunk, n - i0);
        if (stage_codes)
            copy_rows(codes + size_t(i0) * plane, cols, static_cast<const uint8_t*>(sl.h_codes.p), pitch, cols,
                      size_t(rows) * cnt);
        if (stage_hist)
            copy_rows(reinterpret_cast<uint8_t*>(hist32 + size_t(i0) * hist_per_img), 0,
                      static_cast<const uint8_t*>(sl.h_hist.p), 0, sizeof(uint32_t) * hist_per_img * cnt, 1);
        pending[slot_i] = -1;
        return ALDP_OK;
    };
    for (int ch = 0; ch < n_chunks; ++ch) {
        const int si = ch % kSlots;
        Slot& sl = c.slot[si];
        const cudaStream_t st = sl.stream;
        const int i0 = ch * chunk, cnt = std::min(chunk, n - i0);
        const uint8_t* src = px + size_t(i0) * plane;
        if (staged) {
            // the slot's previous chunk out (its staging is about to be reused)
            // and this chunk in, at the same time on separate copy pools; the
            // previous H2D from h_px finished before that chunk's event fired
            HOST_CUDA_TRY(cudaEventSynchronize(sl.done));
            std::thread in;
            if (stage_px)
                in = std::thread(copy_rows, static_cast<uint8_t*>(sl.h_px.p), size_t(pitch), src, size_t(cols),
                                 size_t(cols), size_t(rows) * cnt);
            s = drain(si);
            if (in.joinable()) in.join();
            if (s != ALDP_OK) return s;
        }
        if (stage_px) {
            HOST_CUDA_TRY(cudaMemcpyAsync(sl.d_px, sl.h_px.p, img_bytes * cnt, cudaMemcpyHostToDevice, st));
        } else if (pitch == cols) {
            HOST_CUDA_TRY(cudaMemcpyAsync(sl.d_px, src, img_bytes * cnt, cudaMemcpyHostToDevice, st));
        } else {
            HOST_CUDA_TRY(cudaMemcpy2DAsync(sl.d_px, pitch, src, cols, cols, size_t(rows) * cnt,
                                            cudaMemcpyHostToDevice, st));
        }
        aldp_ldp_args a{};
        a.d_pixels = sl.d_px;
        a.img_stride = int64_t(img_bytes);
        a.rows = rows;
        a.cols = cols;
        a.pitch = pitch;
        a.n_images = cnt;
        a.k = k;
        a.cell_rows = cell_rows;
        a.cell_cols = cell_cols;
        a.d_codes = codes ? sl.d_codes : nullptr;
        a.codes_img_stride = int64_t(img_bytes);
        a.codes_pitch = pitch;
        a.d_hist = hist32 ? sl.d_hist : nullptr;
        s = lbp ? aldp_lbp_batch(&a, st) : aldp_ldp_batch(&a, st);
        if (s != ALDP_OK) return hfail(s, aldp_last_error());
        if (codes) {
            uint8_t* dst = codes + size_t(i0) * plane;
            if (stage_codes)
                HOST_CUDA_TRY(cudaMemcpyAsync(sl.h_codes.p, sl.d_codes, img_bytes * cnt, cudaMemcpyDeviceToHost, st));
            else if (pitch == cols)
                HOST_CUDA_TRY(cudaMemcpyAsync(dst, sl.d_codes, img_bytes * cnt, cudaMemcpyDeviceToHost, st));
            else
                HOST_CUDA_TRY(cudaMemcpy2DAsync(dst, cols, sl.d_codes, pitch, cols, size_t(rows) * cnt,
                                                cudaMemcpyDeviceToHost, st));
        }
        if (hist32) {
            void* hdst = stage_hist ? sl.h_hist.p : static_cast<void*>(hist32 + size_t(i0) * hist_per_img);
            HOST_CUDA_TRY(cudaMemcpyAsync(hdst, sl.d_hist, sizeof(uint32_t) * hist_per_img * cnt,
                                          cudaMemcpyDeviceToHost, st));
        }
        if (staged) {
            HOST_CUDA_TRY(cudaEventRecord(sl.done, st));
            pending[si] = ch;
        }
    }
    for (int i = 0; i < used; ++i) {
        s = drain(i);
        if (s != ALDP_OK) return s;
    }
    for (int i = 0; i < used; ++i) HOST_CUDA_TRY(cudaStreamSynchronize(c.slot[i].stream));
    return ALDP_OK;
}

static aldp_status widen(const uint32_t* h32, uint64_t* h64, size_t n) {
    for (size_t i = 0; i < n; ++i) h64[i] = h32[i];
    return ALDP_OK;
}

// ---------------------------------------------------------------------------
// generators
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
    return mix64(mix64(mix64(seed) ^ a) ^ b);
}
__device__ __forceinline__ float u01(uint64_t h) {  // [0, 1)
    return float(h >> 40) * (1.0f / 16777216.0f);
}

constexpr int kMaxBlobs = 256;
constexpr int kMaxRects = 512;

// grid: (row chunks, images); each CTA rebuilds its image's parameters.
__global__ void gen_faces_kernel(uint8_t* out, int rows, int cols, int pitch, int64_t stride,
                                 int blobs, uint64_t seed, int64_t first) {
    __shared__ float bx[kMaxBlobs], by[kMaxBlobs], binv[kMaxBlobs], bamp[kMaxBlobs];
    __shared__ float g[4];
    const int64_t gidx = first + blockIdx.y;
    const uint64_t is = hash3(seed, 0xFACEull, uint64_t(gidx));
    for (int b = threadIdx.x; b < blobs; b += blockDim.x) {
        bx[b] = u01(hash3(is, b, 1)) * rows;
        by[b] = u01(hash3(is, b, 2)) * cols;
        const float sigma = 5.0f + 55.0f * u01(hash3(is, b, 3));
        binv[b] = -0.5f / (sigma * sigma);
        bamp[b] = -80.0f + 160.0f * u01(hash3(is, b, 4));
    }
    if (threadIdx.x == 0) {
        const float th = 6.2831853f * u01(hash3(is, 0x9A, 1));
        const float lo = 40.0f + 80.0f * u01(hash3(is, 0x9A, 2));
        const float hi = 120.0f + 100.0f * u01(hash3(is, 0x9A, 3));
        // intensity = lo + (hi - lo) * t, t = projection on (cos, sin) in [0, 1]
        const float cx = cosf(th), cy = sinf(th);
        const float span = fabsf(cx) * (rows - 1) + fabsf(cy) * (cols - 1) + 1e-6f;
        g[0] = cx * (hi - lo) / span;
        g[1] = cy * (hi - lo) / span;
        g[2] = lo - fminf(0.0f, cx * (rows - 1)) * (hi - lo) / span -
               fminf(0.0f, cy * (cols - 1)) * (hi - lo) / span;
        g[3] = 0.0f;
    }
    __syncthreads();
    uint8_t* img = out + blockIdx.y * stride;
    const int rows_per = (rows + gridDim.x - 1) / gridDim.x;
    const int x0 = blockIdx.x * rows_per, x1 = min(rows, x0 + rows_per);
    for (int64_t t = threadIdx.x; t < int64_t(x1 - x0) * cols; t += blockDim.x) {
        const int x = x0 + int(t / cols), y = int(t % cols);
        float v = g[2] + g[0] * x + g[1] * y;
        for (int b = 0; b < blobs; ++b) {
            const float dx = x - bx[b], dy = y - by[b];
            v += bamp[b] * __expf((dx * dx + dy * dy) * binv[b]);
        }
        const uint64_t h = hash3(is, 0x7E57ull, uint64_t(x) * uint64_t(cols) + uint64_t(y));
        const float u1 = fmaxf(u01(h), 1e-7f), u2 = float(uint32_t(h) >> 8) * (1.0f / 16777216.0f);
        v += 6.0f * sqrtf(-2.0f * __logf(u1)) * __cosf(6.2831853f * u2);
        img[int64_t(x) * pitch + y] = uint8_t(fminf(fmaxf(rintf(v), 0.0f), 255.0f));
    }
}

__global__ void gen_ties_kernel(uint8_t* out, int rows, int cols, int pitch, int64_t stride,
                                uint64_t seed, int64_t first) {
    __shared__ int rx0[kMaxRects], ry0[kMaxRects], rx1[kMaxRects], ry1[kMaxRects];
    __shared__ uint8_t rv[kMaxRects];
    __shared__ int n_rects;
    const int64_t gidx = first + blockIdx.y;
    const uint64_t is = hash3(seed, 0x71E5ull, uint64_t(gidx));
    if (threadIdx.x == 0) {
        // paint until the summed rectangle area reaches ln 2 of the image, so
        // the expected union of uniformly placed rectangles is ~50%
        const double target = 0.6931 * double(rows) * cols;
        double area = 0;
        int n = 0;
        const int side_max = max(4, min(rows, cols) / 4);
        while (area < target && n < kMaxRects) {
            const int h = 2 + int(u01(hash3(is, n, 1)) * side_max);
            const int w = 2 + int(u01(hash3(is, n, 2)) * side_max);
            const int x = int(u01(hash3(is, n, 3)) * rows), y = int(u01(hash3(is, n, 4)) * cols);
            rx0[n] = x;
            ry0[n] = y;
            rx1[n] = min(rows, x + h);
            ry1[n] = min(cols, y + w);
            rv[n] = uint8_t(hash3(is, n, 5) % 3);
            area += double(rx1[n] - x) * (ry1[n] - y);
            ++n;
        }
        n_rects = n;
    }
    __syncthreads();
    uint8_t* img = out + blockIdx.y * stride;
    const int rows_per = (rows + gridDim.x - 1) / gridDim.x;
    const int x0 = blockIdx.x * rows_per, x1 = min(rows, x0 + rows_per);
    for (int64_t t = threadIdx.x; t < int64_t(x1 - x0) * cols; t += blockDim.x) {
        const int x = x0 + int(t / cols), y = int(t % cols);
        uint8_t v = uint8_t(hash3(is, 0xB1ull, uint64_t(x) * uint64_t(cols) + uint64_t(y)) % 3);
        for (int r = n_rects - 1; r >= 0; --r)  // painter's order: last rectangle wins
            if (x >= rx0[r] && x < rx1[r] && y >= ry0[r] && y < ry1[r]) {
                v = rv[r];
                break;
            }
        img[int64_t(x) * pitch + y] = v;
    }
}

}  // namespace aldp_b200

using namespace aldp_b200;

extern "C" {

aldp_status aldp_ldp_histogram(const uint8_t* pixels, int rows, int cols, int k, int path,
                               uint64_t* bins56) {
    (void)path;  // Naive and Accelerated are identical by contract (descriptors.hpp:53-54)
    if (k != 3) return hfail(ALDP_EINVAL, "the 56-bin histogram layout requires k == 3");
    uint32_t h32[56];
    aldp_status s = host_batch(pixels, 1, rows, cols, 3, 0, 0, nullptr, h32, nullptr);
    if (s != ALDP_OK) return s;
    return widen(h32, bins56, 56);
}

aldp_status aldp_windowed_features(const uint8_t* pixels, int rows, int cols, int window,
                                   int path, uint64_t* out, size_t out_len) {
    // path: ALDP_PATH_NAIVE / ALDP_PATH_ACCELERATED (Ldp / Aldp, 56 bins) or
    // ALDP_DESC_LBP (256 bins) -- windowing.cpp:43-58
    if (path != ALDP_PATH_NAIVE && path != ALDP_PATH_ACCELERATED && path != ALDP_DESC_LBP)
        return hfail(ALDP_EINVAL, "unknown descriptor");
    if (window < 3) return hfail(ALDP_EINVAL, "window side must be >= 3, got " + std::to_string(window));
    if (window > rows || window > cols)
        return hfail(ALDP_EINVAL, "window side " + std::to_string(window) + " exceeds image " +
                                      std::to_string(rows) + "x" + std::to_string(cols));
    const bool lbp = path == ALDP_DESC_LBP;
    const size_t nb = lbp ? 256 : 56;
    const int64_t cells = aldp_grid_cells(rows, cols, window, window);
    if (out_len < size_t(cells) * nb) return hfail(ALDP_ERANGE, "output buffer too small");
    uint32_t* h32 = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * size_t(cells) * nb));
    if (!h32) return hfail(ALDP_ENOMEM, "host allocation failed");
    aldp_status s = host_batch(pixels, 1, rows, cols, 3, window, window, nullptr, h32, nullptr, lbp);
    if (s == ALDP_OK) widen(h32, out, size_t(cells) * nb);
    std::free(h32);
    return s;
}

aldp_status aldp_lbp_histogram(const uint8_t* pixels, int rows, int cols, uint64_t* bins256) {
    uint32_t h32[256];
    aldp_status s = host_batch(pixels, 1, rows, cols, 3, 0, 0, nullptr, h32, nullptr, true);
    if (s != ALDP_OK) return s;
    return widen(h32, bins256, 256);
}

aldp_status aldp_lbp_code_map(const uint8_t* pixels, int rows, int cols, uint8_t* codes) {
    if (!codes) return hfail(ALDP_EINVAL, "null codes buffer");
    return host_batch(pixels, 1, rows, cols, 3, 0, 0, codes, nullptr, nullptr, true);
}

aldp_status aldp_lbp_batch_host(const uint8_t* pixels, int n_images, int rows, int cols, int cell_rows,
                                int cell_cols, uint8_t* codes, uint32_t* hist, void* stream) {
    return host_batch(pixels, n_images, rows, cols, 3, cell_rows, cell_cols, codes, hist,
                      static_cast<cudaStream_t>(stream), true);
}

aldp_status aldp_ldp_code_map(const uint8_t* pixels, int rows, int cols, int k, int path,
                              uint8_t* codes) {
    (void)path;
    if (!codes) return hfail(ALDP_EINVAL, "null codes buffer");
    return host_batch(pixels, 1, rows, cols, k, 0, 0, codes, nullptr, nullptr);
}

aldp_status aldp_ldp_batch_host(const uint8_t* pixels, int n_images, int rows, int cols, int k,
                                int cell_rows, int cell_cols, uint8_t* codes, uint32_t* hist,
                                void* stream) {
    return host_batch(pixels, n_images, rows, cols, k, cell_rows, cell_cols, codes, hist,
                      static_cast<cudaStream_t>(stream));
}

aldp_status aldp_gen_faces(uint8_t* d_out, int n_images, int rows, int cols, int pitch,
                           int64_t img_stride, int blobs, uint64_t seed, int64_t first_index,
                           void* stream) {
    if (n_images < 0 || rows < 1 || cols < 1 || pitch < cols || blobs < 0 || blobs > kMaxBlobs)
        return hfail(ALDP_EINVAL, "gen_faces: bad arguments");
    if (n_images == 0) return ALDP_OK;
    const int chunks = std::max(1, std::min(rows, (rows * cols + 65535) / 65536));
    // grid.y is limited to 65535: launch in slabs of images
    for (int done = 0; done < n_images; done += 65535) {
        const int cnt = std::min(65535, n_images - done);
        gen_faces_kernel<<<dim3(chunks, cnt), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            d_out + int64_t(done) * img_stride, rows, cols, pitch, img_stride, blobs, seed,
            first_index + done);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return hfail(ALDP_ECUDA, std::string("gen_faces: ") + cudaGetErrorString(e));
    return ALDP_OK;
}

aldp_status aldp_gen_ties(uint8_t* d_out, int n_images, int rows, int cols, int pitch,
                          int64_t img_stride, uint64_t seed, int64_t first_index, void* stream) {
    if (n_images < 0 || rows < 1 || cols < 1 || pitch < cols)
        return hfail(ALDP_EINVAL, "gen_ties: bad arguments");
    if (n_images == 0) return ALDP_OK;
    const int chunks = std::max(1, std::min(rows, (rows * cols + 65535) / 65536));
    for (int done = 0; done < n_images; done += 65535) {
        const int cnt = std::min(65535, n_images - done);
        gen_ties_kernel<<<dim3(chunks, cnt), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            d_out + int64_t(done) * img_stride, rows, cols, pitch, img_stride, seed,
            first_index + done);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return hfail(ALDP_ECUDA, std::string("gen_ties: ") + cudaGetErrorString(e));
    return ALDP_OK;
}

}  // extern "C"
