/*
 * aldp_cuda.h -- C-ABI of the B200 LDP path (libaldp_b200.so).
 *
 * Plain C: pointers, sizes and status codes; no C++ or torch types cross this
 * boundary. The C++ drop-in (include/aldp/*.hpp, namespace aldp) and the
 * Python host layer (paper_1810_11518_b200/__init__.py, ctypes) both sit on
 * top of it. See INTEGRATION.md for the binding a reference maintainer adds.
 *
 * Semantics follow the reference exactly (paths relative to the reference
 * tree):
 *  - responses: the eight Kirsch compass responses, clamp-to-edge border
 *    (proj/src/image.cpp:36-40, proj/src/kirsch.cpp:63-157);
 *  - code: top-k directions by (response desc, index asc), exactly k bits,
 *    signed responses (proj/src/descriptors.cpp:83-102);
 *  - bins: rank among the popcount-k codes in ascending code order
 *    (proj/src/descriptors.cpp:25-45,104-113; the reference defines k == 3
 *    only, 56 bins -- other k are this library's extension, C(8,k) bins);
 *  - histograms: every pixel of the image (proj/src/descriptors.cpp:123-139),
 *    or per cell with each cell clamped as an independent image, floor grid,
 *    row-major cells (proj/src/windowing.cpp:8-19,35-63; rectangular cells
 *    are this library's extension of the square `window`).
 *
 * Thread safety: every entry point may be called concurrently from several
 * host threads; device work is ordered on the caller's stream.
 */
#ifndef ALDP_CUDA_H
#define ALDP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ALDP_OK = 0,
    ALDP_EINVAL = 1, /* maps to std::invalid_argument in the C++ layer */
    ALDP_ERANGE = 2, /* maps to std::out_of_range */
    ALDP_ECUDA = 3,  /* CUDA runtime failure -> std::runtime_error */
    ALDP_ENOMEM = 4, /* device/host allocation failure -> std::runtime_error */
    ALDP_EIO = 5     /* file I/O or PGM format error -> std::runtime_error (pgm.hpp:15-17) */
} aldp_status;

/* Response path selector, mirroring aldp::ResponsePath (kirsch.hpp:88) and
 * the Ldp/Aldp descriptors (descriptors.hpp:13). Both values produce
 * identical outputs by contract (descriptors.hpp:53-54); both run the same
 * B200 kernel. */
enum { ALDP_PATH_NAIVE = 0, ALDP_PATH_ACCELERATED = 1 };
/* Descriptor selector for aldp_windowed_features: LBP (Descriptor::Lbp). */
enum { ALDP_DESC_LBP = 2 };

/* One batched launch over device-resident images.
 *
 *  d_pixels    n_images images of rows x cols uint8, row pitch `pitch`
 *              bytes, image stride `img_stride` bytes.
 *  k           1..7 (the reference's ldp_code range, descriptors.hpp:26).
 *  cell_rows,  0,0: one whole-image histogram per image (ldp_histogram).
 *  cell_cols   otherwise a floor grid of cell_rows x cell_cols cells, each
 *              clamped as an independent image (windowed_features); both
 *              must be in [3, rows] x [3, cols].
 *  d_codes     nullable. Code map, whole-image clamp (the per-pixel code of
 *              descriptors.cpp:129-136), row pitch codes_pitch, image stride
 *              codes_img_stride.
 *  d_hist      nullable. uint32 [n_images][grid_cells][aldp_n_bins(k)]
 *              (uint16 with hist_u16); every bin is overwritten, stream-ordered
 *              (a memset, or on narrow cells whole-cell stores plus a zeroing
 *              launch for the cells that straddle a 128-column tile). Narrow
 *              cells store 16 bytes at a time: d_hist 16-byte aligned (8 for
 *              uint16) keeps that path, otherwise the memset + atomics path.
 *
 * Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 * No hidden allocation; caller owns every buffer. */
typedef struct {
    const uint8_t* d_pixels;
    int64_t img_stride;
    int rows, cols, pitch;
    int n_images;
    int k;
    int cell_rows, cell_cols;
    uint8_t* d_codes;
    int64_t codes_img_stride;
    int codes_pitch;
    uint32_t* d_hist;
    /* 0 (default): every cell is clamped as an independent image, the
     * reference's windowed_features semantics (windowing.cpp:42). 1: cells are
     * cut from the whole-image code map (each pixel counted with its code-map
     * code), the paper's "code image, then regional histograms" reading.
     * Appended last so zero-initialised callers keep the reference rule. */
    int cell_from_map;
    /* Rows of a larger resident image that exist above row 0 / below the last
     * row of this view (0 or 1; default 0 = clamp at the view's edges). With 1
     * the view's edge rows see the real neighbour row instead of a clamped
     * copy, so a tall frame can be processed as bands with identical codes
     * and histograms (cells must then start at a multiple of cell_rows). */
    int rows_above, rows_below;
    /* 1: d_hist holds uint16 counts, [n_images][grid_cells][bins] (4-byte
     * aligned; every bin count is even), for a compact multi-GPU gather. Valid
     * only while no histogram can reach 65536 (cell area, or rows * cols for
     * whole-image histograms, below 65536) -> ALDP_EINVAL otherwise. */
    int hist_u16;
} aldp_ldp_args;

aldp_status aldp_ldp_batch(const aldp_ldp_args* args, void* stream);

/* Kernel selection for aldp_ldp_batch: AUTO picks the packed sm_100a kernel
 * whenever the layout allows it (pitches, strides and base pointers 8-byte
 * aligned -- any width and any k -- and at most 5 cells per 128 columns, or
 * up to 16 for LDP k != 4 with cells of >= 9 columns) and the generic
 * per-pixel kernel otherwise. FAST fails with
 * ALDP_EINVAL when the layout does not allow it. Both are CUDA; there is no
 * CPU path. */
enum { ALDP_KERNEL_AUTO = 0, ALDP_KERNEL_FAST = 1, ALDP_KERNEL_GENERIC = 2 };
aldp_status aldp_ldp_batch_ex(const aldp_ldp_args* args, int kernel, void* stream);

/* LBP descriptor (descriptors.cpp:141-168): code bit i set when ring
 * neighbour i (clockwise from the top-left) >= the centre pixel; 256 bins
 * indexed by the code. Same argument block as aldp_ldp_batch (k ignored),
 * d_hist is uint32 [n_images][grid_cells][256]. Same border and cell rules. */
aldp_status aldp_lbp_batch(const aldp_ldp_args* args, void* stream);
aldp_status aldp_lbp_batch_ex(const aldp_ldp_args* args, int kernel, void* stream);

/* Kernel launches the last aldp_ldp_batch* / aldp_lbp_batch* call on this
 * host thread made: 0 .. 3 (the LDP/LBP kernel; a second, codes-only launch
 * for the rows of a cell grid's overhang; on narrow cells a launch that zeroes
 * the cells straddling a 128-column tile edge). */
int aldp_last_launch_count(void);

/* Negative control for parity harnesses (the analogue of the reference's
 * FaultInjection, include/aldp/verify.hpp:14-20): while mode is 1, every
 * aldp_ldp_batch* / aldp_lbp_batch* call ends with a one-thread launch that
 * flips bit 0 of image 0's code at (0, 0) and adds one count to bin 0 of
 * image 0's first histogram (the product kernels are untouched). 0 turns it
 * off. The environment variable ALDP_FAULT_INJECT sets the initial mode.
 * Returns the old mode. */
int aldp_debug_fault(int mode);

/* Number of histogram bins for k: C(8, k) (56 for k == 3), 0 if k invalid. */
int aldp_n_bins(int k);

/* Number of cells of the floor grid (windowing.cpp:8-19 generalised):
 * (rows / cell_rows) * (cols / cell_cols); 1 for cell_rows == 0. Returns -1
 * for invalid geometry (cell < 3 or larger than the image). */
int64_t aldp_grid_cells(int rows, int cols, int cell_rows, int cell_cols);

/* ---- host-buffer entry points: the reference's public functions ----
 * These copy host pixels to the device, run aldp_ldp_batch on an internal
 * per-thread stream, and copy results back. They replace, one for one:   */

/* aldp::ldp_histogram (include/aldp/descriptors.hpp:55). k must be 3
 * (descriptors.cpp:124-126) -> ALDP_EINVAL otherwise; image >= 3x3. */
aldp_status aldp_ldp_histogram(const uint8_t* pixels, int rows, int cols, int k, int path,
                               uint64_t* bins56);

/* aldp::windowed_features (include/aldp/windowing.hpp:34-36): path selects
 * Descriptor::Ldp / ::Aldp (ALDP_PATH_NAIVE / _ACCELERATED, 56 bins per
 * window) or ::Lbp (ALDP_DESC_LBP, 256 bins). out is [grid_cells][bins]
 * uint64 in row-major window order; out_len must be >= cells*bins. window < 3
 * or larger than the image -> ALDP_EINVAL (windowing.cpp:9-17). */
aldp_status aldp_windowed_features(const uint8_t* pixels, int rows, int cols, int window,
                                   int path, uint64_t* out, size_t out_len);

/* NEW (the reference has no code-map entry point; this is the code that
 * descriptors.cpp:129-136 computes per pixel): codes[rows*cols]. */
aldp_status aldp_ldp_code_map(const uint8_t* pixels, int rows, int cols, int k, int path,
                              uint8_t* codes);

/* aldp::lbp_histogram (descriptors.hpp:66-67): 256 uint64 bins. */
aldp_status aldp_lbp_histogram(const uint8_t* pixels, int rows, int cols, uint64_t* bins256);

/* LBP code map (per-pixel lbp_code, descriptors.cpp:141-157). */
aldp_status aldp_lbp_code_map(const uint8_t* pixels, int rows, int cols, uint8_t* codes);

/* Host batch, LBP descriptor (hist uint32 [n][cells][256]). */
aldp_status aldp_lbp_batch_host(const uint8_t* pixels, int n_images, int rows, int cols, int cell_rows,
                                int cell_cols, uint8_t* codes, uint32_t* hist, void* stream);

/* Host batch: n contiguous rows x cols images in host memory (pinned or
 * pageable) -> optional host code maps and uint32 histograms, one H2D and
 * D2H per call, device buffers cached per thread. The end-to-end path. */
aldp_status aldp_ldp_batch_host(const uint8_t* pixels, int n_images, int rows, int cols, int k,
                                int cell_rows, int cell_cols, uint8_t* codes, uint32_t* hist,
                                void* stream);

/* aldp::make_random (include/aldp/image.hpp:44, reference image.cpp:75-83):
 * rows x cols bytes, std::mt19937(seed) low byte per pixel, row-major (the
 * config-1 input). Host memory; rows, cols >= 3. */
aldp_status aldp_make_random(uint8_t* out, int rows, int cols, uint32_t seed);

/* ---- several GPUs in one process ----
 * aldp_ldp_batch_host over n_devices GPUs: the images are split into
 * contiguous ranges, one per entry of `devices` (NULL: every visible device,
 * n_devices ignored), and each range runs the chunked H2D / kernel / D2H
 * pipeline of aldp_ldp_batch_host on its device from its own persistent host
 * worker thread (its pinned staging and streams are reused across calls).
 * Images are independent, so there is no collective: each device copies its
 * codes and histograms straight into its slice of the caller's buffers.
 * Results are identical for any device list (a device may repeat). The
 * reference's only concurrency is the same fan-out over image ranges, on CPU
 * threads (proj/src/verify.cpp:85-98). Blocks until every range is done. */
aldp_status aldp_ldp_batch_host_multi(const uint8_t* pixels, int n_images, int rows, int cols, int k,
                                      int cell_rows, int cell_cols, uint8_t* codes, uint32_t* hist,
                                      const int* devices, int n_devices);
aldp_status aldp_lbp_batch_host_multi(const uint8_t* pixels, int n_images, int rows, int cols, int cell_rows,
                                      int cell_cols, uint8_t* codes, uint32_t* hist, const int* devices,
                                      int n_devices);

/* Device-resident batches on several GPUs: args[i] (device pointers on
 * devices[i]) is launched on devices[i], stream streams[i] (NULL entries or
 * NULL array: the legacy default stream), all asynchronously; the calling
 * thread's current device is restored. */
aldp_status aldp_ldp_batch_multi(const aldp_ldp_args* args, const int* devices, void* const* streams, int n);

/* Gathers n device buffers into one buffer on dst_device, back to back in
 * order (srcs[i], bytes[i] on src_devices[i]), with peer copies over NVLink
 * (cudaMemcpyPeerAsync) ordered on `stream` (a stream of dst_device). Used
 * for the per-image histogram gather to one GPU. */
aldp_status aldp_gather_peer(void* dst, int dst_device, const void* const* srcs, const int* src_devices,
                             const size_t* bytes, int n, void* stream);

/* ---- response field and the equivalence sweep ---- */

/* Device batch of aldp::response_field (include/aldp/kirsch.hpp:91-92,
 * src/kirsch.cpp:193-208): d_out is int16 [n][rows][cols][8] (16 B/px,
 * 16-byte aligned), direction-minor like ResponseVector::m. path selects the
 * literal masks (ALDP_PATH_NAIVE) or the identity (ALDP_PATH_ACCELERATED);
 * both give identical values. Clamp borders. Image < 3x3 -> ALDP_EINVAL. */
aldp_status aldp_response_field_batch(const uint8_t* d_pixels, int64_t img_stride, int rows, int cols,
                                      int pitch, int n_images, int path, int16_t* d_out, void* stream);
/* Same, int32 output (the reference's ResponseVector width, 32 B/px). */
aldp_status aldp_response_field_batch32(const uint8_t* d_pixels, int64_t img_stride, int rows, int cols,
                                        int pitch, int n_images, int path, int32_t* d_out, void* stream);
/* Host buffers: out = int32 [rows*cols][8], the reference's
 * std::vector<ResponseVector> flattened (kirsch.cpp:193-208). */
aldp_status aldp_response_field(const uint8_t* pixels, int rows, int cols, int path, int32_t* out);

/* aldp::FaultInjection (include/aldp/verify.hpp:14-20): adds delta to column
 * term term_index (0..14, ColumnTerms::a) at pixel (x, y) of image
 * image_index before reconstruction. */
typedef struct {
    int image_index, x, y, term_index, delta;
} aldp_fault;

/* aldp::VerifyResult + Mismatch (verify.hpp:22-37), flattened. Counts follow
 * the reference's bookkeeping for the given thread count (verify.cpp:63-111);
 * `mismatches` (NEW) is the total number of mismatching (pixel, direction)
 * pairs the full device sweep saw. */
typedef struct {
    uint64_t images_checked, pixels_checked, mismatches;
    int has_mismatch; /* !VerifyResult::ok() */
    int image_index, x, y, direction, naive_value, accelerated_value;
} aldp_verify_result;

/* aldp::verify_equivalence (verify.hpp:43-46): `images` (clamped to >= 1)
 * seeded random images with sides in [3, 64] derived from `seed` exactly as
 * the reference does; the sweep runs on the device. fault may be NULL. A
 * term_index outside [0, 15) -> ALDP_ERANGE. */
aldp_status aldp_verify_equivalence(int images, uint32_t seed, const aldp_fault* fault, int threads,
                                    aldp_verify_result* result);
/* aldp::verify_image (verify.hpp:49-51) on host pixels. */
aldp_status aldp_verify_image(const uint8_t* pixels, int rows, int cols, const aldp_fault* fault,
                              int image_index, aldp_verify_result* result);
/* Device batch of equal-size images (the sweep at scale); `threads` only
 * shapes the reported counts as in verify_equivalence. */
aldp_status aldp_verify_batch(const uint8_t* d_pixels, int64_t img_stride, int rows, int cols, int pitch,
                              int n_images, const aldp_fault* fault, int threads,
                              aldp_verify_result* result, void* stream);

/* ---- on-disk input and report formats ---- */

/* aldp::load_pgm (include/aldp/pgm.hpp:15-18, src/pgm.cpp:59-125): P5/P2,
 * maxval <= 255, '#' comments. Writes *rows / *cols (height / width); with
 * out == NULL only the header is read (size query). Format and I/O errors ->
 * ALDP_EIO with the reference's "<path>: <what>" message; cap too small ->
 * ALDP_EINVAL. */
aldp_status aldp_load_pgm(const char* path, uint8_t* out, size_t cap, int* rows, int* cols);
/* aldp::save_pgm (pgm.hpp:20-23): maxval 255, ascii != 0 -> P2. */
aldp_status aldp_save_pgm(const char* path, const uint8_t* pixels, int rows, int cols, int ascii);
/* n equal-size PGM files decoded on `threads` host threads into out
 * [n][rows][cols] (e.g. pinned, then aldp_ldp_batch_host). A file of another
 * size -> ALDP_EINVAL. */
aldp_status aldp_load_pgm_batch(const char* const* paths, int n, int rows, int cols, uint8_t* out, int threads);

/* The CLI's `extract` (tools/aldp_main.cpp:59-96) as one call: CSV header
 * "identifier,descriptor,bin_0..", one row per file (window == 0) or per
 * window "<path>#w<i>" (window >= 3), descriptor "lbp" | "ldp" | "aldp"
 * (case-insensitive), out_path NULL or "" -> stdout. Files are decoded by a
 * thread pool (threads < 1: all cores) one group ahead of the B200, which
 * extracts runs of equal-size images from pinned staging. Rows already
 * written stay written when a later file fails (as the reference streams). */
aldp_status aldp_extract_files(const char* const* paths, int n, const char* descriptor, int window,
                               const char* out_path, int threads);

/* aldp::measured_ops (bench.hpp:42-44): per-pixel (mults, adds) of the
 * reference's arithmetic model; descriptor = ALDP_PATH_NAIVE (LDP),
 * ALDP_PATH_ACCELERATED (ALDP) or ALDP_DESC_LBP. */
aldp_status aldp_op_counts(int descriptor, int* mults, int* adds);

/* The CLI's `bench` (aldp_main.cpp:128-165, bench.cpp:134-178): series
 * "images" (side `size`, default 260, prefixes `counts`) or "window" (side
 * default 300, `windows`), median of `repeats` (>= 3), all three descriptors
 * or the one named, CSV in the reference's schema to out_path (NULL/"" ->
 * stdout). Every timed extraction runs on the B200. */
aldp_status aldp_bench_csv(const char* series, int size, const int* counts, int n_counts, const int* windows,
                           int n_windows, int repeats, uint32_t seed, const char* descriptor,
                           const char* out_path);

/* Message for the last non-OK status returned on this host thread. */
const char* aldp_last_error(void);

/* ---- synthetic inputs (device generators, not part of the timed path) ----
 * Deterministic, keyed by (seed, first_index + i) so any sharding of a batch
 * sees identical bytes. */

/* Face-like images (BASELINE.json configs 2, 4, 5): linear gradient with a
 * seeded direction and endpoints, `blobs` Gaussian blobs (sigma U[5,60] px,
 * amplitude U[-80,80], centres uniform), N(0,6) noise, rounded and clamped. */
aldp_status aldp_gen_faces(uint8_t* d_out, int n_images, int rows, int cols, int pitch,
                           int64_t img_stride, int blobs, uint64_t seed, int64_t first_index,
                           void* stream);

/* Tie-heavy images (config 3): i.i.d. {0,1,2}, then constant rectangles
 * painted until about half the area is covered. */
aldp_status aldp_gen_ties(uint8_t* d_out, int n_images, int rows, int cols, int pitch,
                          int64_t img_stride, uint64_t seed, int64_t first_index, void* stream);

/* Library identity (for load checks): "aldp_b200 <version> sm_100a". */
const char* aldp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ALDP_CUDA_H */
