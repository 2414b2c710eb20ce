// ldp_fast_launch.cuh -- host launcher of the packed kernel (ldp_fast.cuh),
// shared by ldp_kernels.cu and ldp_fast_cells.cu. The cell-histogram
// instantiations live in ldp_fast_cells.cu, which is compiled with
// `-Xptxas --register-usage-level=10`: that ptxas schedule is faster for the
// cell kernel (C5 +1.5 %, C4 +2 %) and slower for the whole-image kernel
// (C3 -2.5 %), measured A/B.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include "aldp_cuda.h"
#include "ldp_common.cuh"
#include "ldp_fast.cuh"

namespace aldp_b200 {

aldp_status set_error(aldp_status s, const std::string& msg);  // ldp_kernels.cu
int fast_n_sms();                                               // ldp_kernels.cu
void count_launch();                                            // ldp_kernels.cu (aldp_last_launch_count)

inline aldp_status fast_cuda_fail(cudaError_t e, const char* what) {
    return set_error(ALDP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <int K, int NW, bool CELLS, bool CODES, bool HIST, bool HALO, int NC = kMaxTileCells>
aldp_status launch_fast_t(const FastParams& p, cudaStream_t st) {
    auto kern = ldp_fast_kernel<K, NW, CELLS, CODES, HIST, HALO, NC>;
    constexpr int NSEG = FastLayout<K, NW, NC>::NSEG;
    const size_t smem = FastLayout<K, NW, NC>::BYTES;
    // The shared-memory opt-in is a per-device function attribute: set it once
    // per device this process launches on (several GPUs in one process work).
    constexpr int kMaxDev = 64;
    static std::once_flag once[kMaxDev];
    static cudaError_t attr_err[kMaxDev];
    static int per_sm_dev[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) return fast_cuda_fail(cudaErrorInvalidDevice, "fast kernel setup");
    std::call_once(once[dev], [&] {
        int ps = 1;
        attr_err[dev] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (attr_err[dev] == cudaSuccess)
            attr_err[dev] = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, kFastWarps * 32, smem);
        per_sm_dev[dev] = ps < 1 ? 1 : ps;
    });
    if (attr_err[dev] != cudaSuccess) return fast_cuda_fail(attr_err[dev], "fast kernel setup");
    const int per_sm = per_sm_dev[dev];
    const int64_t warp_tiles = (p.n_tiles + NSEG - 1) / NSEG;
    const int64_t want = (warp_tiles + kFastWarps - 1) / kFastWarps;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(per_sm) * fast_n_sms())));
    kern<<<grid, kFastWarps * 32, smem, st>>>(p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fast_cuda_fail(e, "ldp_fast_kernel launch");
    return ALDP_OK;
}

// The cell-histogram launches (CELLS = HIST = true): K = 0..7, with and
// without the code map, plain frames and band views. X is `template` (the
// definitions, ldp_fast_cells.cu) or `extern template` (ldp_kernels.cu).
#define ALDP_FAST_CELL_INST_K(X, K)                                                              \
    X aldp_status launch_fast_t<K, 2, true, true, true, false>(const FastParams&, cudaStream_t);  \
    X aldp_status launch_fast_t<K, 2, true, false, true, false>(const FastParams&, cudaStream_t); \
    X aldp_status launch_fast_t<K, 2, true, true, true, true>(const FastParams&, cudaStream_t);   \
    X aldp_status launch_fast_t<K, 2, true, false, true, true>(const FastParams&, cudaStream_t);
// Narrow cells (9 .. 31 columns: up to kNarrowTileCells per tile), LDP k != 4.
#define ALDP_FAST_NARROW_INST_K(X, K)                                                                             \
    X aldp_status launch_fast_t<K, 2, true, true, true, false, kNarrowTileCells>(const FastParams&, cudaStream_t);  \
    X aldp_status launch_fast_t<K, 2, true, false, true, false, kNarrowTileCells>(const FastParams&, cudaStream_t); \
    X aldp_status launch_fast_t<K, 2, true, true, true, true, kNarrowTileCells>(const FastParams&, cudaStream_t);   \
    X aldp_status launch_fast_t<K, 2, true, false, true, true, kNarrowTileCells>(const FastParams&, cudaStream_t);
#define ALDP_FAST_NARROW_INSTANTIATIONS(X)                                                    \
    ALDP_FAST_NARROW_INST_K(X, 1) ALDP_FAST_NARROW_INST_K(X, 2) ALDP_FAST_NARROW_INST_K(X, 3) \
    ALDP_FAST_NARROW_INST_K(X, 5) ALDP_FAST_NARROW_INST_K(X, 6) ALDP_FAST_NARROW_INST_K(X, 7)
#define ALDP_FAST_CELL_INSTANTIATIONS(X)                                              \
    ALDP_FAST_CELL_INST_K(X, 0) ALDP_FAST_CELL_INST_K(X, 1) ALDP_FAST_CELL_INST_K(X, 2) \
    ALDP_FAST_CELL_INST_K(X, 3) ALDP_FAST_CELL_INST_K(X, 4) ALDP_FAST_CELL_INST_K(X, 5) \
    ALDP_FAST_CELL_INST_K(X, 6) ALDP_FAST_CELL_INST_K(X, 7)

}  // namespace aldp_b200
