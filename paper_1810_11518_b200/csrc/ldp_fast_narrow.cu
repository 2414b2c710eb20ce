// ldp_fast_narrow.cu -- the narrow-cell instantiations of the packed LDP
// kernel (cells of 9 .. 31 columns, e.g. the paper's 10 / 20 / 25-pixel
// windows, Table 3): count-only regions for up to 16 cells per tile
// (ldp_fast.cuh FastLayout). A translation unit of their own so they build in
// parallel with the other instantiations.
#include <cuda_runtime.h>
#include <cstdint>
#include "aldp_cuda.h"
#include "ldp_common.cuh"
#include "ldp_fast_launch.cuh"

namespace aldp_b200 {
ALDP_FAST_NARROW_INSTANTIATIONS(template)
}  // namespace aldp_b200
