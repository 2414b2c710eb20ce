// ldp_fast_cells.cu -- the cell-histogram instantiations of the packed LDP /
// LBP kernel (the C2 / C4 / C5 hot path), compiled apart from ldp_kernels.cu
// so they can take their own ptxas options (see ldp_fast_launch.cuh).
#include <cuda_runtime.h>
#include <cstdint>
#include "aldp_cuda.h"
#include "ldp_common.cuh"
#include "ldp_fast_launch.cuh"

namespace aldp_b200 {
ALDP_FAST_CELL_INSTANTIATIONS(template)
}  // namespace aldp_b200
