// Instantiation of the engine kernels for M = 1 limbs (real and complex).
#define PSE_KERNELS_IMPL
// 512-thread blocks like the larger precisions: the CTA-local dataflow kernel
// runs a whole job group on one block's 16 warps
#ifndef PSE_LANE_THREADS
#define PSE_LANE_THREADS 512
#endif
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(1)
}  // namespace pse
