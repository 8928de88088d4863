// Instantiation of the engine kernels for M = 2 limbs (real and complex).
#define PSE_KERNELS_IMPL
// 512-thread blocks like the larger precisions: the CTA-local dataflow kernel
// runs a whole job group on one block's 16 warps
#ifndef PSE_LANE_THREADS
#ifdef PSE_M2_THREADS
#define PSE_LANE_THREADS PSE_M2_THREADS
#else
#define PSE_LANE_THREADS 512
#endif
#endif
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(2)
}  // namespace pse
