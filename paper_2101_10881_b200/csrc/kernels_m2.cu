// Instantiation of the engine kernels for M = 2 limbs (real and complex).
#define PSE_KERNELS_IMPL
#if !defined(PSE_LANE_THREADS) && defined(PSE_M2_THREADS)
#define PSE_LANE_THREADS PSE_M2_THREADS
#endif
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(2)
}  // namespace pse
