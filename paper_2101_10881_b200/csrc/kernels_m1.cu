// Instantiation of the engine kernels for M = 1 limbs (real and complex).
#define PSE_KERNELS_IMPL
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(1)
}  // namespace pse
