// Instantiation of the engine kernels for M = 3 limbs (real and complex).
#define PSE_KERNELS_IMPL
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(3)
}  // namespace pse
