// Instantiation of the engine kernels for M = 2 limbs (real and complex).
#define PSE_KERNELS_IMPL
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(2)
}  // namespace pse
