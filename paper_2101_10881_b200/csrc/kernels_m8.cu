// Instantiation of the engine kernels for M = 8 limbs (real and complex).
#define PSE_KERNELS_IMPL
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(8)
}  // namespace pse
