// Instantiation of the engine kernels for M = 8 limbs (real and complex).
#define PSE_KERNELS_IMPL
// 512-thread blocks (one per SM): the 16 warps an SM holds start together,
// which keeps the instruction stream they share in cache (C2 -2%, C3' -6%
// against four 128-thread blocks); the register and shared-memory budget per
// thread is unchanged. M <= 2 keeps 128: its lighter threads fit more warps.
#ifndef PSE_LANE_THREADS
#ifdef PSE_M8_THREADS
#define PSE_LANE_THREADS PSE_M8_THREADS
#else
#define PSE_LANE_THREADS 512
#endif
#endif
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(8)
}  // namespace pse
