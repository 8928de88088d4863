// Instantiation of the engine kernels for M = 1 limbs (real and complex).
#define PSE_KERNELS_IMPL
// 1024-thread blocks: the CTA-local dataflow kernel runs a whole job group on
// one block, and at M = 1 (a DMUL + DADD per step, <= 64 registers) 32 warps
// hide its latencies better than 16 (C3 m=1: 0.495 -> 0.394 ms)
#ifndef PSE_LANE_THREADS
#ifdef PSE_M1_THREADS
#define PSE_LANE_THREADS PSE_M1_THREADS
#else
#define PSE_LANE_THREADS 1024
#endif
#endif
#include "kernels.cuh"

namespace pse {
PSE_INSTANTIATE(1)
}  // namespace pse
