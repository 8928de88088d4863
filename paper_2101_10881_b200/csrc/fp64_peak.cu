// FP64 issue-rate microbenchmark: the roofline denominator for the
// convolution kernels (the peak must be measured on the box;
// MEASURED_PEAKS.json carries only HBM and bf16 tensor figures).
//
// Each thread runs CH independent dependency chains of DADD (or DFMA) so the
// FP64 pipe, not latency, is the limit; the grid fills every SM. Two shapes
// are timed (16 chains x 4 blocks/SM, 32 chains x 2 blocks/SM, ~2 ms each)
// and the best rate is the peak: with 8 chains x 8 blocks/SM the same
// kernel stays ~4% below (17.0 vs 17.8 T lane-ops/s at 1965 MHz, where
// 148 SMs x 64 lanes give 18.6 T).
#include <cuda_runtime.h>

#include <cstdint>

#include "host_graph.hpp"

namespace pse {
namespace {

constexpr int kIters = 16384;

template <bool FMA, int kChains>
__global__ void __launch_bounds__(256) k_fp64_peak(double* sink, double seed) {
  double a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
  const double b = 1.0000000001, e = 1e-12;
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if constexpr (FMA)
        a[c] = __fma_rn(a[c], b, e);
      else
        a[c] = __dadd_rn(a[c], e);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s = __dadd_rn(s, a[c]);
  if (s == 12345.678) sink[threadIdx.x] = s;  // keep the work alive
}

}  // namespace
}  // namespace pse

extern "C" {

// out[4] = DADD lane-ops/s, DFMA lane-ops/s (one FMA = one instruction),
//          blocks launched, ms of the DADD run
int pse_fp64_peak(int32_t device, double* out) {
  if (cudaSetDevice(device) != cudaSuccess) {
    pse::set_error("cudaSetDevice failed");
    return PSE_ECUDA;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(double)) != cudaSuccess) {
    pse::set_error("cudaMalloc failed");
    return PSE_ECUDA;
  }
  int blocks = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double rate[2] = {0, 0};
  float last = 0;
  for (int shape = 0; shape < 2; ++shape) {
    const int chains = shape ? 32 : 16, nb = sms * (shape ? 2 : 4);
    for (int f = 0; f < 2; ++f) {
      for (int rep = 0; rep < 3; ++rep) {  // warm-up + best of 2
        cudaEventRecord(e0);
        if (shape == 0 && f) pse::k_fp64_peak<true, 16><<<nb, 256>>>(sink, 1.0);
        if (shape == 0 && !f) pse::k_fp64_peak<false, 16><<<nb, 256>>>(sink, 1.0);
        if (shape == 1 && f) pse::k_fp64_peak<true, 32><<<nb, 256>>>(sink, 1.0);
        if (shape == 1 && !f) pse::k_fp64_peak<false, 32><<<nb, 256>>>(sink, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(nb) * 256 * chains * pse::kIters;
        if (rep > 0 && ops / (ms * 1e-3) > rate[f]) {
          rate[f] = ops / (ms * 1e-3);
          if (!f) last = ms, blocks = nb;
        }
      }
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) {
    pse::set_error("fp64 peak kernel failed");
    return PSE_ECUDA;
  }
  out[0] = rate[0];
  out[1] = rate[1];
  out[2] = blocks;
  out[3] = last;
  return PSE_OK;
}

}  // extern "C"
