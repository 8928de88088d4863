// Standalone FP64 issue-rate check (longer runs and more chains than the
// in-library pse_fp64_peak) with the SM clock read from %clock64 / globaltimer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64pk tools/fp64_peak_check.cu
#include <cstdio>
template <int CH>
__global__ void __launch_bounds__(256) pk(double* sink, double seed, int iters, long long* clk) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
  const double e = 1e-12;
  long long c0 = clock64();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __dadd_rn(a[c], e);
  }
  long long c1 = clock64();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s = __dadd_rn(s, a[c]);
  if (s == 12345.678) sink[threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = (long long)(t1 - t0); }
}
template <int CH>
void run(int sms, int bps, int iters) {
  double* sink; long long* clk; cudaMalloc(&sink, 4096); cudaMalloc(&clk, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); pk<CH><<<sms * bps, 256>>>(sink, 1.0, iters, clk); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
  double ops = double(sms) * bps * 256 * CH * double(iters);
  printf("chains %2d blocks/SM %d iters %6d: %.3f ms  %.2f T lane-ops/s  (block0 clock %.0f MHz)  ideal@clk %.2f T\n", CH, bps, iters, best,
         ops / (best * 1e-3) / 1e12, h[0] / (h[1] * 1e-3), sms * 64.0 * h[0] / (h[1] * 1e-3) * 1e-6);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8>(sms, 8, 4096); run<8>(sms, 8, 65536); run<16>(sms, 4, 65536); run<4>(sms, 8, 65536); run<8>(sms, 4, 65536);
  return 0;
}
