// Microbenchmark: FP64 issue rate of independent DADD chains mixed with
// independent integer instructions (tools only). Tests whether an FP64
// warp-instruction (2 cycles on a 16-lane pipe) also holds the scheduler's
// dispatch for 2 cycles: if so, K integer ops per 8 DADDs cost K extra issue
// cycles and the DADD rate falls as 16 / (16 + K) of peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64mix tools/fp64_mix.cu
#include <cstdio>
#include <cstdint>

template <int NINT>
__global__ void __launch_bounds__(512, 1) mix(double* out, unsigned* uo, int n, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = out[c * 512 + threadIdx.x];
  unsigned u[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) u[c] = uo[c * 512 + threadIdx.x];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = __dadd_rn(x[c], b);
#pragma unroll
      for (int k = 0; k < NINT; ++k) asm volatile("lop3.b32 %0, %0, %1, 0x55aa, 0x96;" : "+r"(u[k % 8]) : "r"(u[(k + 3) % 8]));
    }
  }
  double s = 0;
  unsigned t = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) { s += x[c]; t ^= u[c]; }
  out[blockIdx.x * 512 + threadIdx.x] = s;
  uo[blockIdx.x * 512 + threadIdx.x] = t;
}

template <int NINT>
void run(double* out, unsigned* uo, int sms) {
  const int n = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<NINT><<<sms, 512>>>(out, uo, 100, 1e-9);
  cudaEventRecord(e0);
  mix<NINT><<<sms, 512>>>(out, uo, n, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaError_t err = cudaGetLastError();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dadd = double(sms) * 512 * n * 32;
  printf("int ops per 8 DADD %2d: %.2f T DADD lane-ops/s (%.3f ms) %s\n", NINT, dadd / (ms * 1e-3) / 1e12, ms,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  unsigned* uo;
  cudaMalloc(&out, sizeof(double) * sms * 512 * 8);
  cudaMalloc(&uo, sizeof(unsigned) * sms * 512 * 8);
  cudaMemset(out, 0, sizeof(double) * sms * 512 * 8);
  cudaMemset(uo, 0, sizeof(unsigned) * sms * 512 * 8);
  run<0>(out, uo, sms);
  run<2>(out, uo, sms);
  run<4>(out, uo, sms);
  run<6>(out, uo, sms);
  run<8>(out, uo, sms);
  run<12>(out, uo, sms);
  run<16>(out, uo, sms);
  return 0;
}
