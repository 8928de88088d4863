// Microbenchmark: FP64 issue rate of independent DADD chains mixed with
// integer / shared-memory instructions at the ratios of the conv kernel's
// instruction stream (tools only; measures what the FP64 pipe sustains when
// it shares the issue port). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64mix tools/fp64_mix.cu
#include <cstdio>
#include <cstdint>

template <int NINT, bool STS>
__global__ void __launch_bounds__(512, 1) mix(double* out, int n, double a, double b) {
  __shared__ double sm[512 * 4];
  double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  unsigned u0 = threadIdx.x, u1 = u0 * 3, u2 = u0 * 5, u3 = u0 * 7;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
      x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
      // NINT integer ops per 8 DADDs, independent chains
#pragma unroll
      for (int k = 0; k < NINT; ++k) {
        if (k % 4 == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u0) : "r"(u1), "r"(u2));
        if (k % 4 == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(u1) : "r"(u3));
        if (k % 4 == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0xe8;" : "+r"(u2) : "r"(u0), "r"(u3));
        if (k % 4 == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(u3) : "r"(u2));
      }
      if (STS) sm[threadIdx.x + 512 * (r & 3)] = x0;
    }
  }
  out[blockIdx.x * 512 + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + u0 + u1 + u2 + u3 + sm[threadIdx.x];
}

template <int NINT, bool STS>
void run(double* out, int sms) {
  const int n = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<NINT, STS><<<sms, 512>>>(out, 100, 1.0, 1e-9);
  cudaEventRecord(e0);
  mix<NINT, STS><<<sms, 512>>>(out, n, 1.0, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dadd = double(sms) * 512 * n * 32;
  printf("int per 8 DADD %d sts %d: %.2f T DADD lane-ops/s (%.3f ms)\n", NINT, STS, dadd / (ms * 1e-3) / 1e12, ms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 512);
  run<0, false>(out, sms);
  run<2, false>(out, sms);
  run<4, false>(out, sms);
  run<6, false>(out, sms);
  run<8, false>(out, sms);
  run<4, true>(out, sms);
  run<6, true>(out, sms);
  return 0;
}
