// Microbenchmark: dependent-chain latency (cycles) of DADD / DFMA / DSETP+FSEL
// and LDS on sm_100a, one warp. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/fp64_latency.cu
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, int n) {
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, y); x = __dadd_rn(x, -y); }
  long long t1 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) { z = __fma_rn(z, 1.0000001, y); z = __fma_rn(z, 0.9999999, -y); }
  long long t2 = clock64();
  __shared__ double sm[64];
  sm[threadIdx.x] = a;
  __syncthreads();
  unsigned addr = (unsigned)__cvta_generic_to_shared(sm + threadIdx.x);
  double w = 0;
  for (int i = 0; i < n; ++i) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    addr += (v == 12345.0) ? 8 : 0;
    w = __dadd_rn(w, v);
  }
  long long t3 = clock64();
  out[threadIdx.x] = x + z + w;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 512); cudaMalloc(&c, 64);
  int n = 1 << 16;
  for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(o, c, 1.5, n);
  long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", h[0] / (2.0 * n));
  printf("DFMA dependent latency: %.2f cycles\n", h[1] / (2.0 * n));
  printf("LDS->ISETP->addr->LDS chain: %.2f cycles/iter\n", h[2] / (1.0 * n));
  return 0;
}
