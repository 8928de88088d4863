// Microbenchmark: FP64 issue rate of ONE warp per SM sub-partition (and of
// 2 / 4 warps) on sm_100a: K independent acc += a*b chains (DMUL + DADD per
// step). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_warp_rate tools/fp64_warp_rate.cu
#include <cstdio>
template <int K>
__global__ void rate(double* out, long long* cyc, double a, int n) {
  double acc[K], b[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    acc[k] = -0.0;
    b[k] = a + k;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(b[k], a));
    a = __dadd_rn(a, 1e-300);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int K>
void run(int warps, double* o, long long* c) {
  int n = 1 << 14;
  rate<K><<<1, 32 * warps>>>(o, c, 1.5, n);
  rate<K><<<1, 32 * warps>>>(o, c, 1.5, n);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("K=%2d chains, %d warp(s)/SM: %.2f cycles per step per warp (%.2f cycles per FP64 instr)\n", K, warps,
         h / (double)n, h / (double)n / (2 * K + 1));
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 1 << 20);
  cudaMalloc(&c, 64);
  for (int w : {1, 4, 8}) {
    run<1>(w, o, c);
    run<2>(w, o, c);
    run<4>(w, o, c);
    run<8>(w, o, c);
  }
  return 0;
}
