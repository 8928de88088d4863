// Microbenchmark of the convolution step at M = 10 (analysis only, not the
// product): every thread runs one accumulation chain acc = x0*y, acc += x_i*y
// for T steps, exactly the layered k_conv inner loop (x warp-uniform, y per
// lane, limb-split layout, lane in shared memory, 512-thread blocks, one per
// SM), in variants that drop or change parts of the md_mul / md_add, to
// split the step's time between them. Prints ns per step and the algorithmic
// FP64 rate; a checksum per variant shows which ones are bit-identical to V0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17
//        -I paper_2101_10881_b200/csrc -DPSE_LANE_THREADS=512 -o /tmp/step_bench tools/step_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "md.cuh"

using namespace pse;
constexpr int M = 10;
constexpr int kThreads = PSE_LANE_THREADS;  // chains per block
constexpr int LANE_ROWS = MdTraits<M>::LANE_CONV;

// exp_mul_fast with parts switchable: STAGE bit 1 = compaction, bit 2 = tighten
template <int STAGE>
__device__ __forceinline__ void exp_mul_v(const double (&x)[M], const double (&y)[M], double (&out)[M], Lane ln) {
  if constexpr (STAGE == 3) {
    exp_mul_fast<M>(x, y, out, ln);
  } else {
    constexpr int CAP = MdTraits<M>::CAP;
    const unsigned lim = ln.base + CAP * kRow;
    detail::Passes st;
    st.top = ln.base;
    st.step = ln.step;
    int fed = 0, pushes = 0;
    double e1p = 0.0;
    auto feed = [&](double t) {
      if (fed == 0) st.s1 = t;
      else if (fed == 1) two_sum(t, st.s1, st.s1, st.s2);
      else if (fed == 2) two_sum(t, st.s1, st.s1, e1p);
      else {
        double e1, e2;
        two_sum(t, st.s1, st.s1, e1);
        two_sum(e1p, st.s2, st.s2, e2);
        if (pushes < CAP) detail::push<false>(st, e2, lim);
        else detail::push<true>(st, e2, lim);
        ++pushes;
        e1p = e1;
      }
      ++fed;
    };
    double pr[M];
    {
      double er[M];
#pragma unroll
      for (int i = 0; i < M; ++i) two_prod(x[i], y[M - 1 - i], pr[i], er[i]);
#pragma unroll
      for (int i = M - 1; i >= 0; --i) feed(er[i]);
    }
#pragma unroll
    for (int i = M - 1; i >= 1; --i) feed(__dmul_rn(x[i], y[M - i]));
#pragma unroll
    for (int k = M - 1; k >= 1; --k) {
      double pn[M], en[M];
#pragma unroll
      for (int i = 0; i < k; ++i) two_prod(x[i], y[k - 1 - i], pn[i], en[i]);
#pragma unroll
      for (int i = k - 1; i >= 0; --i) feed(en[i]);
#pragma unroll
      for (int i = k; i >= 0; --i) feed(pr[i]);
#pragma unroll
      for (int i = 0; i < k; ++i) pr[i] = pn[i];
    }
    feed(pr[0]);
    {
      double e;
      two_sum(e1p, st.s2, st.s2, e);
      detail::push<true>(st, e, lim);
      two_sum(st.s1, st.s2, st.s2, e);
      detail::push<true>(st, e, lim);
    }
    if constexpr (STAGE & 1) {
      double eps = st.s2;
      unsigned a = st.top - kRow, ea = st.top - kRow;
      const unsigned elim = st.top - (M + 1) * kRow;
      const unsigned base1 = ln.base + kRow;
      double n0 = lds64(a);
#pragma unroll 1
      while (a >= ln.base && ea != elim) {
        const double n1 = lds64_at<-static_cast<int>(kRow)>(a);
        emit_step<true>(eps, n0, ea, ln.step);
        if (a < base1 || ea == elim) break;
        n0 = lds64_at<-2 * static_cast<int>(kRow)>(a);
        emit_step<true>(eps, n1, ea, ln.step);
        a -= 2 * kRow;
      }
      sts64(ea, eps);
      const unsigned jb = st.top - kRow - ea;
      static_for<M>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        out[k] = lds64_at_if<-(k + 1) * static_cast<int>(kRow), k * kRow>(st.top, jb);
      });
      if constexpr (STAGE & 2) tighten_fast<M, true>(out);
    } else {
      // stream only: keep the results alive
      out[0] = st.s2;
#pragma unroll
      for (int k = 1; k < M; ++k) out[k] = __longlong_as_double(static_cast<long long>(st.top + k));
    }
  }
}

// V: 0 production step; 1 mul only; 2 mul stream only; 3 mul without tighten;
//    4 add only (product = x + lane-dependent y, no md_mul)
template <int V>
__global__ void __launch_bounds__(kThreads, 512 / kThreads) kstep(const double* __restrict__ X, const double* __restrict__ Y,
                                                     double* out, int T, int S) {
  extern __shared__ double smem[];
  Lane ln = make_lane(smem);
  const int tid = threadIdx.x;
  const double* Yb = Y + static_cast<size_t>(blockIdx.x % 8) * M * S;
  double o[M];
  unsigned long long ck = 0;
  acc_init<M>(ln);
#pragma unroll 1
  for (int i = 0; i < T; ++i) {
    double xr[M], yr[M], p[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      xr[q] = __ldg(X + q * S + i);
      yr[q] = __ldg(Yb + q * S + tid + T - 1 - i);
    }
    if constexpr (V == 0) exp_mul_v<3>(xr, yr, p, ln);
    else if constexpr (V == 1) exp_mul_v<3>(xr, yr, p, ln);
    else if constexpr (V == 2) exp_mul_v<0>(xr, yr, p, ln);
    else if constexpr (V == 3) exp_mul_v<1>(xr, yr, p, ln);
    else {
#pragma unroll
      for (int q = 0; q < M; ++q) p[q] = yr[q];
    }
    if constexpr (V == 0 || V == 4) {
      if (i == 0) {
#pragma unroll
        for (int q = 0; q < M; ++q) o[q] = p[q];
        acc_store<M>(p, ln);
      } else {
        acc_add<M>(p, o, ln);
      }
    } else {
#pragma unroll
      for (int q = 0; q < M; ++q) ck ^= static_cast<unsigned long long>(__double_as_longlong(p[q])) + q;
    }
  }
  if constexpr (V == 0 || V == 4) {
#pragma unroll
    for (int q = 0; q < M; ++q) ck ^= static_cast<unsigned long long>(__double_as_longlong(o[q])) * (q + 1);
  }
  out[blockIdx.x * kThreads + tid] = __longlong_as_double(static_cast<long long>(ck));
}


template <class F>
float time_kernel(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <int V>
void run(const char* name, const double* X, const double* Y, double* out, int T, int S, int blocks, double peak) {
  const size_t sh = static_cast<size_t>(LANE_ROWS) * kThreads * sizeof(double);
  cudaFuncSetAttribute(kstep<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sh));
  float ms = time_kernel([&] { kstep<V><<<blocks, kThreads, sh>>>(X, Y, out, T, S); }, 5);
  cudaError_t e = cudaGetLastError();
  std::vector<unsigned long long> h(blocks * kThreads);
  cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long c = 0;
  for (auto v : h) c = c * 1000003ull + v;
  const double steps = static_cast<double>(blocks) * kThreads * T;
  const double ops = static_cast<double>(blocks) * kThreads * (T * 1944.0 + (T - 1) * 279.0);
  // cycles per warp-step on one SM sub-partition (4 per SM) at 1965 MHz
  const double cyc = ms * 1.965e6 / (steps / 32.0 / (148.0 * 4));
  printf("V%d %-28s %8.3f ms  %7.1f cyc/warp-step/SMSP  alg %.2f T ops/s  frac %.3f  ck %016llx %s\n", V, name, ms,
         cyc, ops / ms / 1e9, ops / ms / 1e9 / peak, c,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 128;
  const int waves = argc > 2 ? atoi(argv[2]) : 4;
  const double peak = 18.0;  // measured FP64 issue rate, T lane-ops/s
  const int S = 1024;
  const int blocks = 148 * (512 / kThreads) * waves;  // V0-V4: two 256-thread blocks per SM; V5: one block (256 chains) per SM
  // random md values like the reference's random_md: limb k ~ U(-1,1) 2^-53k, renormalised by exp_add with 0
  std::vector<double> hx(M * S), hy(8 * M * S);
  unsigned long long s = 0x9e3779b97f4a7c15ull;
  auto rnd = [&] {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    return static_cast<double>(s >> 11) * 0x1p-52 - 1.0;
  };
  auto fill = [&](double* v, int n) {
    for (int j = 0; j < n; ++j) {
      double t[M];
      for (int q = 0; q < M; ++q) t[q] = rnd() * ldexp(1.0, -53 * q);
      // renormalise on the host: vec_sum + err_branch + tighten as the reference's renormalize
      double sum = t[M - 1];
      for (int i = M - 2; i >= 0; --i) {
        double a = t[i], ss = a + sum, bv = ss - a, av = ss - bv;
        t[i + 1] = (a - av) + (sum - bv);
        sum = ss;
      }
      t[0] = sum;
      for (int q = 0; q < M; ++q) v[q * S + j] = t[q];  // (not fully renormalised; fine for timing)
    }
  };
  fill(hx.data(), S);
  for (int b = 0; b < 8; ++b) fill(hy.data() + b * M * S, S);
  double *X, *Y, *out;
  cudaMalloc(&X, hx.size() * 8);
  cudaMalloc(&Y, hy.size() * 8);
  cudaMalloc(&out, static_cast<size_t>(blocks) * kThreads * 8);
  cudaMemcpy(X, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(Y, hy.data(), hy.size() * 8, cudaMemcpyHostToDevice);
  printf("T=%d steps, %d blocks of %d threads, lane %d rows\n", T, blocks, kThreads, LANE_ROWS);
  run<0>("production mul+add", X, Y, out, T, S, blocks, peak);
  if (argc > 3) return 0;  // V0 only
  run<1>("mul only", X, Y, out, T, S, blocks, peak);
  run<2>("mul stream only", X, Y, out, T, S, blocks, peak);
  run<3>("mul, no tighten", X, Y, out, T, S, blocks, peak);
  run<4>("add only", X, Y, out, T, S, blocks, peak);
  return 0;
}
