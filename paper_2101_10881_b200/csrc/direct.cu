// Independent device evaluator: eval_direct (proj/src/oracle_direct.cpp:41-78)
// restated for the GPU, for `verify` (proj/tools/pseval.cpp:97-118) to check
// the engine against.
//
// Independent of the engine on both axes the engine could be wrong in:
//  * the algorithm: no job graph -- every monomial's value term
//    a_k * z_i1^e1 * z_i2^e2 * ... and every derivative term is formed by its
//    own left-to-right product chain (oracle_direct.cpp:55-76), then summed
//    in monomial order; the engine's reverse-mode forward/backward/cross
//    products and its addition tree are not used;
//  * the arithmetic: the literal md operations (exp_add_lit / exp_mul_lit in
//    md.cuh, restatements of expansion.hpp:142-211 over local arrays), not
//    the register-streamed ones every engine kernel runs.
// Parallel shape: one block per product chain, one thread per output
// coefficient, a block barrier between consecutive convolutions (each
// coefficient of a product needs every lower one of the previous); then one
// thread per (row, coefficient) folds the terms of a row in order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "md.cuh"
#include "pse_b200.h"

namespace pse {
void set_error(const std::string& msg);  // host_graph.cpp

namespace {

struct DirectArgs {
  int d, Q;               // Q = parts * M
  const double* stat;     // [Q][rows][d+1], rows = 1 + N + n
  int rows;
  const int* chain_coeff; // [nchains] static slot of the chain's coefficient a_k
  const int* chain_off;   // [nchains+1] into chain_z
  const int* chain_z;     // static slots of the factors, in multiplication order
  const int* chain_scale; // [nchains] series_scale_int factor (1 = none)
  double* buf;            // [nchains][2][Q][d+1] ping-pong products
  const int* row_off;     // [n+2] into row_chain: row 0 = value, 1+i = gradient i
  const int* row_chain;   // chain ids in summation order
  double* out;            // [Q][n+1][d+1]
};

template <int M>
__device__ void md_add_l(const double* x, const double* y, double* z) {
  if constexpr (M == 1)
    z[0] = __dadd_rn(x[0], y[0]);
  else
    exp_add_lit<M>(x, y, z);
}
template <int M>
__device__ void md_sub_l(const double* x, const double* y, double* z) {
  double ny[M];
  for (int q = 0; q < M; ++q) ny[q] = -y[q];
  md_add_l<M>(x, ny, z);
}
template <int M>
__device__ void md_mul_l(const double* x, const double* y, double* z) {
  if constexpr (M == 1)
    z[0] = __dmul_rn(x[0], y[0]);
  else
    exp_mul_lit<M>(x, y, z);
}

// limb-split series access: part p, limb q of coefficient j at s[(p*M+q)*(d+1)+j]
template <int M>
__device__ void get(const double* s, int stride, int part, int j, double* v) {
  for (int q = 0; q < M; ++q) v[q] = s[(part * M + q) * stride + j];
}
template <int M>
__device__ void put(double* s, int stride, int part, int j, const double* v) {
  for (int q = 0; q < M; ++q) s[(part * M + q) * stride + j] = v[q];
}

// coefficient k of conv(x, y) (pseries.cpp:37-64), literal md arithmetic
template <int M, bool CPLX>
__device__ void conv_coeff(const double* x, int xs, const double* y, int ys, int k, double* re, double* im) {
  double a[M], b[M], p[M], p2[M], t[M];
  for (int i = 0; i <= k; ++i) {
    if constexpr (!CPLX) {
      get<M>(x, xs, 0, i, a);
      get<M>(y, ys, 0, k - i, b);
      md_mul_l<M>(a, b, p);
      if (i == 0)
        for (int q = 0; q < M; ++q) re[q] = p[q];
      else
        md_add_l<M>(re, p, re);
    } else {
      double ai[M], bi[M];
      get<M>(x, xs, 0, i, a);
      get<M>(x, xs, 1, i, ai);
      get<M>(y, ys, 0, k - i, b);
      get<M>(y, ys, 1, k - i, bi);
      md_mul_l<M>(a, b, p);
      md_mul_l<M>(ai, bi, p2);
      md_sub_l<M>(p, p2, t);  // pre
      if (i == 0)
        for (int q = 0; q < M; ++q) re[q] = t[q];
      else
        md_add_l<M>(re, t, re);
      md_mul_l<M>(a, bi, p);
      md_mul_l<M>(ai, b, p2);
      md_add_l<M>(p, p2, t);  // pim
      if (i == 0)
        for (int q = 0; q < M; ++q) im[q] = t[q];
      else
        md_add_l<M>(im, t, im);
    }
  }
}

// one block per chain: t = a_k; t = conv(t, z) for each factor; scale
template <int M, bool CPLX>
__global__ void k_direct_chain(DirectArgs a) {
  constexpr int P = CPLX ? 2 : 1;
  const int c = blockIdx.x;
  const int d1 = a.d + 1;
  const int64_t sw = static_cast<int64_t>(a.Q) * d1;
  double* b0 = a.buf + static_cast<int64_t>(c) * 2 * sw;
  double* b1 = b0 + sw;
  const int stat_stride = a.rows * d1;  // limb q of slot s at stat[q*rows*d1 + s*d1 + j]
  const double* coeff = a.stat + static_cast<int64_t>(a.chain_coeff[c]) * d1;
  for (int j = threadIdx.x; j < d1; j += blockDim.x)
    for (int q = 0; q < a.Q; ++q) b0[q * d1 + j] = coeff[static_cast<int64_t>(q) * stat_stride + j];
  __syncthreads();
  double* cur = b0;
  double* nxt = b1;
  for (int f = a.chain_off[c]; f < a.chain_off[c + 1]; ++f) {
    const double* z = a.stat + static_cast<int64_t>(a.chain_z[f]) * d1;
    for (int k = threadIdx.x; k < d1; k += blockDim.x) {
      double re[M], im[M];
      conv_coeff<M, CPLX>(cur, d1, z, stat_stride, k, re, im);
      put<M>(nxt, d1, 0, k, re);
      if constexpr (CPLX) put<M>(nxt, d1, 1, k, im);
    }
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  const int sc = a.chain_scale[c];
  for (int k = threadIdx.x; k < d1; k += blockDim.x) {
    for (int part = 0; part < P; ++part) {
      double v[M], s[M], r[M];
      get<M>(cur, d1, part, k, v);
      if (sc != 1) {  // series_scale_int (pseries.cpp:85-93): md_mul(x_k, c)
        for (int q = 0; q < M; ++q) s[q] = q == 0 ? static_cast<double>(sc) : 0.0;
        md_mul_l<M>(v, s, r);
      } else {
        for (int q = 0; q < M; ++q) r[q] = v[q];
      }
      put<M>(b0, d1, part, k, r);  // final product in buffer 0
    }
  }
}

// one thread per (row, part, coefficient): value = a0 + v_1 + v_2 + ...;
// gradient i = first term, then series_add(acc, t) (oracle_direct.cpp:62, 76)
template <int M, bool CPLX>
__global__ void k_direct_rows(DirectArgs a, int nrows) {
  constexpr int P = CPLX ? 2 : 1;
  const int d1 = a.d + 1;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<int64_t>(nrows) * P * d1) return;
  const int k = static_cast<int>(g % d1);
  const int part = static_cast<int>((g / d1) % P);
  const int row = static_cast<int>(g / (static_cast<int64_t>(d1) * P));
  const int64_t sw = static_cast<int64_t>(a.Q) * d1;
  double acc[M], t[M];
  int first = a.row_off[row];
  if (row == 0) {
    const int stat_stride = a.rows * d1;
    for (int q = 0; q < M; ++q) acc[q] = a.stat[static_cast<int64_t>(part * M + q) * stat_stride + k];  // a0
  } else if (first < a.row_off[row + 1]) {
    get<M>(a.buf + static_cast<int64_t>(a.row_chain[first]) * 2 * sw, d1, part, k, acc);
    ++first;
  } else {
    for (int q = 0; q < M; ++q) acc[q] = 0.0;  // variable in no monomial: zero series
  }
  for (int e = first; e < a.row_off[row + 1]; ++e) {
    get<M>(a.buf + static_cast<int64_t>(a.row_chain[e]) * 2 * sw, d1, part, k, t);
    md_add_l<M>(acc, t, acc);
  }
  const int64_t plane = static_cast<int64_t>(nrows) * d1;
  for (int q = 0; q < M; ++q) a.out[(part * M + q) * plane + static_cast<int64_t>(row) * d1 + k] = acc[q];
}

template <int M, bool CPLX>
void launch(const DirectArgs& a, int nchains, int nrows, int threads) {
  if (nchains > 0) k_direct_chain<M, CPLX><<<nchains, threads>>>(a);
  const int64_t n = static_cast<int64_t>(nrows) * (CPLX ? 2 : 1) * (a.d + 1);
  k_direct_rows<M, CPLX><<<static_cast<unsigned>((n + 127) / 128), 128>>>(a, nrows);
}

void dispatch(int m, bool cplx, const DirectArgs& a, int nchains, int nrows, int threads) {
#define PSE_DIRECT_CASE(MM) \
  case MM: cplx ? launch<MM, true>(a, nchains, nrows, threads) : launch<MM, false>(a, nchains, nrows, threads); break;
  switch (m) {
    PSE_DIRECT_CASE(1)
    PSE_DIRECT_CASE(2)
    PSE_DIRECT_CASE(3)
    PSE_DIRECT_CASE(4)
    PSE_DIRECT_CASE(5)
    PSE_DIRECT_CASE(8)
    PSE_DIRECT_CASE(10)
    default: throw std::invalid_argument("unsupported precision level");
  }
#undef PSE_DIRECT_CASE
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t total_degree(int nk, const int32_t* exps) {
  if (!exps) return nk;
  int64_t q = 0;
  for (int j = 0; j < nk; ++j) q += exps[j];
  return q;
}

}  // namespace
}  // namespace pse

extern "C" {

// within_oracle_guard (oracle_direct.cpp:32-39): N * max total degree * (d+1)^2 <= 1e7
int pse_within_oracle_guard(int32_t d, int32_t N, const int32_t* nvars, const int32_t* exponents) {
  if (!nvars || N < 0 || d < 0) return PSE_EINVAL;
  int64_t worst = 1, pos = 0;
  for (int k = 0; k < N; ++k) {
    const bool has = exponents && [&] {
      for (int j = 0; j < nvars[k]; ++j)
        if (exponents[pos + j] != 0) return true;
      return false;
    }();
    worst = std::max(worst, pse::total_degree(nvars[k], has ? exponents + pos : nullptr));
    pos += nvars[k];
  }
  const int64_t d1 = static_cast<int64_t>(d) + 1;
  return static_cast<int64_t>(N) * worst * d1 * d1 <= 10000000LL ? 1 : 0;
}

int pse_eval_direct(int32_t n, int32_t d, int32_t m, int32_t mode, int32_t N, const int32_t* nvars,
                    const int32_t* indices, const int32_t* exponents, const double* stat, double* vg_out,
                    int32_t device) {
  try {
    if (!nvars || !indices || !stat || !vg_out) throw std::invalid_argument("null argument");
    if (m != 1 && m != 2 && m != 3 && m != 4 && m != 5 && m != 8 && m != 10)
      throw std::invalid_argument("unsupported precision level");
    if (mode != PSE_MODE_REAL && mode != PSE_MODE_COMPLEX) throw std::invalid_argument("unsupported mode");
    if (n < 1) throw std::invalid_argument("polynomial needs at least one variable");
    if (d < 0) throw std::invalid_argument("negative truncation degree");
    if (pse_within_oracle_guard(d, N, nvars, exponents) != 1)
      throw std::invalid_argument("instance exceeds the direct-evaluation size guard");
    const int rows = 1 + N + n;
    // chains in oracle_direct.cpp's order: per monomial, the value term, then
    // the derivative term of each position j
    std::vector<int> coeff, off{0}, zs, scale, row_off, row_chain;
    std::vector<std::vector<int>> row_terms(1 + n);
    int64_t pos = 0;
    for (int k = 0; k < N; ++k) {
      const int nk = nvars[k];
      if (nk < 1) throw std::invalid_argument("monomial without variables");
      bool has = false;
      if (exponents)
        for (int j = 0; j < nk; ++j) has = has || exponents[pos + j] != 0;
      auto ex = [&](int j) { return has ? exponents[pos + j] : 1; };
      for (int j = 0; j < nk; ++j) {
        if (indices[pos + j] < 1 || indices[pos + j] > n) throw std::invalid_argument("variable index out of range");
        if (ex(j) < 1) throw std::invalid_argument("exponents must be positive");
      }
      auto chain = [&](int skip) {  // skip = position whose exponent drops by one (-1: value term)
        coeff.push_back(1 + k);
        for (int l = 0; l < nk; ++l)
          for (int q = 0; q < ex(l) - (l == skip ? 1 : 0); ++q) zs.push_back(N + indices[pos + l]);
        off.push_back(static_cast<int>(zs.size()));
        scale.push_back(skip >= 0 && ex(skip) != 1 ? ex(skip) : 1);
        return static_cast<int>(coeff.size()) - 1;
      };
      row_terms[0].push_back(chain(-1));
      for (int j = 0; j < nk; ++j) row_terms[indices[pos + j]].push_back(chain(j));
      pos += nk;
    }
    row_off.push_back(0);
    for (auto& r : row_terms) {
      row_chain.insert(row_chain.end(), r.begin(), r.end());
      row_off.push_back(static_cast<int>(row_chain.size()));
    }
    const int Q = (mode == PSE_MODE_COMPLEX ? 2 : 1) * m;
    const int nchains = static_cast<int>(coeff.size());
    pse::ck(cudaSetDevice(device), "cudaSetDevice");
    std::vector<void*> owned;
    auto up = [&](const void* h, size_t bytes) {
      void* p = nullptr;
      pse::ck(cudaMalloc(&p, std::max<size_t>(bytes, 8)), "cudaMalloc");
      owned.push_back(p);
      if (h && bytes) pse::ck(cudaMemcpy(p, h, bytes, cudaMemcpyHostToDevice), "H2D");
      return p;
    };
    try {
      pse::DirectArgs a{};
      a.d = d;
      a.Q = Q;
      a.rows = rows;
      a.stat = static_cast<const double*>(up(stat, sizeof(double) * Q * rows * (d + 1)));
      a.chain_coeff = static_cast<const int*>(up(coeff.data(), sizeof(int) * coeff.size()));
      a.chain_off = static_cast<const int*>(up(off.data(), sizeof(int) * off.size()));
      a.chain_z = static_cast<const int*>(up(zs.data(), sizeof(int) * zs.size()));
      a.chain_scale = static_cast<const int*>(up(scale.data(), sizeof(int) * scale.size()));
      a.buf = static_cast<double*>(up(nullptr, sizeof(double) * 2 * static_cast<size_t>(nchains) * Q * (d + 1)));
      a.row_off = static_cast<const int*>(up(row_off.data(), sizeof(int) * row_off.size()));
      a.row_chain = static_cast<const int*>(up(row_chain.data(), sizeof(int) * row_chain.size()));
      a.out = static_cast<double*>(up(nullptr, sizeof(double) * Q * (n + 1) * (d + 1)));
      const int threads = std::min(256, ((d + 1 + 31) / 32) * 32);
      pse::dispatch(m, mode == PSE_MODE_COMPLEX, a, nchains, n + 1, threads);
      pse::ck(cudaGetLastError(), "direct launch");
      pse::ck(cudaMemcpy(vg_out, a.out, sizeof(double) * Q * (n + 1) * (d + 1), cudaMemcpyDeviceToHost), "D2H");
    } catch (...) {
      for (void* p : owned) cudaFree(p);
      throw;
    }
    for (void* p : owned) cudaFree(p);
    return PSE_OK;
  } catch (const std::invalid_argument& e) {
    pse::set_error(e.what());
    return PSE_EINVAL;
  } catch (const std::exception& e) {
    pse::set_error(e.what());
    return PSE_ECUDA;
  }
}

}  // extern "C"
