// Device multiple-double (expansion) arithmetic for sm_100a -- bit-exact with
// the reference CPU library proj/include/pseval/expansion.hpp:31-211.
//
// Every +, -, * is an explicit round-to-nearest intrinsic (__dadd_rn,
// __dsub_rn, __dmul_rn, __fma_rn), so nvcc can never contract them; this
// plays the role of the reference's -ffp-contract=off (CMakeLists.txt:12-15).
//
// Two implementations of each operation live here:
//   *_lit  literal restatements of the reference loops over local arrays;
//          used by the md unit kernel and as the exact slow path;
//   *_fast register-streamed versions used by the convolution engine:
//     exp_mul: the NT = M(M+1)+(M-1) term array is never materialised. The
//       terms are regenerated in reverse order (diagonal by diagonal) and
//       fed straight into vec_sum pass 1, whose outputs feed pass 2 one step
//       behind (both passes run backward, expansion.hpp:61-69). Only the
//       NONZERO pass-2 outputs are pushed to a per-thread shared-memory
//       stack; vec_sum_err_branch (expansion.hpp:74-90) pops it forward.
//       Exact zeros are no-ops in vec_sum_err_branch except that a +0 turns
//       a running -0 into +0, which can only happen when every term is zero,
//       and tighten() maps [-0, +0, ...] to +0 anyway (M >= 2) -- so the
//       compaction is bit-exact. If a thread ever has more than CAP nonzero
//       terms it recomputes the product with the literal algorithm.
//     exp_add: the magnitude merge (expansion.hpp:150-153) needs dynamic
//       indices, so x and y are staged in the thread's shared-memory lane;
//       the 2M merged terms live in registers.
//
// Shared-memory lanes use an [index][thread] layout: word i of thread t is at
// base[i * blockDim + t], so lanes of a warp never bank-conflict whatever
// index each of them uses.
#pragma once

#include <cstdint>

namespace pse {

// ---------------------------------------------------------------- EFTs
// two_sum: expansion.hpp:31-38 (Knuth, branch-free, 6 flops)
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  const double ss = __dadd_rn(a, b);
  const double bv = __dsub_rn(ss, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(ss, bv)), __dsub_rn(b, bv));
  s = ss;
}

// fast_two_sum: expansion.hpp:40-46
__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
  const double ss = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(ss, a));
  s = ss;
}

// two_prod: expansion.hpp:48-55 (DMUL + DFMA)
__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  const double pp = __dmul_rn(a, b);
  e = __fma_rn(a, b, -pp);
  p = pp;
}

__device__ __forceinline__ bool bits_differ(double a, double b) {
  return __double_as_longlong(a) != __double_as_longlong(b);
}

// ------------------------------------------------------------- literal
__device__ __forceinline__ void vec_sum_lit(double* x, int n) {
  double s = x[n - 1];
  for (int i = n - 2; i >= 0; --i) {
    double e;
    two_sum(x[i], s, s, e);
    x[i + 1] = e;
  }
  x[0] = s;
}

__device__ __forceinline__ void vec_sum_err_branch_lit(const double* e, int n, double* out, int m) {
  int j = 0;
  double eps = e[0];
  for (int i = 1; i < n; ++i) {
    double r, t;
    fast_two_sum(eps, e[i], r, t);
    if (t != 0.0) {
      out[j++] = r;
      if (j == m) return;
      eps = t;
    } else {
      eps = r;
    }
  }
  out[j++] = eps;
  while (j < m) out[j++] = 0.0;
}

// tighten: expansion.hpp:92-114 (register array, static indices)
template <int M>
__device__ __forceinline__ void tighten(double (&w)[M]) {
#pragma unroll 1
  for (int pass = 0; pass < M; ++pass) {
    bool changed = false;
#pragma unroll
    for (int i = 0; i + 1 < M; ++i) {
      double s, e;
      two_sum(w[i], w[i + 1], s, e);
      if (bits_differ(s, w[i]) || bits_differ(e, w[i + 1])) {
        w[i] = s;
        w[i + 1] = e;
        changed = true;
      }
    }
    if (!changed) break;
  }
}

__device__ __forceinline__ void tighten_lit(double* w, int m) {
  for (int pass = 0; pass < m; ++pass) {
    bool changed = false;
    for (int i = 0; i + 1 < m; ++i) {
      double s, e;
      two_sum(w[i], w[i + 1], s, e);
      if (bits_differ(s, w[i]) || bits_differ(e, w[i + 1])) {
        w[i] = s;
        w[i + 1] = e;
        changed = true;
      }
    }
    if (!changed) return;
  }
}

// exp_add literal: expansion.hpp:142-158
template <int M>
__device__ __noinline__ void exp_add_lit(const double* x, const double* y, double* out) {
  if constexpr (M == 1) {
    out[0] = __dadd_rn(x[0], y[0]);
  } else {
    double t[2 * M];
    int i = 0, j = 0, p = 0;
    while (i < M && j < M) t[p++] = fabs(x[i]) >= fabs(y[j]) ? x[i++] : y[j++];
    while (i < M) t[p++] = x[i++];
    while (j < M) t[p++] = y[j++];
    vec_sum_lit(t, 2 * M);
    vec_sum_err_branch_lit(t, 2 * M, out, M);
    tighten_lit(out, M);
  }
}

// exp_mul literal: expansion.hpp:177-211
template <int M>
__device__ __noinline__ void exp_mul_lit(const double* x, const double* y, double* out) {
  if constexpr (M == 1) {
    out[0] = __dmul_rn(x[0], y[0]);
  } else {
    constexpr int NT = M * (M + 1) + (M - 1);
    double t[NT];
    double carry[M], next[M];
    int pos = 0, ncarry = 0;
    for (int k = 0; k <= M; ++k) {
      int nn = 0;
      const int ilo = k - (M - 1) > 0 ? k - (M - 1) : 0;
      const int ihi = k < M - 1 ? k : M - 1;
      for (int i = ilo; i <= ihi; ++i) {
        if (k < M) {
          double pr, er;
          two_prod(x[i], y[k - i], pr, er);
          t[pos++] = pr;
          next[nn++] = er;
        } else {
          t[pos++] = __dmul_rn(x[i], y[k - i]);
        }
      }
      for (int c = 0; c < ncarry; ++c) t[pos++] = carry[c];
      for (int c = 0; c < nn; ++c) carry[c] = next[c];
      ncarry = nn;
    }
    vec_sum_lit(t, NT);
    vec_sum_lit(t, NT);
    vec_sum_err_branch_lit(t, NT, out, M);
    tighten_lit(out, M);
  }
}

// ---------------------------------------------------------------- fast
// A thread's private shared-memory lane, [index][thread] layout.
struct Lane {
  double* p;
  int stride;
  __device__ __forceinline__ double& operator[](int i) const { return p[i * stride]; }
};

template <int M>
struct MdTraits {
  static constexpr int NT = M * (M + 1) + (M - 1);
  // stack capacity for nonzero vec_sum pass-2 terms; the measured maximum
  // over 2e5 random full-precision pairs is 39 (M=10) and 31 (M=8); small M
  // reserve the full NT-1 so they can never overflow
  static constexpr int CAP = M == 10 ? 48 : M == 8 ? 40 : (NT - 1 > 2 * M + 1 ? NT - 1 : 2 * M + 1);
  // words per thread in the shared-memory lane (add merge needs 2M + 1)
  static constexpr int LANE = CAP > 2 * M + 1 ? CAP : 2 * M + 1;
};

// out = x + y. Safe for out aliasing x or y (all reads precede writes).
template <int M>
__device__ __forceinline__ void exp_add_fast(const double (&x)[M], const double (&y)[M], double (&out)[M],
                                             Lane sm) {
  if constexpr (M == 1) {
    out[0] = __dadd_rn(x[0], y[0]);
  } else {
#pragma unroll
    for (int q = 0; q < M; ++q) {
      sm[q] = x[q];
      sm[M + q] = y[q];
    }
    // merge by magnitude, ties take x (expansion.hpp:150-153)
    double t[2 * M];
    int i = 0, j = 0;
    double xh = x[0], yh = y[0];
#pragma unroll
    for (int p = 0; p < 2 * M; ++p) {
      const bool take_x = (j >= M) || (i < M && fabs(xh) >= fabs(yh));
      t[p] = take_x ? xh : yh;
      if (p + 1 < 2 * M) {
        const int ni = take_x ? i + 1 : M + j + 1;  // index 2M is a readable spare word
        const double v = sm[ni];
        if (take_x) {
          xh = v;
          ++i;
        } else {
          yh = v;
          ++j;
        }
      }
    }
    // vec_sum over 2M (expansion.hpp:61-69)
    double s = t[2 * M - 1];
#pragma unroll
    for (int q = 2 * M - 2; q >= 0; --q) {
      double e;
      two_sum(t[q], s, s, e);
      t[q + 1] = e;
    }
    t[0] = s;
    // vec_sum_err_branch (expansion.hpp:74-90); emissions go to the lane
    int jj = 0;
    double eps = t[0];
    bool done = false;
#pragma unroll
    for (int q = 1; q < 2 * M; ++q) {
      if (!done) {
        double r, tt;
        fast_two_sum(eps, t[q], r, tt);
        if (tt != 0.0) {
          sm[jj] = r;
          ++jj;
          if (jj == M) done = true;
          eps = tt;
        } else {
          eps = r;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < M; ++q) {
      const double v = sm[q];
      out[q] = q < jj ? v : (q == jj ? eps : 0.0);
    }
    tighten<M>(out);
  }
}

template <int M>
__device__ __forceinline__ void exp_sub_fast(const double (&x)[M], const double (&y)[M], double (&out)[M],
                                             Lane sm) {
  if constexpr (M == 1) {
    out[0] = __dsub_rn(x[0], y[0]);
  } else {
    double ny[M];
#pragma unroll
    for (int q = 0; q < M; ++q) ny[q] = -y[q];
    exp_add_fast<M>(x, ny, out, sm);
  }
}

namespace detail {

// streaming state of the two backward vec_sum passes
struct Passes {
  double s1, s2;
  int sp;
  bool ovf;
};

template <int CAP>
__device__ __forceinline__ void push_nonzero(Passes& st, double v, Lane sm) {
  if (v != 0.0) {
    if (st.sp < CAP)
      sm[st.sp] = v;
    else
      st.ovf = true;
    ++st.sp;
  }
}

// pass-2 step on x1 value v (x1 arrives x1[n-1], x1[n-2], ...)
template <int CAP>
__device__ __forceinline__ void feed2(Passes& st, double v, Lane sm) {
  double e;
  two_sum(v, st.s2, st.s2, e);
  push_nonzero<CAP>(st, e, sm);
}

// pass-1 step on term t (terms arrive t[n-2], t[n-3], ..., t[0])
template <int CAP>
__device__ __forceinline__ void feed(Passes& st, double t, Lane sm) {
  double e;
  two_sum(t, st.s1, st.s1, e);
  feed2<CAP>(st, e, sm);
}

}  // namespace detail

// out = x * y (expansion.hpp:177-211), register-streamed; see file header.
// Safe for out aliasing x or y only if the caller copies first (x, y are read
// until the end of term generation).
template <int M>
__device__ __forceinline__ void exp_mul_fast(const double (&x)[M], const double (&y)[M], double (&out)[M],
                                             Lane sm) {
  if constexpr (M == 1) {
    out[0] = __dmul_rn(x[0], y[0]);
  } else {
    constexpr int CAP = MdTraits<M>::CAP;
    detail::Passes st;
    st.sp = 0;
    st.ovf = false;
    // Reverse term order: section k (k = M..1) = [errors of diagonal k-1,
    // reversed] then [products of diagonal k, reversed]; finally diagonal 0.
    double pr[M];
    {
      double er[M];
#pragma unroll
      for (int i = 0; i < M; ++i) two_prod(x[i], y[M - 1 - i], pr[i], er[i]);
      st.s1 = er[M - 1];  // t[NT-1] seeds pass 1
      double e;
      two_sum(er[M - 2], st.s1, st.s1, e);
      st.s2 = e;  // x1[NT-1] seeds pass 2
#pragma unroll
      for (int i = M - 3; i >= 0; --i) detail::feed<CAP>(st, er[i], sm);
    }
    // diagonal M: plain products (expansion.hpp:197-200)
#pragma unroll
    for (int i = M - 1; i >= 1; --i) detail::feed<CAP>(st, __dmul_rn(x[i], y[M - i]), sm);
#pragma unroll
    for (int k = M - 1; k >= 1; --k) {
      double pn[M], en[M];
#pragma unroll
      for (int i = 0; i < k; ++i) two_prod(x[i], y[k - 1 - i], pn[i], en[i]);
#pragma unroll
      for (int i = k - 1; i >= 0; --i) detail::feed<CAP>(st, en[i], sm);
#pragma unroll
      for (int i = k; i >= 0; --i) detail::feed<CAP>(st, pr[i], sm);
#pragma unroll
      for (int i = 0; i < k; ++i) pr[i] = pn[i];
    }
    detail::feed<CAP>(st, pr[0], sm);  // t[0]
    detail::feed2<CAP>(st, st.s1, sm); // x1[0] = pass-1 sum
    // st.s2 = x2[0]; stack holds nonzero x2[NT-1..1], top = x2[1]
    int jj = 0;
    double eps = st.s2;
    if (!st.ovf) {
      // vec_sum_err_branch over the compacted terms; emission jj is written
      // into a stack word that has already been popped
      int q = st.sp - 1;
      while (q >= 0) {
        const double v = sm[q];
        double r, tt;
        fast_two_sum(eps, v, r, tt);
        if (tt != 0.0) {
          sm[st.sp - 1 - jj] = r;
          ++jj;
          if (jj == M) break;
          eps = tt;
        } else {
          eps = r;
        }
        --q;
      }
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double v = sm[st.sp - 1 - k < 0 ? 0 : st.sp - 1 - k];
        out[k] = k < jj ? v : (k == jj ? eps : 0.0);
      }
      tighten<M>(out);
    } else {
      // rare: more nonzero terms than the lane holds -> literal algorithm
      double xl[M], yl[M], ol[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        xl[k] = x[k];
        yl[k] = y[k];
      }
      exp_mul_lit<M>(xl, yl, ol);
#pragma unroll
      for (int k = 0; k < M; ++k) out[k] = ol[k];
    }
  }
}

}  // namespace pse
