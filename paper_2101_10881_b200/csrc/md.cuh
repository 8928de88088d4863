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
#include <utility>

namespace pse {

// compile-time loop: f(std::integral_constant<int, I>) for I = 0..N-1
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

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
// Every kernel that uses a lane runs kLaneThreads threads per block, so the
// row pitch is a compile-time constant and lane addresses are one 32-bit
// shared-memory register plus an immediate offset.
#ifndef PSE_LANE_THREADS
#define PSE_LANE_THREADS 128
#endif
constexpr int kLaneThreads = PSE_LANE_THREADS;
#ifndef PSE_PUSH_PRED
#define PSE_PUSH_PRED 1
#endif
constexpr unsigned kRow = kLaneThreads * sizeof(double);  // bytes between rows
#ifndef PSE_MERGE_RELOAD
#define PSE_MERGE_RELOAD 1
#endif
constexpr bool kMergeReload = PSE_MERGE_RELOAD;  // exp_add merge: heads re-read (else carried)

// A thread's private shared-memory lane: row r at byte address base + r*kRow.
struct Lane {
  unsigned base;
  unsigned step;  // kRow, held in a register (see make_lane)
};

// Row -1 (the first row of the allocation) is a spare: look-ahead loads may
// touch it harmlessly.
__device__ __forceinline__ Lane make_lane(double* smem) {
  // The row step comes from the block size (every lane kernel runs
  // kLaneThreads threads per block), so ptxas cannot turn it back into an
  // immediate: the predicated row advances (stack pushes, emissions, merge
  // pointers) then read it from one register instead of re-materialising
  // the constant before each of them.
  unsigned step;
  asm("{\n\t.reg .b32 n;\n\tmov.u32 n, %%ntid.x;\n\tshl.b32 %0, n, 3;\n\t}" : "=r"(step));
  return Lane{static_cast<unsigned>(__cvta_generic_to_shared(smem + kLaneThreads + threadIdx.x)), step};
}

// volatile: the stack's stores and loads must keep their program order
__device__ __forceinline__ void sts64(unsigned addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v));
}
__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
// static row offsets: the offset is an immediate of the instruction
template <int OFF>
__device__ __forceinline__ void sts64_at(unsigned base, double v) {
  asm volatile("st.shared.f64 [%0+%2], %1;" ::"r"(base), "d"(v), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ double lds64_at(unsigned base) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(base), "n"(OFF));
  return v;
}

// v = (lim >= THR) ? word at base+OFF : +0.0 -- predicated load, no selects
template <int OFF, unsigned THR>
__device__ __forceinline__ double lds64_at_if(unsigned base, unsigned lim) {
  double v;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ge.u32 p, %2, %3;\n\t"
      "mov.b64 %0, 0;\n\t"
      "@p ld.shared.f64 %0, [%1+%4];\n\t}"
      : "=d"(v)
      : "r"(base), "r"(lim), "n"(THR), "n"(OFF));
  return v;
}

// v != 0.0 (either sign) on the integer pipe: one LOP3 + one ISETP
__device__ __forceinline__ bool nonzero(double v) {
  return ((static_cast<unsigned>(__double2hiint(v)) & 0x7fffffffu) | static_cast<unsigned>(__double2loint(v))) != 0u;
}

// One vec_sum_err_branch step (expansion.hpp:80-87) against a shared-memory
// emission row: (r, tt) = fast_two_sum(eps, v); if tt != 0 (either sign) r is
// stored at row ea, ea moves one row (down when DOWN) and eps = tt, otherwise
// eps = r. In PTX so the store, the row advance and the eps select all hang
// off one predicate (LOP3.P, @P STS, @P IADD, 2 SEL).
// The row advance is `step` (a register: see make_lane) upward, or the
// immediate -kRow downward (ptxas emits a predicated VIADD for that one).
template <bool DOWN>
__device__ __forceinline__ void emit_step(double& eps, double v, unsigned& ea, unsigned step) {
  double r, tt;
  fast_two_sum(eps, v, r, tt);
  if constexpr (DOWN) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, t;\n\t"
        "mov.b64 {lo, hi}, %3;\n\t"
        "and.b32 t, hi, 0x7fffffff;\n\t"
        "or.b32 t, t, lo;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "@p st.shared.f64 [%1], %2;\n\t"
        "@p add.u32 %1, %1, %4;\n\t"
        "selp.f64 %0, %3, %2, p;\n\t}"
        : "=d"(eps), "+r"(ea)
        : "d"(r), "d"(tt), "n"(0u - kRow));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, t;\n\t"
        "mov.b64 {lo, hi}, %3;\n\t"
        "and.b32 t, hi, 0x7fffffff;\n\t"
        "or.b32 t, t, lo;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "@p st.shared.f64 [%1], %2;\n\t"
        "@p add.u32 %1, %1, %4;\n\t"
        "selp.f64 %0, %3, %2, p;\n\t}"
        : "=d"(eps), "+r"(ea)
        : "d"(r), "d"(tt), "r"(step));
  }
}

// bitwise inequality accumulator: d |= bits(a) ^ bits(b)
__device__ __forceinline__ unsigned diff_bits(double a, double b, unsigned d) {
  return d | (static_cast<unsigned>(__double2loint(a)) ^ static_cast<unsigned>(__double2loint(b))) |
         (static_cast<unsigned>(__double2hiint(a)) ^ static_cast<unsigned>(__double2hiint(b)));
}

// tighten (expansion.hpp:92-114). The reference writes (s, e) back only when
// a bit differs; writing unconditionally is the same, because equal bits
// leave the value unchanged. Only the "did anything change" flag needs the
// comparison, accumulated with XOR/OR on the integer pipe.
template <int M>
__device__ __forceinline__ unsigned tighten_pass(double (&w)[M]) {
  unsigned diff = 0;
#pragma unroll
  for (int i = 0; i + 1 < M; ++i) {
    double s, e;
    two_sum(w[i], w[i + 1], s, e);
    diff = diff_bits(s, w[i], diff_bits(e, w[i + 1], diff));
    w[i] = s;
    w[i + 1] = e;
  }
  return diff;
}

// True iff a tighten pass over w would change nothing. For finite a, the pair
// (a, b) is a fixed point of two_sum exactly when fl(a+b) == a bitwise and b
// is not -0: then bv = a - a = +0, s - bv = a and e = +0 + b = b (which is
// +0, not -0, when b = -0). The pairs are tested independently (one DADD
// each, no chain), and if all are fixed points the sequential pass is a no-op.
//
// Precondition (holds for every caller: tighten runs on the output of
// vec_sum_err_branch, and on its own output): no w[i], i >= 1, is -0.
//  * two_sum's error e = (a - av) + (b - bv) is never -0: both terms would
//    have to be -0, i.e. a = b = -0 and av = bv = +0, but then
//    av = s - bv = -0. So vec_sum tails and tighten's w[i+1] are never -0.
//  * err_branch emits r only when t != 0, and then r != 0; the final eps sits
//    at position >= 1 only after a step with a term that is nonzero (popped
//    stack terms) or not -0 (vec_sum tails), after which fl(eps + v) is not
//    -0. Padding is +0.
// So the "b is not -0" half of the test is vacuous here. Non-finite values:
// if w[0] is finite and some later w[i] is not, the first pair (finite a,
// non-finite b) has fl(a+b) non-finite != a and is caught by the bit test;
// so checking w[0] alone for inf/nan completes the test.
template <int M>
__device__ __forceinline__ bool tighten_fixed(const double (&w)[M]) {
  unsigned diff = 0;
#pragma unroll
  for (int i = 0; i + 1 < M; ++i) diff = diff_bits(__dadd_rn(w[i], w[i + 1]), w[i], diff);
  const unsigned ah = static_cast<unsigned>(__double2hiint(w[0]));
  return diff == 0u && (ah & 0x7ff00000u) != 0x7ff00000u;
}

// tighten (expansion.hpp:92-114): at most M passes, stop at the first pass
// that changes nothing. Testing "would the next pass change nothing"
// (tighten_fixed) replaces that final no-op pass -- 9 independent DADDs
// instead of 9 chained two_sums -- with identical results.
template <int M, bool PF>
__device__ __forceinline__ void tighten_fast(double (&w)[M]) {
  // PF: the first pass runs unconditionally. On a fixed point a pass changes
  // nothing (see tighten_fixed), so this only skips the first test; the
  // remaining M-1 passes keep the test -- same passes, same bits. It pays
  // where a warp nearly always has a lane that needs the pass: md_add
  // outputs (M = 2 / 3 / 10: 8 / 16 / 46% of them need one) and md_mul
  // outputs from M = 5 (M = 3 / 4 / 5 / 10: 0 / 5 / 9.5 / 29%;
  // tools/md_stats.c).
  if constexpr (PF) tighten_pass<M>(w);
#pragma unroll 1
  for (int pass = PF ? 1 : 0; pass < M; ++pass) {
    if (tighten_fixed<M>(w)) return;
    tighten_pass<M>(w);
  }
}

template <int M>
struct MdTraits {
  static constexpr int NT = M * (M + 1) + (M - 1);
  // Stack capacity for nonzero vec_sum pass-2 terms. The measured maximum over
  // 2e5 random full-precision pairs is 39 (M=10) and 31 (M=8), the 99th
  // percentile 31 and 24 (M=10 keeps 42 so four blocks of the convolution,
  // accumulator rows included, fit one SM's shared memory); small M reserve the full NT-1 so they never overflow.
  static constexpr int CAP = M == 10 ? 42 : M == 8 ? 40 : NT - 1;
  // rows per thread: the spare row -1, then CAP + one sacrificial row; the add
  // merge reads up to row 2M+2 (look-ahead past the y block)
  static constexpr int LANE = 1 + ((CAP + 1 > 2 * M + 3) ? CAP + 1 : 2 * M + 3);
  // the convolution's accumulator rows follow (acc_store / acc_add), plus
  // the row the merge's look-ahead reads past the accumulator. At M=10:
  // 55 rows x 128 threads x 8 B = 56,320 B per block, 4 blocks per SM.
  static constexpr int ACC = LANE - 1;
  static constexpr int LANE_CONV = LANE + M + 1;
};

// Merge, vec_sum, vec_sum_err_branch and tighten of an md_add
// (expansion.hpp:142-158) whose operands already sit in the thread's lane:
// x at rows XR..XR+M-1, y at rows YR..YR+M-1, heads (and, for LAT, the
// second elements) passed in registers. Emissions use rows 0..2M-1, so x or
// y rows below 2M are consumed before they are overwritten. Without LAT the
// merge needs sentinels in rows XR+M (NaN) and YR+M (+0).
// LAT = latency-optimised merge (for latency-bound callers such as the split
// path's accumulation chains): each side's head AND next element live in
// registers, so the shared-memory refill is not on the compare chain. The
// default keeps only the heads (fewer instructions, for throughput-bound
// callers). Both produce the same merged sequence.
template <int M, bool LAT, int XR, int YR>
__device__ __forceinline__ void exp_add_core(double xh, double xn, double yh, double yn, double (&out)[M], Lane ln) {
  // merge by magnitude, ties take x (expansion.hpp:150-153)
  double t[2 * M];
  [[maybe_unused]] int i = 0;  // LAT: x elements taken; y taken = p - i
  if constexpr (!LAT) {
    // Sentinels end both runs: NaN after x (|NaN| >= |y| is false, so an
    // exhausted x never wins) and +0 after y (|x| >= 0 holds for every
    // non-NaN x, so an exhausted y never wins). Both cannot be exhausted
    // within 2M steps, so the comparison alone replays the reference's
    // merge and tail copies. (NaN data is outside the bit-exact contract:
    // NaN bit patterns already differ between the host and the device.)
    if constexpr (kMergeReload) {
      // both heads re-read from the lane after every step (one of the two
      // loads is redundant): fewer selects than carrying them in registers
      // (C2 -1.6% in tools/step_bench.cu)
      unsigned xa = ln.base + XR * kRow, ya = ln.base + YR * kRow;
#pragma unroll
      for (int p = 0; p < 2 * M; ++p) {
        const bool take_x = fabs(xh) >= fabs(yh);
        t[p] = take_x ? xh : yh;
        if (p + 1 < 2 * M) {
          // one predicated add per pointer (a select would cost two)
          asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
              "@p add.u32 %0, %0, %3;\n\t@!p add.u32 %1, %1, %3;\n\t}"
              : "+r"(xa), "+r"(ya)
              : "r"(static_cast<unsigned>(take_x)), "r"(ln.step));
          xh = lds64(xa);
          yh = lds64(ya);
        }
      }
    } else {
      unsigned xa = ln.base + (XR + 1) * kRow, ya = ln.base + (YR + 1) * kRow;
#pragma unroll
      for (int p = 0; p < 2 * M; ++p) {
        const bool take_x = fabs(xh) >= fabs(yh);
        t[p] = take_x ? xh : yh;
        if (p + 1 < 2 * M) {
          const double v = lds64(take_x ? xa : ya);
          xh = take_x ? v : xh;
          yh = take_x ? yh : v;
          xa += take_x ? kRow : 0u;
          ya += take_x ? 0u : kRow;
        }
      }
    }
  } else {
    unsigned xa = ln.base + (XR + 2) * kRow, ya = ln.base + (YR + 2) * kRow;
#pragma unroll
    for (int p = 0; p < 2 * M; ++p) {
      const bool take_x = (p - i >= M) || (i < M && fabs(xh) >= fabs(yh));
      t[p] = take_x ? xh : yh;
      if (p + 1 < 2 * M) {
        const double v = lds64(take_x ? xa : ya);  // element after next
        xh = take_x ? xn : xh;
        yh = take_x ? yh : yn;
        xn = take_x ? v : xn;
        yn = take_x ? yn : v;
        xa += take_x ? kRow : 0u;
        ya += take_x ? 0u : kRow;
        i += take_x ? 1 : 0;
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
  // vec_sum_err_branch (expansion.hpp:74-90); emission jj goes to row jj.
  // The reference stops at the M-th emission; running on is harmless here
  // because later emissions land in rows >= M, which are never read, and
  // eps is only used when fewer than M were emitted -- so no per-step guard.
  unsigned ea = ln.base;
  double eps = t[0];
#pragma unroll
  for (int q = 1; q < 2 * M; ++q) emit_step<false>(eps, t[q], ea, ln.step);
  // rows 0..jj-1 hold the emissions; eps goes to row jj (when jj >= M it is
  // never read) and rows beyond jj read as zero
  sts64(ea, eps);
  const unsigned jb = ea - ln.base;
  static_for<M>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    out[q] = lds64_at_if<q * kRow, q * kRow>(ln.base, jb);
  });
  tighten_fast<M, true>(out);
}

// out = x + y (expansion.hpp:142-158), operands in registers. Safe for out
// aliasing x or y.
template <int M, bool LAT = false>
__device__ __forceinline__ void exp_add_fast(const double (&x)[M], const double (&y)[M], double (&out)[M], Lane ln) {
  if constexpr (M == 1) {
    out[0] = __dadd_rn(x[0], y[0]);
  } else {
#pragma unroll
    // x at rows 0..M-1 + NaN sentinel at row M, y at rows M+1..2M + zero
    // sentinel at row 2M+1 (the LAT merge ignores the sentinels)
    static_for<M>([&](auto q) {
      sts64_at<decltype(q)::value * kRow>(ln.base, x[decltype(q)::value]);
      sts64_at<(M + 1 + decltype(q)::value) * kRow>(ln.base, y[decltype(q)::value]);
    });
    if constexpr (!LAT) {
      sts64_at<M * kRow>(ln.base, __longlong_as_double(0x7ff8000000000000ll));
      sts64_at<(2 * M + 1) * kRow>(ln.base, 0.0);
    }
    exp_add_core<M, LAT, 0, M + 1>(x[0], x[1], y[0], y[1], out, ln);
  }
}

// Accumulator kept in the lane (rows MdTraits<M>::ACC..ACC+M-1) instead of
// registers, so it is not live across the register-hungry md_mul between
// two accumulation steps.
template <int M>
__device__ __forceinline__ void acc_store(const double (&v)[M], Lane ln);
template <int M>
__device__ __forceinline__ void acc_add(const double (&y)[M], double (&out)[M], Lane ln);

template <int M>
__device__ __forceinline__ void exp_sub_fast(const double (&x)[M], const double (&y)[M], double (&out)[M], Lane ln) {
  if constexpr (M == 1) {
    out[0] = __dsub_rn(x[0], y[0]);
  } else {
    double ny[M];
#pragma unroll
    for (int q = 0; q < M; ++q) ny[q] = -y[q];
    exp_add_fast<M>(x, ny, out, ln);
  }
}

namespace detail {

// Streaming state of the two backward vec_sum passes and the compacted
// stack of nonzero pass-2 outputs (top = byte address of the next free row).
struct Passes {
  double s1, s2;
  unsigned top;
  unsigned step;  // kRow, held in a register (see push)
};

// push v if nonzero; `clamp` (pushes beyond the first CAP) redirects the
// store to the sacrificial row lim once the stack is full -- overflow is then
// detected from the count and handled by the literal slow path
template <bool CLAMP>
__device__ __forceinline__ void push(Passes& st, double v, unsigned lim) {
  // store, then advance top by one row iff v != 0 (either sign): written in
  // PTX so ptxas emits a predicated add (STS + LOP3.P + @P IADD)
  const unsigned addr = CLAMP ? min(st.top, lim) : st.top;
#if PSE_PUSH_PRED
  // only nonzero terms are stored (about a quarter of them at M = 10): less
  // shared-memory traffic, the store waiting on the zero test (C3' 25.70 ->
  // 25.31 ms, C2 32.85 -> 32.67)
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, t;\n\t"
      "mov.b64 {lo, hi}, %2;\n\t"
      "and.b32 t, hi, 0x7fffffff;\n\t"
      "or.b32 t, t, lo;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "@p st.shared.f64 [%1], %2;\n\t"
      "@p add.u32 %0, %0, %3;\n\t}"
      : "+r"(st.top)
      : "r"(addr), "d"(v), "r"(st.step));
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, t;\n\t"
      "st.shared.f64 [%1], %2;\n\t"
      "mov.b64 {lo, hi}, %2;\n\t"
      "and.b32 t, hi, 0x7fffffff;\n\t"
      "or.b32 t, t, lo;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "@p add.u32 %0, %0, %3;\n\t}"
      : "+r"(st.top)
      : "r"(addr), "d"(v), "n"(kRow));
#endif
}

// pass-1 step on term t (terms arrive t[n-2], t[n-3], ..., t[0]) followed by
// the pass-2 step on the error it produces (x1 arrives x1[n-1], x1[n-2], ...)
template <bool CLAMP>
__device__ __forceinline__ void feed(Passes& st, double t, unsigned lim) {
  double e1, e2;
  two_sum(t, st.s1, st.s1, e1);
  two_sum(e1, st.s2, st.s2, e2);
  push<CLAMP>(st, e2, lim);
}

}  // namespace detail

// out = x * y (expansion.hpp:177-211), register-streamed; see file header.
template <int M>
__device__ __forceinline__ void exp_mul_fast(const double (&x)[M], const double (&y)[M], double (&out)[M], Lane ln) {
  if constexpr (M == 1) {
    out[0] = __dmul_rn(x[0], y[0]);
  } else {
    constexpr int CAP = MdTraits<M>::CAP;
    const unsigned lim = ln.base + CAP * kRow;
    detail::Passes st;
    st.top = ln.base;
    st.step = ln.step;  // see make_lane (-70 instructions per md_mul at M = 10)
    // Pass 2 runs one term behind pass 1: the pass-1 error of term i is
    // consumed by pass 2 while pass 1 processes term i+1, so the two
    // two_sums of a step are independent and interleave (ILP 2). The
    // sequence of operations on each pass is unchanged.
    int fed = 0;      // compile-time after unrolling
    int pushes = 0;
    double e1p = 0.0; // pending pass-1 error (next pass-2 input)
    auto feed = [&](double t) {
      if (fed == 0) {
        st.s1 = t;  // t[NT-1] seeds pass 1
      } else if (fed == 1) {
        two_sum(t, st.s1, st.s1, st.s2);  // x1[NT-1] seeds pass 2
      } else if (fed == 2) {
        two_sum(t, st.s1, st.s1, e1p);
      } else {
        double e1, e2;
        two_sum(t, st.s1, st.s1, e1);
        two_sum(e1p, st.s2, st.s2, e2);
        if (pushes < CAP)
          detail::push<false>(st, e2, lim);
        else
          detail::push<true>(st, e2, lim);
        ++pushes;
        e1p = e1;
      }
      ++fed;
    };
    // Reverse term order: section k (k = M..1) = [errors of diagonal k-1,
    // reversed] then [products of diagonal k, reversed]; finally diagonal 0.
    // One diagonal of products is held while the next diagonal's errors are
    // fed.
    double pr[M];
    {
      double er[M];
#pragma unroll
      for (int i = 0; i < M; ++i) two_prod(x[i], y[M - 1 - i], pr[i], er[i]);
#pragma unroll
      for (int i = M - 1; i >= 0; --i) feed(er[i]);
    }
    // diagonal M: plain products (expansion.hpp:197-200)
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
    feed(pr[0]);  // t[0]
    {             // drain pass 2: x1[1] (pending), then x1[0] = the pass-1 sum
      double e;
      two_sum(e1p, st.s2, st.s2, e);
      detail::push<true>(st, e, lim);
      two_sum(st.s1, st.s2, st.s2, e);
      detail::push<true>(st, e, lim);
    }
    // st.s2 = x2[0]; rows [0, count) hold the nonzero x2[NT-1..1], x2[1] on top
    const int count = static_cast<int>((st.top - ln.base) / kRow);
    if (count <= CAP) {
      // vec_sum_err_branch over the compacted terms (popped top-down, one
      // row of look-ahead); emission jj overwrites row count-1-jj, which has
      // already been consumed. Two pops per trip; the emission count is
      // tested once per trip, so a trip may pop one term after the M-th
      // emission (where the reference returns): that emission lands in a
      // row that is never read and eps is then unused. The look-ahead load
      // may read the spare row -1, never below.
      double eps = st.s2;
      unsigned a = st.top - kRow;        // row of the next term to pop
      unsigned ea = st.top - kRow;       // row of the next emission
      // ea <= elim <=> M emitted. Signed: with fewer than M+1 terms on the
      // stack elim lies below the lane and, near the bottom of the shared
      // window, below address 0 (as an unsigned bound it wrapped, and the
      // loop popped nothing: x*1 lost every limb but the first).
      const int elim = static_cast<int>(st.top) - (M + 1) * static_cast<int>(kRow);
      const unsigned base1 = ln.base + kRow;
      double n0 = lds64(a);
#pragma unroll 1
      while (a >= ln.base && static_cast<int>(ea) > elim) {
        const double n1 = lds64_at<-static_cast<int>(kRow)>(a);  // row a-1 >= spare row
        emit_step<true>(eps, n0, ea, ln.step);
        if (a < base1) break;
        n0 = lds64_at<-2 * static_cast<int>(kRow)>(a);  // row a-2 >= spare row (a-1 >= base)
        emit_step<true>(eps, n1, ea, ln.step);
        a -= 2 * kRow;
      }
      // emission k sits at row top-1-k; eps goes to the next emission row
      // (at most M+1 and at most `count` emissions: ea >= the spare row -1)
      sts64(ea, eps);
      const unsigned jb = st.top - kRow - ea;  // jj rows, in bytes
      static_for<M>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        out[k] = lds64_at_if<-(k + 1) * static_cast<int>(kRow), k * kRow>(st.top, jb);
      });
      tighten_fast<M, (M >= 5)>(out);
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

// once per thread before the first acc_add: the NaN sentinel after the
// accumulator rows (never overwritten: acc_store writes rows ACC..ACC+M-1)
template <int M>
__device__ __forceinline__ void acc_init(Lane ln) {
  sts64_at<(MdTraits<M>::ACC + M) * kRow>(ln.base, __longlong_as_double(0x7ff8000000000000ll));
}

template <int M>
__device__ __forceinline__ void acc_store(const double (&v)[M], Lane ln) {
  static_for<M>([&](auto q) {
    sts64_at<(MdTraits<M>::ACC + decltype(q)::value) * kRow>(ln.base, v[decltype(q)::value]);
  });
}

// out = acc + y (expansion.hpp:142-158, x = the accumulator), then acc = out
template <int M>
__device__ __forceinline__ void acc_add(const double (&y)[M], double (&out)[M], Lane ln) {
  if constexpr (M == 1) {
    out[0] = __dadd_rn(lds64_at<MdTraits<M>::ACC * kRow>(ln.base), y[0]);
  } else {
    static_for<M>([&](auto q) { sts64_at<(M + decltype(q)::value) * kRow>(ln.base, y[decltype(q)::value]); });
    sts64_at<2 * M * kRow>(ln.base, 0.0);  // y's sentinel (x's: acc_init)
    const double xh = lds64_at<MdTraits<M>::ACC * kRow>(ln.base);
    exp_add_core<M, false, MdTraits<M>::ACC, M>(xh, 0.0, y[0], 0.0, out, ln);
  }
  acc_store<M>(out, ln);
}

}  // namespace pse
