// Device kernels of the evaluate-and-differentiate engine, templated on the
// limb count M (1,2,3,4,5,8,10) and complex mode. Instantiated once per M in
// kernels_m<M>.cu so the heavy M=8/10 bodies compile in parallel.
//
// Arena layout in HBM (one per evaluation point):
//   arena[point][slot][q][S],  q = part*M + limb, S = (d+1) rounded up to 4
// i.e. a slot's series is one contiguous, limb-split structure of arrays:
// lanes that own consecutive coefficients load consecutive doubles of the
// same limb (coalesced), and a whole slot is a single 32B-aligned span.
#pragma once

#include <cstdint>
#include <cstdlib>

#include <cuda_runtime.h>

#include "md.cuh"

namespace pse {

struct Geom {
  int d;              // truncation degree
  int S;              // padded coefficient stride
  int Q;              // slabs per slot (P * M)
  int64_t slot_words; // Q * S
  int64_t point_words;// device slots * Q * S
};

// Phase stamps (RunReport per-layer times, executor.hpp:31-43): kernels
// record %globaltimer into a per-plan array with atomics -- a phase's start as
// atomicMax of the inverted time (so one zero-fill resets every slot), its end
// as atomicMax of the time -- see Plan::read_stamps in engine.cu.
using Stamp = unsigned long long;
__device__ __forceinline__ Stamp global_ns() {
  Stamp t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// one atomic per block at entry: the phase cannot start before this
__device__ __forceinline__ void stamp_begin(Stamp* s) {
  if (s && threadIdx.x == 0) atomicMax(s, ~global_ns());
}
// one atomic per converged group of lanes on the way out
__device__ __forceinline__ void stamp_finish(Stamp* s) {
  if (s) {
    const unsigned mask = __activemask();
    if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(mask) - 1)) atomicMax(s, global_ns());
  }
}

struct ConvArgs {
  double* arena;
  Geom G;
  const int4* jobs;  // (in1, in2, out, copy) of one conv layer
  int njobs;
  int npairs;        // coefficient pairs per job: (d+2)/2
  int batch;
  Stamp* t_begin;    // conv stage start (inverted), or null
  Stamp* t_end;      // this layer's end, or null
};

struct AddArgs {
  double* arena;
  Geom G;
  const int2* jobs;  // (src, dst): dst := dst + src
  int njobs;
  int batch;
  Stamp* t_begin;    // tail start (inverted), or null
  Stamp* t_end;
};

struct ScaleArgs {
  double* arena;
  Geom G;
  const int2* items;  // (slot, factor) -- factors are small exact integers
  int nitems;
  int batch;
  Stamp* t_begin;
  Stamp* t_end;
};

struct ExtractArgs {
  const double* arena;
  Geom G;
  const int* row_slot;   // [nrows] slot or -1 (zero series)
  const int* row_mult;   // [nrows] integer multiplier
  int nrows;
  int batch;
  double* out;           // [Q][batch][nrows][d+1]
  Stamp* t_begin;
  Stamp* t_end;
};

struct MdArgs {
  int op;    // 0 add, 1 sub, 2 mul
  int impl;  // 0 fast (engine path), 1 literal
  int64_t count;
  const double* x;  // [count][M]
  const double* y;
  double* out;
};

// Split convolution for layers too small to fill the GPU with one thread per
// coefficient pair: every product x_i*y_{k-i} of the layer is computed
// independently (conv_prod), then each coefficient's ascending-i md_add chain
// runs over the stored products (conv_accum). The operation order of conv()
// is unchanged, so the result is bit-identical to the fused kernel.
struct SplitArgs {
  double* arena;
  Geom G;
  const int4* jobs;
  int njobs;
  int batch;
  double* prod;          // scratch: [point][job][T][Q], T = (d+1)(d+2)/2
  const int2* tri;       // [T] (k, i) of triangular product index k(k+1)/2 + i
  int T;
  Stamp* t_begin;
  Stamp* t_end;
};

// Banded convolution (deep graphs, few jobs per layer). A conv job's output
// coefficients are cut into bands of width W (16 or 32) -- band 0 = [0, W0)
// with W0 = d % W + 1, then full bands, so that every rectangular task has W
// busy lanes -- and the accumulation chain of a coefficient k (steps
// i = 0..k, ascending) into segments at the same boundaries.
// A task (job, band b, segment s <= b) runs the steps i in segment s of the
// chains of every k in band b; the running sum is carried between segments
// in the output slot itself (exact binary64 words), so the operation order of
// conv() is unchanged and the result is bit-identical. A task needs only
// band s of in1 and bands <= b-s of in2, so a job's low bands finish -- and
// unlock the next layer -- while its high bands still accumulate: the host
// schedules tasks over that dependency graph.
// A warp descriptor is kSlots int4 slots of 8 lanes each; a task fills W/8
// (rectangular, copy) or W/16 (diagonal) aligned slots, each holding the
// task as {job, k0 = first coefficient of the band, i0 = first step, kind}:
//   kind -1  rectangular task (s < b): lane t of the task owns k = k0 + t,
//            the steps i of segment s (all < k0 <= k);
//   kind -2  diagonal task (s == b), W/2 lanes: lane j owns k = k0+j and
//            k = k0+width-1-j, steps k0..k -- width+1 steps per lane;
//   kind -3  copy job, band k0: out := in1 on coefficients k0 + t;
//   kind -4  empty slot.
constexpr int kBandW = 32;  // widest band
constexpr int kSlots = 4;   // 8-lane slots per warp descriptor

struct BandArgs {
  double* arena;
  Geom G;
  const int4* jobs;   // (in1, in2, out, flags) of every banded conv job;
                      // flags: 2 = in1 and 4 = in2 produced by a conv job,
                      // bits 8+ = the job's graph conv layer
  const int4* tasks;  // kSlots slots per warp descriptor, one wave
  int ntasks;         // warp descriptors
  int batch;
  int W;              // band width
  Stamp* stamps;      // [0] conv start (inverted), [1 + layer] layer ends; or null
};

struct FlowArgs {
  double* arena;
  Geom G;
  const int4* jobs;     // as BandArgs
  const int4* tasks;    // kSlots slots per warp descriptor, in scheduled order
  const int* dep_off;   // [nunits+1] CSR of the descriptors each one waits for
  const int* deps;
  int nunits;
  int batch;
  unsigned* flags;      // [batch][nunits], zero before the launch
  unsigned long long* counter;  // zero before the launch
  int W;                // band width
  Stamp* stamps;        // as BandArgs
};

// CTA-local dataflow (deep graphs at small precisions, where the global
// dataflow kernel's per-task hand-out and flag round trips through L2 dwarf a
// task's arithmetic): ONE block per independent job group (whole monomials)
// and point, its warps taking the group's band x segment tasks from a
// shared-memory counter in scheduled order and waiting on shared-memory
// completion flags -- a CTA-scope fence instead of a GPU-scope one, a
// shared-memory poll instead of an L2 round trip.
struct CtaArgs {
  double* arena;
  Geom G;
  const int4* jobs;      // as BandArgs (every job of every group)
  const int4* tasks;     // kSlots slots per warp descriptor, groups one after another
  const int* group_off;  // [ngroups+1] first descriptor of each group
  const int* dep_off;    // [ndesc+1] CSR of the descriptors each one waits for,
  const int* deps;       //   as indices local to the group
  int ngroups;
  int batch;
  int W;
  Stamp* stamps;         // as BandArgs
};

// CTA-local layered convolution (deep graphs of few large job groups at small
// precisions): ONE block per independent job group and point runs the
// group's conv layers in order, a block barrier between layers -- no task
// hand-out, no completion flags. At M >= 2 (only when forced) every thread
// takes whole coefficient pairs (k, d-k) of the layer's jobs, as k_conv
// does, reading operands this block wrote earlier through L1; at M = 1 (the
// default there) the operands are staged in shared memory and every thread
// runs a register block of adjacent chains (ctl_group_m1). A layer's
// critical path is its longest chain: d+1 dependent steps, at M = 1 one
// DMUL + DADD each.
struct CtlArgs {
  double* arena;
  Geom G;
  const int4* jobs;       // (in1, in2, out, copy | graph conv layer << 8), groups' layers one after another
  const int* layer_off;   // [nlayers+1] first job of each (group, layer)
  const int* group_off;   // [ngroups+1] first (group, layer) of each group
  int ngroups;
  int batch;
  int npairs;             // (d+2)/2
  Stamp* stamps;          // as BandArgs
  // M = 1 (real): each (group, layer)'s input series live in shared memory.
  // The group's job table and lists are copied to shared memory once; the
  // next layer's inputs are prefetched (cp.async) while a layer computes,
  // except those the layer itself produces, which its chains write straight
  // into the next layer's buffer as well as to the arena. stage_slot entries
  // are slot * 2 + (1 if produced by the previous layer).
  const int* stage_off;   // [nlayers+1] first entry of each (group, layer)'s list
  const int* stage_slot;
  const int4* sidx;       // per job: staged (in1, in2) in its layer's list, its out in the next layer's (or -1)
  const int* gjob_off;    // [ngroups+1] first job of each group
  int max_stage;          // longest list
};

struct Launchers {
  void (*conv)(const ConvArgs&, cudaStream_t);
  void (*conv_band)(const BandArgs&, cudaStream_t);
  void (*conv_flow)(const FlowArgs&, int blocks, cudaStream_t);
  int (*band_blocks_per_sm)(bool flow);
  // CTA-local dataflow: returns false (nothing launched) when a group's
  // completion flags do not fit next to the lanes in shared memory
  bool (*conv_cta)(const CtaArgs&, int max_units, cudaStream_t);
  bool (*cta_fits)(int max_units);
  void (*conv_ctl)(const CtlArgs&, size_t table_bytes, cudaStream_t);
  bool (*ctl_fits)(int max_stage, int d, size_t table_bytes);
  void (*conv_prod)(const SplitArgs&, cudaStream_t);
  void (*conv_accum)(const SplitArgs&, cudaStream_t);
  void (*add)(const AddArgs&, cudaStream_t);
  void (*scale)(const ScaleArgs&, cudaStream_t);
  void (*extract)(const ExtractArgs&, cudaStream_t);
  void (*md)(const MdArgs&, cudaStream_t);
  void (*prepare)();  // sets kernel attributes on the current device
  int lane_words;
  int threads;        // threads per block of the lane kernels (per-M translation unit)
};

#ifdef PSE_KERNELS_IMPL

constexpr int kConvThreads = kLaneThreads;

constexpr size_t kCtaSmemMax = 227 * 1024;  // dynamic shared memory of one block
#ifndef PSE_CTA_SLEEP
#define PSE_CTA_SLEEP 20  // ns between polls of a shared-memory completion flag (0: spin)
#endif
// resident blocks per SM for a target expressed in 128-thread blocks (the
// register budget stays the same whatever the block size)
constexpr int blocks_for(int minb128) { return minb128 * 128 / kConvThreads > 0 ? minb128 * 128 / kConvThreads : 1; }
constexpr int kAddThreads = kLaneThreads;

// limb q of coefficient j at src[q*S + j]: one pointer walked by S (a 64-bit
// add per limb instead of re-deriving every address from the indices)
template <int M>
__device__ __forceinline__ void load_md(const double* __restrict__ src, int S, int j, double (&v)[M]) {
  const double* p = src + j;
#pragma unroll
  for (int q = 0; q < M; ++q) {
    v[q] = __ldg(p);
    p += S;
  }
}

// coh: the series may be written during this kernel by other SMs, so it is
// read through L2 (ld.global.cg) instead of the non-coherent read-only path
template <int M, bool CTA = false>
__device__ __forceinline__ void load_md_sel(const double* __restrict__ src, int S, int j, double (&v)[M], bool coh) {
  const double* p = src + j;
#pragma unroll
  for (int q = 0; q < M; ++q) {
    v[q] = coh ? (CTA ? __ldca(p) : __ldcg(p)) : __ldg(p);
    p += S;
  }
}

// words this kernel itself wrote (plain coherent loads, not the read-only path)
template <int M>
__device__ __forceinline__ void load_md_rw(const double* src, int S, int j, double (&v)[M]) {
#pragma unroll
  for (int q = 0; q < M; ++q) v[q] = src[q * S + j];
}

template <int M>
__device__ __forceinline__ void store_md(double* dst, int S, int j, const double (&v)[M]) {
#pragma unroll
  for (int q = 0; q < M; ++q) dst[q * S + j] = v[q];
}

template <int M>
__device__ __forceinline__ void copy_md(double (&d)[M], const double (&s)[M]) {
#pragma unroll
  for (int q = 0; q < M; ++q) d[q] = s[q];
}

// ------------------------------------------------------------- convolution
// One thread per (point, job, coefficient pair). Pair p owns output
// coefficients k1 = p and k2 = d - p, so every thread performs d+2 products
// (when d is even the middle pair k1 = k2 = d/2 performs d/2+1) and warps
// stay load-balanced. Each z_k is accumulated by one thread in ascending i
// exactly as conv() does (pseries.cpp:41-48): acc = x0*y_k, then
// acc = md_add(acc, x_i*y_{k-i}) -- the bit-exactness contract.
// Consecutive lanes are consecutive pairs of one job: x_i is a broadcast
// load and y_{k-i} a coalesced one.
// MINB = resident blocks per SM the register allocation targets (4 -> 128
// registers, 3 -> 168, 2 -> 255). Large M trade occupancy for the ILP that
// ptxas only exposes with more registers; selectable at run time for tuning
// (PSE_CONV_MINB), default from conv_default_minb<M>().
// complex convolutions keep the real accumulator in the lane (55 rows at
// M = 10) for M >= 5; small M keep both in registers so that the dataflow
// kernel's operand staging still fits next to the lanes
template <int M>
__host__ __device__ constexpr bool cplx_acc_lane() {
  return M >= 5;
}

template <int M>
constexpr int conv_default_minb() {
  return 4;
}

// operand loads of a coefficient-pair chain: the read-only path, or (COH:
// the operand may have been written earlier in the same launch by this
// block) L1-cached coherent loads
template <bool COH>
__device__ __forceinline__ double ld_op(const double* p) {
  if constexpr (COH)
    return __ldca(p);
  else
    return __ldg(p);
}
template <int M, bool COH>
__device__ __forceinline__ void load_md_op(const double* __restrict__ src, int S, int j, double (&v)[M]) {
  const double* p = src + j;
#pragma unroll
  for (int q = 0; q < M; ++q) {
    v[q] = ld_op<COH>(p);
    p += S;
  }
}

// the chains of coefficient pair `pair` of job J (slots of one point at base)
template <int M, bool CPLX, bool COH>
__device__ __forceinline__ void conv_pair_at(const int4 J, double* base, const Geom& G, int pair, Lane sm) {
  const int S = G.S, d = G.d;
  const double* __restrict__ X = base + static_cast<int64_t>(J.x) * G.slot_words;
  const double* __restrict__ Y = base + static_cast<int64_t>(J.y) * G.slot_words;
  double* Z = base + static_cast<int64_t>(J.z) * G.slot_words;
  const int k1 = pair, k2 = d - pair;
  constexpr int Q = CPLX ? 2 * M : M;

  if (J.w & 1) {  // copy job (executor.cpp:130-133): out := in1
#pragma unroll 1
    for (int q = 0; q < Q; ++q) {
      Z[q * S + k1] = X[q * S + k1];
      if (k2 != k1) Z[q * S + k2] = X[q * S + k2];
    }
    return;
  }

  const int n1 = k1 + 1;
  const int total = k2 > k1 ? d + 2 : n1;
  if constexpr (!CPLX && M == 1) {
    // a plain DMUL / DADD chain: the accumulator stays in a register
    double acc = 0.0;
#pragma unroll 1
    for (int t = 0; t < total; ++t) {
      const bool second = t >= n1;
      const int kk = second ? k2 : k1;
      const int i = second ? t - n1 : t;
      const double p = __dmul_rn(ld_op<COH>(X + i), ld_op<COH>(Y + kk - i));
      acc = i == 0 ? p : __dadd_rn(acc, p);
      if (i == kk) Z[kk] = acc;
    }
  } else if constexpr (!CPLX) {
    // the accumulator lives in the lane (acc_add), not in registers, so it is
    // not live across the md_mul
    acc_init<M>(sm);
#pragma unroll 1
    for (int t = 0; t < total; ++t) {
      const bool second = t >= n1;
      const int kk = second ? k2 : k1;
      const int i = second ? t - n1 : t;
      double xr[M], yr[M], p[M], o[M];
      load_md_op<M, COH>(X, S, i, xr);
      load_md_op<M, COH>(Y, S, kk - i, yr);
      exp_mul_fast<M>(xr, yr, p, sm);
      if (i == 0) {
        copy_md<M>(o, p);
        acc_store<M>(p, sm);
      } else {
        acc_add<M>(p, o, sm);
      }
      if (i == kk) store_md<M>(Z, S, kk, o);
    }
  } else if constexpr (cplx_acc_lane<M>()) {
    // Complex, M >= 5: two passes over the coefficient chains -- the real
    // parts (re = mul(xr,yr) - mul(xi,yi), acc_re += re), then the imaginary
    // parts (im = mul(xr,yi) + mul(xi,yr), acc_im += im) -- through ONE loop
    // body of two md_muls, the accumulator in the lane. The reference's
    // per-product order (pseries.cpp:49-59) is kept within each part and the
    // two accumulations are independent, so the results are the same bits;
    // one operand pair and one accumulator are live at a time (no spills) and
    // the loop carries two inlined md_muls instead of four.
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      acc_init<M>(sm);
      double* Zp = Z + part * M * S;
      const double* Y1 = part ? Y + M * S : Y;  // y of the first product: yr (re) / yi (im)
      const double* Y2 = part ? Y : Y + M * S;  // y of the second: yi (re) / yr (im)
      const int sgn = part ? 0 : static_cast<int>(0x80000000u);
#pragma unroll 1
      for (int t = 0; t < total; ++t) {
        const bool second = t >= n1;
        const int kk = second ? k2 : k1;
        const int i = second ? t - n1 : t;
        double xa[M], yb[M], p1[M], p2[M], pr[M];
        load_md_op<M, COH>(X, S, i, xa);
        load_md_op<M, COH>(Y1, S, kk - i, yb);
        exp_mul_fast<M>(xa, yb, p1, sm);  // xr * yr | xr * yi
        load_md_op<M, COH>(X + M * S, S, i, xa);
        load_md_op<M, COH>(Y2, S, kk - i, yb);
        exp_mul_fast<M>(xa, yb, p2, sm);  // xi * yi | xi * yr
        // md_sub = exp_add of the negation (expansion.hpp:160-170): flip the
        // sign bits for the real part, branch-free
#pragma unroll
        for (int q = 0; q < M; ++q)
          p2[q] = __hiloint2double(__double2hiint(p2[q]) ^ sgn, __double2loint(p2[q]));
        exp_add_fast<M>(p1, p2, pr, sm);
        if (i == 0) {
          copy_md<M>(p1, pr);
          acc_store<M>(pr, sm);
        } else {
          acc_add<M>(pr, p1, sm);
        }
        if (i == kk) store_md<M>(Zp, S, kk, p1);
      }
    }
  } else {
    // accumulators (re, im). For M >= 5 the real one lives in the lane
    // (cplx_acc_lane), so its M registers are free while the four md_muls
    // run; the real part is added as soon as it is formed. The reference's
    // order per product (pseries.cpp:49-59) is kept: re = mul(xr,yr) -
    // mul(xi,yi); im = mul(xr,yi) + mul(xi,yr); acc += each -- the two
    // accumulations are independent, so doing re's first changes nothing.
    constexpr bool LANE_RE = cplx_acc_lane<M>();
    double ar[LANE_RE ? 1 : M], ai[M], o[M];
    if constexpr (LANE_RE) acc_init<M>(sm);
#pragma unroll 1
    for (int t = 0; t < total; ++t) {
      const bool second = t >= n1;
      const int kk = second ? k2 : k1;
      const int i = second ? t - n1 : t;
      // (xr + i xi)(yr + i yi): pseries.cpp:50-51 operand order; each md_mul
      // loads its own operands (L1 hits) so that at most one pair is live
      double xa[M], yb[M], p1[M], p2[M], pr[M];
      load_md_op<M, COH>(X, S, i, xa);
      load_md_op<M, COH>(Y, S, kk - i, yb);
      exp_mul_fast<M>(xa, yb, p1, sm);  // xr * yr
      load_md_op<M, COH>(X + M * S, S, i, xa);
      load_md_op<M, COH>(Y + M * S, S, kk - i, yb);
      exp_mul_fast<M>(xa, yb, p2, sm);  // xi * yi
      exp_sub_fast<M>(p1, p2, pr, sm);
      if constexpr (LANE_RE) {
        if (i == 0) {
          copy_md<M>(o, pr);
          acc_store<M>(pr, sm);
        } else {
          acc_add<M>(pr, o, sm);
        }
        if (i == kk) store_md<M>(Z, S, kk, o);
      } else {
        if (i == 0) copy_md<M>(ar, pr);
        else exp_add_fast<M>(ar, pr, ar, sm);
        if (i == kk) store_md<M>(Z, S, kk, ar);
      }
      load_md_op<M, COH>(X, S, i, xa);
      exp_mul_fast<M>(xa, yb, p1, sm);  // xr * yi
      load_md_op<M, COH>(X + M * S, S, i, xa);
      load_md_op<M, COH>(Y, S, kk - i, yb);
      exp_mul_fast<M>(xa, yb, p2, sm);  // xi * yr
      exp_add_fast<M>(p1, p2, pr, sm);
      if constexpr (LANE_RE) {
        // the imaginary running sum lives in the output slot's imaginary
        // words (this thread's own, L1-resident): no register is live
        // across the four md_muls (ptxas spilled them otherwise)
        if (i == 0) {
          store_md<M>(Z + M * S, S, kk, pr);
        } else {
          load_md_rw<M>(Z + M * S, S, kk, ai);
          exp_add_fast<M>(ai, pr, ai, sm);
          store_md<M>(Z + M * S, S, kk, ai);
        }
      } else {
        if (i == 0) copy_md<M>(ai, pr);
        else exp_add_fast<M>(ai, pr, ai, sm);
        if (i == kk) store_md<M>(Z + M * S, S, kk, ai);
      }
    }
  }
}

template <int M, bool CPLX>
__device__ __forceinline__ void conv_pair(const ConvArgs& a, int64_t g, Lane sm) {
  const int pair = static_cast<int>(g % a.npairs);
  const int64_t r = g / a.npairs;
  const int jb = static_cast<int>(r % a.njobs);
  const int64_t pt = r / a.njobs;
  conv_pair_at<M, CPLX, false>(a.jobs[jb], a.arena + pt * a.G.point_words, a.G, pair, sm);
}

template <int M, bool CPLX, int MINB>
__global__ void __launch_bounds__(kConvThreads, blocks_for(MINB)) k_conv(const ConvArgs a) {
  extern __shared__ double smem[];
  stamp_begin(a.t_begin);
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < static_cast<int64_t>(a.batch) * a.njobs * a.npairs) conv_pair<M, CPLX>(a, g, make_lane(smem));
  stamp_finish(a.t_end);
}

// ------------------------------------------------- banded convolution (deep)
// See BandArgs. Every lane runs at most two chain pieces (kA: steps
// iaA..ibA, then kB: steps iaB..ibB) through ONE loop body, like k_conv's
// coefficient pair. A piece that starts past i = 0 resumes from the partial
// sum its job's previous segment stored in Z[k]; every piece ends by storing
// its sum there (final once i reaches k).
// COH (dataflow kernel): inputs produced inside the launch (flag bits 2 =
// in1 and 4 = in2 of the job's .w) may have been written by other SMs during
// it and are read through L2; other inputs keep the read-only path.
// Dataflow tasks of short steps (M <= 4) stage their operand windows in
// shared memory first -- the in1 segment (<= W words per limb) and the in2
// range the task reads (<= 2W) -- so a task pays one L2 round trip instead
// of one per step. kStageSlots words per limb and warp: the task whose first
// slot is f uses words [32f, 32f + 3W) (x first, then y).
constexpr int kStageSlots = 128;
template <int M, bool COH>
__host__ __device__ constexpr bool band_stage() {
  return COH && M <= 4;
}

// lanes of a task of kind `kind` (band width W)
__device__ __forceinline__ int band_task_lanes(int kind, int W) { return kind == -2 ? W / 2 : W; }

// loads of data produced during the launch: through L2 (.cg) when the
// producer may sit on another SM; through L1 (.ca) when every producer runs
// on this SM (CTA-local dataflow: the SM's own stores keep its L1 coherent)
template <bool CTA>
__device__ __forceinline__ double ld_prod(const double* p) {
  if constexpr (CTA)
    return __ldca(p);
  else
    return __ldcg(p);
}

template <int M, bool CPLX, bool COH, bool CTA = false>
__device__ __forceinline__ void band_task(double* arena, const Geom& G, const int4* __restrict__ jobs,
                                          const int4* __restrict__ slots, int W, int64_t pt, int lane, Lane sm,
                                          double* __restrict__ stg) {
  const int S = G.S, d = G.d;
  constexpr int Q = CPLX ? 2 * M : M;
  constexpr bool STAGE = band_stage<M, COH>();
  double* base = arena + pt * G.point_words;
  // band 0 is [0, W0) with W0 = d % W + 1, the others are full
  const int W0 = d % W + 1;
  const int4 T = slots[lane >> 3];
  const int kind = T.w;
  const int span = band_task_lanes(kind, W);
  const int lt = lane & (span - 1);  // lane within the task
  const int width = T.y == 0 ? W0 : W;
  // staged windows: x_i at word xo + i - xb, y_j at word yo + j - yb
  int xb = 0, yb = 0, xo = 0, yo = 0;
  if constexpr (STAGE) {
#pragma unroll 1
    for (int f = 0; f < kSlots; ++f) {
      const int4 Tf = slots[f];
      if (Tf.w == -4 || Tf.w == -3 || (f & (band_task_lanes(Tf.w, W) / 8 - 1)) != 0) continue;
      const bool dg = Tf.w == -2;
      const int ws = Tf.z == 0 ? W0 : W;  // segment width (rectangular)
      const int4 Jh = jobs[Tf.x];
      const double* Xh = base + static_cast<int64_t>(Jh.x) * G.slot_words;
      const double* Yh = base + static_cast<int64_t>(Jh.y) * G.slot_words;
      const bool chx = COH && (Jh.w & 2), chy = COH && (Jh.w & 4);
      const int hxb = dg ? Tf.y : Tf.z, hyb = dg ? 0 : Tf.y - Tf.z - ws + 1;
      const int hxo = 32 * f, hyo = hxo + W, ny = dg ? W : 2 * W;
#pragma unroll 1
      for (int q = 0; q < Q; ++q) {
        for (int e = lane; e < W; e += 32) {
          const int ix = hxb + e;
          if (ix <= d) stg[q * kStageSlots + hxo + e] = chx ? ld_prod<CTA>(Xh + q * S + ix) : __ldg(Xh + q * S + ix);
        }
        for (int e = lane; e < ny; e += 32) {
          const int iy = hyb + e;
          if (iy >= 0 && iy <= d) stg[q * kStageSlots + hyo + e] = chy ? ld_prod<CTA>(Yh + q * S + iy) : __ldg(Yh + q * S + iy);
        }
      }
    }
    if (kind != -4 && kind != -3) {
      const int f0 = (lane >> 3) & ~(span / 8 - 1);  // first slot of this lane's task
      const int ws = T.z == 0 ? W0 : W;
      xb = kind == -2 ? T.y : T.z;
      yb = kind == -2 ? 0 : T.y - T.z - ws + 1;
      xo = 32 * f0;
      yo = xo + W;
    }
    __syncwarp();
  }
  if (kind == -4) return;
  const int job = T.x;
  int kA, iaA, ibA, kB = -1, iaB = 0, ibB = -1;
  if (kind != -2) {
    if (lt >= width) return;
    kA = T.y + lt;
    iaA = T.z;
    ibA = (T.z == 0 ? W0 : T.z + W) - 1;
  } else {
    const int j = lt;
    if (2 * j >= width) return;
    kA = T.y + j;
    iaA = T.y;
    ibA = kA;
    kB = T.y + width - 1 - j;
    iaB = T.y;
    ibB = kB;
    if (kB == kA) kB = -1;
  }
  if (kA > d) return;
  const int4 J = jobs[job];
  const double* __restrict__ X = base + static_cast<int64_t>(J.x) * G.slot_words;
  const double* __restrict__ Y = base + static_cast<int64_t>(J.y) * G.slot_words;
  double* Z = base + static_cast<int64_t>(J.z) * G.slot_words;
  const bool cx = COH && (J.w & 2), cy = COH && (J.w & 4);
  if (kind == -3) {  // copy job (executor.cpp:130-133)
#pragma unroll 1
    for (int q = 0; q < Q; ++q) Z[q * S + kA] = cx ? ld_prod<CTA>(X + q * S + kA) : X[q * S + kA];
    return;
  }
  // operand loads: limb part*M+q of x_i / y_j
  auto ldx = [&](int part, int i, double(&v)[M]) {
    if constexpr (STAGE) {
#pragma unroll
      for (int q = 0; q < M; ++q) v[q] = stg[(part * M + q) * kStageSlots + xo + i - xb];
    } else {
      load_md_sel<M, CTA>(X + part * M * S, S, i, v, cx);
    }
  };
  auto ldy = [&](int part, int j, double(&v)[M]) {
    if constexpr (STAGE) {
#pragma unroll
      for (int q = 0; q < M; ++q) v[q] = stg[(part * M + q) * kStageSlots + yo + j - yb];
    } else {
      load_md_sel<M, CTA>(Y + part * M * S, S, j, v, cy);
    }
  };
  const int nA = ibA - iaA + 1;
  const int total = nA + (kB >= 0 ? ibB - iaB + 1 : 0);
  if constexpr (!CPLX && M == 1) {
    // A plain DMUL / DADD chain per piece with the accumulator in a register
    // and the operands walked by pointer (x up, y down): the generic step's
    // index selects would cost ~15 integer instructions per two FP64 ones.
    // Partial sums resume from Z, as the generic path.
    auto piece = [&](int k, int ia, int ib) {
      const double* xp;
      const double* yp;
      bool gx = false, gy = false;  // operand read from global memory (else staged)
      if constexpr (STAGE) {
        xp = stg + xo + ia - xb;
        yp = stg + yo + (k - ia) - yb;
      } else {
        xp = X + ia;
        yp = Y + (k - ia);
        gx = true;
        gy = true;
      }
      auto rx = [&](int s) { return gx ? (cx ? ld_prod<CTA>(xp + s) : __ldg(xp + s)) : xp[s]; };
      auto ry = [&](int s) { return gy ? (cy ? ld_prod<CTA>(yp - s) : __ldg(yp - s)) : yp[-s]; };
      const int n = ib - ia + 1;
      double acc = ia == 0 ? __dmul_rn(rx(0), ry(0)) : __dadd_rn(ld_prod<CTA>(Z + k), __dmul_rn(rx(0), ry(0)));
#pragma unroll 4
      for (int s2 = 1; s2 < n; ++s2) acc = __dadd_rn(acc, __dmul_rn(rx(s2), ry(s2)));
      Z[k] = acc;
    };
    piece(kA, iaA, ibA);
    if (kB >= 0) piece(kB, iaB, ibB);
  } else if constexpr (!CPLX) {
    acc_init<M>(sm);
    double o[M];
#pragma unroll 1
    for (int t = 0; t < total; ++t) {
      const bool second = t >= nA;
      const int k = second ? kB : kA;
      const int ia = second ? iaB : iaA;
      const int i = second ? iaB + (t - nA) : iaA + t;
      double xr[M], yr[M], p[M];
      ldx(0, i, xr);
      ldy(0, k - i, yr);
      exp_mul_fast<M>(xr, yr, p, sm);
      if (i == 0) {
        copy_md<M>(o, p);
        acc_store<M>(p, sm);
      } else {
        if (i == ia) {  // resume the partial sum of the previous segment
#pragma unroll
          for (int q = 0; q < M; ++q) o[q] = ld_prod<CTA>(Z + q * S + k);
          acc_store<M>(o, sm);
        }
        acc_add<M>(p, o, sm);
      }
      if (i == (second ? ibB : ibA)) store_md<M>(Z, S, k, o);
    }
  } else if constexpr (cplx_acc_lane<M>()) {
    // as k_conv's complex branch for M >= 5: the real parts, then the
    // imaginary parts, one two-md_mul loop body, the accumulator in the lane
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      acc_init<M>(sm);
      const int sgn = part ? 0 : static_cast<int>(0x80000000u);
      double o[M];
#pragma unroll 1
      for (int t = 0; t < total; ++t) {
        const bool second = t >= nA;
        const int k = second ? kB : kA;
        const int ia = second ? iaB : iaA;
        const int i = second ? iaB + (t - nA) : iaA + t;
        double xa[M], yb[M], p1[M], p2[M], pr[M];
        ldx(0, i, xa);
        ldy(part, k - i, yb);
        exp_mul_fast<M>(xa, yb, p1, sm);  // xr * yr | xr * yi
        ldx(1, i, xa);
        ldy(1 - part, k - i, yb);
        exp_mul_fast<M>(xa, yb, p2, sm);  // xi * yi | xi * yr
#pragma unroll
        for (int q = 0; q < M; ++q)  // md_sub for the real part (expansion.hpp:160-170)
          p2[q] = __hiloint2double(__double2hiint(p2[q]) ^ sgn, __double2loint(p2[q]));
        exp_add_fast<M>(p1, p2, pr, sm);
        if (i == 0) {
          copy_md<M>(o, pr);
          acc_store<M>(pr, sm);
        } else {
          if (i == ia) {  // resume the partial sum of the previous segment
#pragma unroll
            for (int q = 0; q < M; ++q) o[q] = ld_prod<CTA>(Z + (part * M + q) * S + k);
            acc_store<M>(o, sm);
          }
          acc_add<M>(pr, o, sm);
        }
        if (i == (second ? ibB : ibA)) store_md<M>(Z + part * M * S, S, k, o);
      }
    }
  } else {
    // complex, M < 5: both accumulators in registers
    constexpr bool LANE_RE = cplx_acc_lane<M>();
    double ar[LANE_RE ? 1 : M], ai[M], o[M];
    if constexpr (LANE_RE) acc_init<M>(sm);
#pragma unroll 1
    for (int t = 0; t < total; ++t) {
      const bool second = t >= nA;
      const int k = second ? kB : kA;
      const int ia = second ? iaB : iaA;
      const int i = second ? iaB + (t - nA) : iaA + t;
      const bool last = i == (second ? ibB : ibA);
      double xa[M], yb[M], p1[M], p2[M], pr[M];  // one operand pair live at a time
      ldx(0, i, xa);
      ldy(0, k - i, yb);
      exp_mul_fast<M>(xa, yb, p1, sm);  // xr * yr
      ldx(1, i, xa);
      ldy(1, k - i, yb);
      exp_mul_fast<M>(xa, yb, p2, sm);  // xi * yi
      exp_sub_fast<M>(p1, p2, pr, sm);
      if constexpr (LANE_RE) {
        if (i == 0) {
          copy_md<M>(o, pr);
          acc_store<M>(pr, sm);
        } else {
          if (i == ia) {  // resume the partial sums of the previous segment
#pragma unroll
            for (int q = 0; q < M; ++q) o[q] = ld_prod<CTA>(Z + q * S + k);
            acc_store<M>(o, sm);
          }
          acc_add<M>(pr, o, sm);
        }
        if (last) store_md<M>(Z, S, k, o);
      } else {
        if (i == 0) {
          copy_md<M>(ar, pr);
        } else {
          if (i == ia) {
#pragma unroll
            for (int q = 0; q < M; ++q) ar[q] = ld_prod<CTA>(Z + q * S + k);
          }
          exp_add_fast<M>(ar, pr, ar, sm);
        }
        if (last) store_md<M>(Z, S, k, ar);
      }
      ldx(0, i, xa);
      exp_mul_fast<M>(xa, yb, p1, sm);  // xr * yi
      ldx(1, i, xa);
      ldy(0, k - i, yb);
      exp_mul_fast<M>(xa, yb, p2, sm);  // xi * yr
      exp_add_fast<M>(p1, p2, pr, sm);
      if constexpr (LANE_RE) {  // imaginary running sum in Z (see k_conv)
        if (i == 0) {
          store_md<M>(Z + M * S, S, k, pr);
        } else {
#pragma unroll
          for (int q = 0; q < M; ++q) ai[q] = ld_prod<CTA>(Z + (M + q) * S + k);
          exp_add_fast<M>(ai, pr, ai, sm);
          store_md<M>(Z + M * S, S, k, ai);
        }
      } else {
        if (i == 0) {
          copy_md<M>(ai, pr);
        } else {
          if (i == ia) {
#pragma unroll
            for (int q = 0; q < M; ++q) ai[q] = ld_prod<CTA>(Z + (M + q) * S + k);
          }
          exp_add_fast<M>(ai, pr, ai, sm);
        }
        if (last) store_md<M>(Z + M * S, S, k, ai);
      }
    }
  }
}

// End stamps of the layers of one warp descriptor's tasks. Lane f < kSlots
// looks up slot f's layer BEFORE the task runs (stamp_slot_layer: the load's
// latency hides behind the task) and records the end time after it
// (stamp_slot_end); -1 = nothing to stamp (empty slot, or not the first slot
// of its task).
__device__ __forceinline__ int stamp_slot_layer(const Stamp* stamps, const int4* __restrict__ jobs,
                                                const int4* __restrict__ slots, int lane) {
  if (!stamps || lane >= kSlots) return -1;
  const int4 T = slots[lane];
  if (T.w == -4) return -1;
  if (lane > 0) {
    const int4 P = slots[lane - 1];
    if (P.x == T.x && P.y == T.y && P.z == T.z && P.w == T.w) return -1;
  }
  return jobs[T.x].w >> 8;
}
__device__ __forceinline__ void stamp_slot_end(Stamp* stamps, int layer) {
  if (layer >= 0) atomicMax(stamps + 1 + layer, global_ns());
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kConvThreads, blocks_for(4)) k_conv_band(const BandArgs a) {
  extern __shared__ double smem[];
  const Lane sm = make_lane(smem);
  if (a.stamps) stamp_begin(a.stamps);
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (gw >= static_cast<int64_t>(a.batch) * a.ntasks) return;
  const int tw = static_cast<int>(gw % a.ntasks);
  const int4* slots = a.tasks + static_cast<int64_t>(tw) * kSlots;
  const int layer = stamp_slot_layer(a.stamps, a.jobs, slots, threadIdx.x & 31);
  band_task<M, CPLX, false>(a.arena, a.G, a.jobs, slots, a.W, gw / a.ntasks, threadIdx.x & 31, sm, nullptr);
  __syncwarp();
  stamp_slot_end(a.stamps, layer);
}

// Dataflow form of the banded convolution: ONE persistent launch. Warps take
// work units (descriptor p of the scheduled order, point b) from a global
// counter in order, wait until the units p depends on are done for point b
// (relaxed polls of their flags + an acquire fence), run the task and publish their own flag
// (stores, fence, release). A unit only waits for units earlier in the
// order, which were taken by running warps before it, so the scheme cannot
// deadlock; a wait that exceeds ~10 s (global timer) traps instead of
// hanging the GPU.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kConvThreads, blocks_for(4)) k_conv_flow(const FlowArgs a) {
  extern __shared__ double smem[];
  const Lane sm = make_lane(smem);
  const int lane = threadIdx.x & 31;
  const int64_t units = static_cast<int64_t>(a.nunits) * a.batch;
  // per-warp staging area after the lanes (band_stage)
  constexpr int Q = CPLX ? 2 * M : M;
  double* stg = smem + kLaneThreads * (CPLX && !cplx_acc_lane<M>() ? MdTraits<M>::LANE : MdTraits<M>::LANE_CONV) +
                (threadIdx.x >> 5) * kStageSlots * Q;
  if (a.stamps) stamp_begin(a.stamps);
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(a.counter, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (static_cast<int64_t>(u) >= units) return;
    const int p = static_cast<int>(u / a.batch);
    const int64_t pt = static_cast<int64_t>(u % a.batch);
    unsigned* fl = a.flags + pt * a.nunits;
    // relaxed polling, then one acquire fence once the flag is seen set (an
    // acquire load per poll would invalidate L1 every iteration)
    for (int e = a.dep_off[p] + lane; e < a.dep_off[p + 1]; e += 32) {
      const unsigned* f = fl + a.deps[e];
      unsigned spins = 0;
      unsigned long long t0 = 0;
      while (ld_relaxed(f) == 0u) {
        __nanosleep(32);
        if ((++spins & 1023u) == 0u) {  // a dependency that never completes: trap after ~10 s
          unsigned long long now;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
          if (t0 == 0) t0 = now;
          else if (now - t0 > 10000000000ull) __trap();
        }
      }
      fence_acquire();
    }
    __syncwarp();
    const int4* slots = a.tasks + static_cast<int64_t>(p) * kSlots;
    const int layer = stamp_slot_layer(a.stamps, a.jobs, slots, lane);
    band_task<M, CPLX, true>(a.arena, a.G, a.jobs, slots, a.W, pt, lane, sm, stg);
    __syncwarp();  // the staging area is rewritten by the next unit
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(fl + p, 1u);
    stamp_slot_end(a.stamps, layer);
  }
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kConvThreads, 1) k_conv_cta(const CtaArgs a) {
  extern __shared__ double smem[];
  const Lane sm = make_lane(smem);
  const int lane = threadIdx.x & 31;
  constexpr int Q = CPLX ? 2 * M : M;
  constexpr int nwarps = kConvThreads / 32;
  double* stg = smem + kLaneThreads * (CPLX && !cplx_acc_lane<M>() ? MdTraits<M>::LANE : MdTraits<M>::LANE_CONV) +
                (threadIdx.x >> 5) * kStageSlots * Q;
  // after the lanes and the staging areas: the hand-out counter, then one
  // completion byte per descriptor of this group
  unsigned* counter = reinterpret_cast<unsigned*>(
      smem + kLaneThreads * (CPLX && !cplx_acc_lane<M>() ? MdTraits<M>::LANE : MdTraits<M>::LANE_CONV) +
      (band_stage<M, true>() ? nwarps * kStageSlots * Q : 0));
  volatile unsigned char* done = reinterpret_cast<volatile unsigned char*>(counter + 1);
  const int grp = blockIdx.x % a.ngroups;
  const int64_t pt = blockIdx.x / a.ngroups;
  const int u0 = a.group_off[grp], nu = a.group_off[grp + 1] - u0;
  for (int i = threadIdx.x; i < nu; i += blockDim.x) done[i] = 0;
  if (threadIdx.x == 0) *counter = 0;
  if (a.stamps) stamp_begin(a.stamps);
  __syncthreads();
  for (;;) {
    unsigned u = 0;
    if (lane == 0) u = atomicAdd(counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (static_cast<int>(u) >= nu) break;
    const int p = u0 + static_cast<int>(u);
    for (int e = a.dep_off[p] + lane; e < a.dep_off[p + 1]; e += 32)
      while (done[a.deps[e]] == 0) {
#if PSE_CTA_SLEEP
        __nanosleep(PSE_CTA_SLEEP);
#endif
      }
    __syncwarp();
    __threadfence_block();
    const int4* slots = a.tasks + static_cast<int64_t>(p) * kSlots;
    const int layer = stamp_slot_layer(a.stamps, a.jobs, slots, lane);
    band_task<M, CPLX, true, true>(a.arena, a.G, a.jobs, slots, a.W, pt, lane, sm, stg);
    __syncwarp();  // the staging area is rewritten by the next unit
    __threadfence_block();
    if (lane == 0) done[u] = 1;
    stamp_slot_end(a.stamps, layer);
  }
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// M = 1 chains in register blocks. A job's d+1 chains z_k = sum_i x_i y_{k-i}
// (ascending i, pseries.cpp:41-48) are cut into blocks of kCtlR adjacent
// chains; thread b of a job runs block b (ctl_block_m1). kCtlR = 3 and four
// chunks per loop trip measured best on C3 at m=1 (conv stage 0.164 ms; R = 2:
// 0.174, 4: 0.202, 5: 0.202; one chain per thread 0.220; pairs of blocks
// b and B-1-b per thread, side by side or one after the other, 0.242-0.248;
// pairs of single chains (k, d-k) 0.252). An accumulator starts at -0
// (x + -0 == x bitwise for every x, so the first sum is the first product,
// as in the reference).
#ifndef PSE_CTL_R
#define PSE_CTL_R 3
#endif
#ifndef PSE_CTL_UNROLL
#define PSE_CTL_UNROLL 4
#endif
constexpr int kCtlR = PSE_CTL_R;
constexpr int kCtlUnroll = PSE_CTL_UNROLL;
constexpr int kCtlOff = 8;           // words in front of each sub-series (the loop's look-ahead)
constexpr int kCtlLS = 512 / kCtlR;  // sub-series stride: d + 1 <= kCtlR * (kCtlLS - kCtlOff - 1)
__host__ __device__ constexpr int ctl_series_words() { return kCtlR * kCtlLS; }
__device__ __forceinline__ int ctl_pos(int j) { return (j % kCtlR) * kCtlLS + kCtlOff + j / kCtlR; }

// One register block of R adjacent M = 1 chains (k0 = bR .. k0+R-1) per
// thread: steps s = 0..k0+R-1 taken R at a time (a "chunk"), the block's
// chains sharing x_s and chain r reusing the y element chain r-1 used one
// step earlier (a ring of R registers), so a step is one x load (a
// broadcast), one y load and R independent DMUL + DADD pairs. The last chunk
// is peeled (chain k0+r ends at its step r). Operands one chunk ahead.
// Staged series are transposed by R (element j at (j % R) * kCtlLS +
// kCtlOff + j / R): the y loads of a warp (consecutive b) are consecutive
// words.
__device__ __forceinline__ void ctl_block_m1(const double* X, const double* Y, double* Z, double* W, int b, int d) {
  constexpr int R = kCtlR, LS = kCtlLS;
  const double* px = X + kCtlOff;
  const double* py = Y + kCtlOff + b;  // y_{R(b-u)} at py[0], y_{R(b-u)-j} at py[(R-j) LS - 1]
  double acc[R], w[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = -0.0;
#pragma unroll
  for (int r = 1; r < R; ++r) w[r] = py[r * LS];  // y_{k0+r}
  double xc[R], yc[R];
  auto load = [&](double (&xv)[R], double (&yv)[R]) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      xv[j] = px[j * LS];
      yv[j] = j == 0 ? py[0] : py[(R - j) * LS - 1];
    }
  };
  load(xc, yc);
#pragma unroll kCtlUnroll
  for (int u = 0; u < b; ++u) {
    ++px;
    --py;
    double xn[R], yn[R];
    load(xn, yn);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      w[(R - j) % R] = yc[j];  // y_{k0-s}, s = uR + j
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(xc[j], w[(r - j + R) % R]));
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      xc[j] = xn[j];
      yc[j] = yn[j];
    }
  }
  // last chunk (u = b): chain r ends at step j = r
#pragma unroll
  for (int j = 0; j < R; ++j) {
    w[(R - j) % R] = yc[j];
#pragma unroll
    for (int r = j; r < R; ++r) acc[r] = __dadd_rn(acc[r], __dmul_rn(xc[j], w[(r - j + R) % R]));
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int k = b * R + r;
    if (k <= d) {
      Z[k] = acc[r];
      if (W) W[r * LS + kCtlOff + b] = acc[r];
    }
  }
}

// M = 1, real: the group's layers with shared-memory operands (see CtlArgs)
__device__ __forceinline__ void ctl_group_m1(const CtlArgs& a, double* smem_d, int grp, double* base) {
  const int d = a.G.d, n1 = d + 1;
  constexpr int SW = ctl_series_words();
  const int nthr = (d + kCtlR) / kCtlR;  // register blocks = threads per job
  const int64_t sw = a.G.slot_words;
  const int jb0 = a.gjob_off[grp], nj = a.gjob_off[grp + 1] - jb0;
  const int lb0 = a.group_off[grp], nl = a.group_off[grp + 1] - lb0;
  if (nl == 0) return;  // a group without conv jobs on this rank (sharded plans)
  const int sb0 = a.stage_off[lb0], ns = a.stage_off[lb0 + nl] - sb0;
  // shared memory: the two stage buffers, then the group's tables
  double* buf0 = smem_d;
  double* buf1 = smem_d + static_cast<size_t>(a.max_stage) * SW;
  int4* sj = reinterpret_cast<int4*>(buf1 + static_cast<size_t>(a.max_stage) * SW);
  int4* sx = sj + nj;
  int* loff = reinterpret_cast<int*>(sx + nj);  // [nl+1], group-relative job index
  int* soff = loff + nl + 1;                    // [nl+1], group-relative entry index
  int* sslot = soff + nl + 1;                   // [ns]
  for (int t = threadIdx.x; t < nj; t += blockDim.x) {
    sj[t] = a.jobs[jb0 + t];
    sx[t] = a.sidx[jb0 + t];
  }
  for (int t = threadIdx.x; t <= nl; t += blockDim.x) {
    loff[t] = a.layer_off[lb0 + t] - jb0;
    soff[t] = a.stage_off[lb0 + t] - sb0;
  }
  for (int t = threadIdx.x; t < ns; t += blockDim.x) sslot[t] = a.stage_slot[sb0 + t];
  __syncthreads();
  // layer 0's inputs: every entry from the arena
  for (int w = threadIdx.x; w < (soff[1] - soff[0]) * n1; w += blockDim.x) {
    const int e = w / n1, c = w - e * n1;
    cp_async8(buf0 + e * SW + ctl_pos(c), base + (sslot[e] >> 1) * sw + c);
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int l = 0; l < nl; ++l) {
    const double* cur = (l & 1) ? buf1 : buf0;
    double* nxt = (l & 1) ? buf0 : buf1;
    const int j0 = loff[l], n = (loff[l + 1] - j0) * nthr;
    if (l + 1 < nl) {
      // prefetch the next layer's inputs that this layer does not produce,
      // by the threads without chains first (counted from the last thread)
      const int e0 = soff[l + 1], nw = (soff[l + 2] - e0) * n1;
      for (int w = blockDim.x - 1 - threadIdx.x; w < nw; w += blockDim.x) {
        const int e = w / n1, c = w - e * n1;
        const int ss = sslot[e0 + e];
        if (!(ss & 1)) cp_async8(nxt + e * SW + ctl_pos(c), base + (ss >> 1) * sw + c);
      }
    }
#pragma unroll 1
    for (int it = threadIdx.x; it < n; it += blockDim.x) {
      const int jl = it / nthr;
      const int q = it - jl * nthr;
      const int4 J = sj[j0 + jl], X4 = sx[j0 + jl];
      double* Z = base + J.z * sw;
      double* W = X4.z >= 0 ? nxt + X4.z * SW : nullptr;
      const double* X = cur + X4.x * SW;
      if (J.w & 1) {  // copy job (executor.cpp:130-133): this thread's block of coefficients
        for (int k = kCtlR * q; k < kCtlR * (q + 1) && k <= d; ++k) {
          const double v = X[ctl_pos(k)];
          Z[k] = v;
          if (W) W[ctl_pos(k)] = v;
        }
      } else {
        ctl_block_m1(X, cur + X4.y * SW, Z, W, q, d);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (a.stamps && threadIdx.x == 0) atomicMax(a.stamps + 1 + (sj[j0].w >> 8), global_ns());
  }
}

// threads per block of k_conv_ctl: the lane kernels' count, except at M = 1
// (real, no lanes): a layer of p2 has at most 4 jobs x 51 register blocks,
// and the blocks want more than the 64 registers a 1024-thread block allows
template <int M, bool CPLX>
__host__ __device__ constexpr int ctl_threads() {
  return M == 1 && !CPLX ? 320 : kConvThreads;
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(ctl_threads<M, CPLX>(), 1) k_conv_ctl(const CtlArgs a) {
  extern __shared__ double smem[];
  const Lane sm = make_lane(smem);
  const int grp = blockIdx.x % a.ngroups;
  double* base = a.arena + static_cast<int64_t>(blockIdx.x / a.ngroups) * a.G.point_words;
  if (a.stamps) stamp_begin(a.stamps);
  const int npairs = a.npairs;
  if constexpr (M == 1 && !CPLX) {
    ctl_group_m1(a, smem, grp, base);
  } else {
#pragma unroll 1
    for (int L = a.group_off[grp]; L < a.group_off[grp + 1]; ++L) {
      const int j0 = a.layer_off[L];
      const int n = (a.layer_off[L + 1] - j0) * npairs;
#pragma unroll 1
      for (int it = threadIdx.x; it < n; it += blockDim.x)
        conv_pair_at<M, CPLX, true>(a.jobs[j0 + it / npairs], base, a.G, it % npairs, sm);
      __syncthreads();
      if (a.stamps && threadIdx.x == 0) atomicMax(a.stamps + 1 + (a.jobs[j0].w >> 8), global_ns());
    }
  }
}

// ------------------------------------------------ split convolution (small)
// Phase A: one thread per (point, job, product index). The product of a
// complex coefficient pair is the (re, im) pair conv() adds to its
// accumulators: sub(mul(re,re), mul(im,im)), add(mul(re,im), mul(im,re)).
template <int M, bool CPLX>
__device__ __forceinline__ void conv_prod_item(const SplitArgs& a, int64_t g, Lane sm) {
  const int off = static_cast<int>(g % a.T);
  const int64_t r = g / a.T;
  const int jb = static_cast<int>(r % a.njobs);
  const int64_t pt = r / a.njobs;
  const int4 J = a.jobs[jb];
  if (J.w) return;  // copy jobs have no products
  const int2 ki = a.tri[off];
  const int S = a.G.S;
  constexpr int Q = CPLX ? 2 * M : M;
  const double* base = a.arena + pt * a.G.point_words;
  const double* X = base + static_cast<int64_t>(J.x) * a.G.slot_words;
  const double* Y = base + static_cast<int64_t>(J.y) * a.G.slot_words;
  double* P = a.prod + (r * a.T + off) * Q;
  double xr[M], yr[M], p[M];
  load_md<M>(X, S, ki.y, xr);
  load_md<M>(Y, S, ki.x - ki.y, yr);
  if constexpr (!CPLX) {
    exp_mul_fast<M>(xr, yr, p, sm);
#pragma unroll
    for (int q = 0; q < M; ++q) P[q] = p[q];
  } else {
    double xi[M], yi[M], p2[M], pim[M];
    load_md<M>(X + M * S, S, ki.y, xi);
    load_md<M>(Y + M * S, S, ki.x - ki.y, yi);
    exp_mul_fast<M>(xr, yr, p, sm);
    exp_mul_fast<M>(xi, yi, p2, sm);
    exp_sub_fast<M>(p, p2, p, sm);
#pragma unroll
    for (int q = 0; q < M; ++q) P[q] = p[q];
    exp_mul_fast<M>(xr, yi, p, sm);
    exp_mul_fast<M>(xi, yr, p2, sm);
    exp_add_fast<M>(p, p2, pim, sm);
#pragma unroll
    for (int q = 0; q < M; ++q) P[M + q] = pim[q];
  }
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kConvThreads) k_conv_prod(const SplitArgs a) {
  extern __shared__ double smem[];
  stamp_begin(a.t_begin);
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < static_cast<int64_t>(a.batch) * a.njobs * a.T) conv_prod_item<M, CPLX>(a, g, make_lane(smem));
}

// Phase B: one thread per (point, job, coefficient pair), the same pairing
// as k_conv; acc = P(k,0), acc = md_add(acc, P(k,i)) for ascending i.
template <int M, bool CPLX>
__device__ __forceinline__ void conv_accum_pair(const SplitArgs& a, int64_t g, Lane sm) {
  const int npairs = (a.G.d + 2) / 2;
  const int pair = static_cast<int>(g % npairs);
  const int64_t r = g / npairs;
  const int jb = static_cast<int>(r % a.njobs);
  const int64_t pt = r / a.njobs;
  const int4 J = a.jobs[jb];
  const int S = a.G.S, d = a.G.d;
  constexpr int Q = CPLX ? 2 * M : M;
  double* base = a.arena + pt * a.G.point_words;
  double* Z = base + static_cast<int64_t>(J.z) * a.G.slot_words;
  const int k1 = pair, k2 = d - pair;
  if (J.w) {
    const double* X = base + static_cast<int64_t>(J.x) * a.G.slot_words;
#pragma unroll 1
    for (int q = 0; q < Q; ++q) {
      Z[q * S + k1] = X[q * S + k1];
      if (k2 != k1) Z[q * S + k2] = X[q * S + k2];
    }
    return;
  }
  const double* P = a.prod + r * a.T * Q;
#pragma unroll 1
  for (int c = 0; c < (k2 != k1 ? 2 : 1); ++c) {
    const int k = c ? k2 : k1;
    const double* Pk = P + static_cast<int64_t>(k) * (k + 1) / 2 * Q;
    // The chain is latency-bound (one warp per scheduler at most), so the
    // next product is fetched while the current md_add runs.
    double ar[M], ai[M], nr[M], ni[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      ar[q] = Pk[q];
      nr[q] = k >= 1 ? Pk[Q + q] : 0.0;
      if constexpr (CPLX) {
        ai[q] = Pk[M + q];
        ni[q] = k >= 1 ? Pk[Q + M + q] : 0.0;
      }
    }
#pragma unroll 1
    for (int i = 1; i <= k; ++i) {
      double p[M], pi[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        p[q] = nr[q];
        if constexpr (CPLX) pi[q] = ni[q];
      }
      if (i < k) {
#pragma unroll
        for (int q = 0; q < M; ++q) {
          nr[q] = Pk[(i + 1) * Q + q];
          if constexpr (CPLX) ni[q] = Pk[(i + 1) * Q + M + q];
        }
      }
      exp_add_fast<M, true>(ar, p, ar, sm);
      if constexpr (CPLX) exp_add_fast<M, true>(ai, pi, ai, sm);
    }
    store_md<M>(Z, S, k, ar);
    if constexpr (CPLX) store_md<M>(Z + M * S, S, k, ai);
  }
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kConvThreads) k_conv_accum(const SplitArgs a) {
  extern __shared__ double smem[];
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < static_cast<int64_t>(a.batch) * a.njobs * ((a.G.d + 2) / 2)) conv_accum_pair<M, CPLX>(a, g, make_lane(smem));
  stamp_finish(a.t_end);
}

// ---------------------------------------------------------------- addition
// One thread per (point, job, coefficient): dst_k := md_add(dst_k, src_k)
// (executor.cpp:144-148, operand order x = dst, y = src).
template <int M, bool CPLX>
__device__ __forceinline__ void add_item(const AddArgs& a, int64_t g, Lane sm) {
  const int d1 = a.G.d + 1;
  const int k = static_cast<int>(g % d1);
  const int64_t r = g / d1;
  const int jb = static_cast<int>(r % a.njobs);
  const int64_t pt = r / a.njobs;
  const int2 J = a.jobs[jb];
  const int S = a.G.S;
  double* base = a.arena + pt * a.G.point_words;
  const double* src = base + static_cast<int64_t>(J.x) * a.G.slot_words;
  double* dst = base + static_cast<int64_t>(J.y) * a.G.slot_words;
#pragma unroll
  for (int part = 0; part < (CPLX ? 2 : 1); ++part) {
    double x[M], y[M], z[M];
    load_md<M>(dst + part * M * S, S, k, x);
    load_md<M>(src + part * M * S, S, k, y);
    exp_add_fast<M>(x, y, z, sm);
    store_md<M>(dst + part * M * S, S, k, z);
  }
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kAddThreads) k_add(const AddArgs a) {
  extern __shared__ double smem[];
  stamp_begin(a.t_begin);
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < static_cast<int64_t>(a.batch) * a.njobs * (a.G.d + 1)) add_item<M, CPLX>(a, g, make_lane(smem));
  stamp_finish(a.t_end);
}

// ------------------------------------------------------------ scale phase
// TermScale (executor.cpp:138-143 -> series_scale_int, pseries.cpp:85-93)
template <int M, bool CPLX>
__device__ __forceinline__ void scale_item(const ScaleArgs& a, int64_t g, Lane sm) {
  const int d1 = a.G.d + 1;
  const int k = static_cast<int>(g % d1);
  const int64_t r = g / d1;
  const int it = static_cast<int>(r % a.nitems);
  const int64_t pt = r / a.nitems;
  const int2 T = a.items[it];
  const int S = a.G.S;
  double* s = a.arena + pt * a.G.point_words + static_cast<int64_t>(T.x) * a.G.slot_words;
  double c[M];
#pragma unroll
  for (int q = 0; q < M; ++q) c[q] = q == 0 ? static_cast<double>(T.y) : 0.0;
#pragma unroll
  for (int part = 0; part < (CPLX ? 2 : 1); ++part) {
    double x[M], z[M];
    load_md<M>(s + part * M * S, S, k, x);
    exp_mul_fast<M>(x, c, z, sm);
    store_md<M>(s + part * M * S, S, k, z);
  }
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kAddThreads) k_scale(const ScaleArgs a) {
  extern __shared__ double smem[];
  stamp_begin(a.t_begin);
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < static_cast<int64_t>(a.batch) * a.nitems * (a.G.d + 1)) scale_item<M, CPLX>(a, g, make_lane(smem));
  stamp_finish(a.t_end);
}

// ----------------------------------------------------------------- extract
// extract (executor.cpp:254-269): value row then one row per variable,
// multiplier applied with md_mul, absent variables give zero series.
template <int M, bool CPLX>
__device__ __forceinline__ void extract_item(const ExtractArgs& a, int64_t g, Lane sm) {
  const int d1 = a.G.d + 1;
  const int k = static_cast<int>(g % d1);
  const int64_t r = g / d1;
  const int row = static_cast<int>(r % a.nrows);
  const int64_t pt = r / a.nrows;
  const int slot = a.row_slot[row];
  const int mult = a.row_mult[row];
  const int S = a.G.S;
  const int64_t plane = static_cast<int64_t>(a.batch) * a.nrows * d1;  // words per q
  double* out = a.out + (pt * a.nrows + row) * d1 + k;
#pragma unroll
  for (int part = 0; part < (CPLX ? 2 : 1); ++part) {
    double x[M];
    if (slot < 0) {
#pragma unroll
      for (int q = 0; q < M; ++q) x[q] = 0.0;
    } else {
      const double* s = a.arena + pt * a.G.point_words + static_cast<int64_t>(slot) * a.G.slot_words;
      load_md<M>(s + part * M * S, S, k, x);
      if (mult != 1) {
        double c[M], z[M];
#pragma unroll
        for (int q = 0; q < M; ++q) c[q] = q == 0 ? static_cast<double>(mult) : 0.0;
        exp_mul_fast<M>(x, c, z, sm);
        copy_md<M>(x, z);
      }
    }
#pragma unroll
    for (int q = 0; q < M; ++q) out[(part * M + q) * plane] = x[q];
  }
}

template <int M, bool CPLX>
__global__ void __launch_bounds__(kAddThreads) k_extract(const ExtractArgs a) {
  extern __shared__ double smem[];
  stamp_begin(a.t_begin);
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < static_cast<int64_t>(a.batch) * a.nrows * (a.G.d + 1)) extract_item<M, CPLX>(a, g, make_lane(smem));
  stamp_finish(a.t_end);
}

// --------------------------------------------------------- md primitives
template <int M>
__global__ void __launch_bounds__(kAddThreads) k_md(const MdArgs a) {
  extern __shared__ double smem[];
  const Lane sm = make_lane(smem);
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= a.count) return;
  double x[M], y[M], z[M];
#pragma unroll
  for (int q = 0; q < M; ++q) {
    x[q] = a.x[c * M + q];
    y[q] = a.y[c * M + q];
  }
  if (a.impl == 1) {
    double ny[M];
    if (a.op == 1) {
#pragma unroll
      for (int q = 0; q < M; ++q) ny[q] = -y[q];
    }
    if (a.op == 0) exp_add_lit<M>(x, y, z);
    else if (a.op == 1) {
      if constexpr (M == 1) z[0] = __dsub_rn(x[0], y[0]);
      else exp_add_lit<M>(x, ny, z);
    } else exp_mul_lit<M>(x, y, z);
  } else {
    if (a.op == 0) exp_add_fast<M>(x, y, z, sm);
    else if (a.op == 1) exp_sub_fast<M>(x, y, z, sm);
    else exp_mul_fast<M>(x, y, z, sm);
  }
#pragma unroll
  for (int q = 0; q < M; ++q) a.out[c * M + q] = z[q];
}

template <int M, bool CPLX>
struct Impl {
  static size_t smem(int threads) { return static_cast<size_t>(threads) * MdTraits<M>::LANE * sizeof(double); }
  static size_t smem_conv(int threads) {
    return static_cast<size_t>(threads) * (CPLX && !cplx_acc_lane<M>() ? MdTraits<M>::LANE : MdTraits<M>::LANE_CONV) *
           sizeof(double);
  }
  static int minb() {
    static const int v = [] {
      const char* e = getenv("PSE_CONV_MINB");
      const int x = e ? atoi(e) : conv_default_minb<M>();
      return (x >= 2 && x <= 5) ? x : conv_default_minb<M>();
    }();
    return v;
  }
  static void conv(const ConvArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.njobs * a.npairs;
    if (n == 0) return;
    const size_t sh = smem_conv(kConvThreads);
    const unsigned grid = static_cast<unsigned>((n + kConvThreads - 1) / kConvThreads);
    switch (M >= 8 ? minb() : 4) {
      case 2: k_conv<M, CPLX, 2><<<grid, kConvThreads, sh, s>>>(a); break;
      case 3: k_conv<M, CPLX, 3><<<grid, kConvThreads, sh, s>>>(a); break;
      case 5: k_conv<M, CPLX, 5><<<grid, kConvThreads, sh, s>>>(a); break;
      default: k_conv<M, CPLX, 4><<<grid, kConvThreads, sh, s>>>(a); break;
    }
  }
  static void conv_band(const BandArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.ntasks * 32;
    if (n == 0) return;
    const size_t sh = smem_conv(kConvThreads);
    k_conv_band<M, CPLX><<<static_cast<unsigned>((n + kConvThreads - 1) / kConvThreads), kConvThreads, sh, s>>>(a);
  }
  static size_t smem_flow() {
    return smem_conv(kConvThreads) +
           (band_stage<M, true>() ? static_cast<size_t>(kConvThreads / 32) * kStageSlots * (CPLX ? 2 * M : M) *
                                        sizeof(double)
                                  : 0);
  }
  static void conv_flow(const FlowArgs& a, int blocks, cudaStream_t s) {
    if (a.nunits == 0) return;
    k_conv_flow<M, CPLX><<<blocks, kConvThreads, smem_flow(), s>>>(a);
  }
  static size_t smem_cta_base() { return smem_flow() + sizeof(unsigned); }
  static bool cta_fits(int max_units) { return smem_cta_base() + static_cast<size_t>(max_units) <= kCtaSmemMax; }
  static bool conv_cta(const CtaArgs& a, int max_units, cudaStream_t s) {
    const size_t sh = smem_cta_base() + static_cast<size_t>(max_units);
    if (sh > kCtaSmemMax) return false;
    if (a.ngroups > 0) k_conv_cta<M, CPLX><<<static_cast<unsigned>(a.ngroups) * a.batch, kConvThreads, sh, s>>>(a);
    return true;
  }
  // shared memory of k_conv_ctl: the lanes, or (M = 1, real) the staged series
  // (M = 1: two stage buffers of max_stage series, then the largest group's
  // tables, `table_bytes`)
  static size_t smem_ctl(int max_stage, int d, size_t table_bytes) {
    return M == 1 && !CPLX ? 2 * static_cast<size_t>(max_stage) * ctl_series_words() * sizeof(double) + table_bytes
                           : smem_conv(kConvThreads);
  }
  static bool ctl_fits(int max_stage, int d, size_t table_bytes) {
    return smem_ctl(max_stage, d, table_bytes) <= kCtaSmemMax &&
           (!(M == 1 && !CPLX) || d + 1 <= kCtlR * (kCtlLS - kCtlOff - 1));
  }
  static void conv_ctl(const CtlArgs& a, size_t table_bytes, cudaStream_t s) {
    if (a.ngroups > 0)
      k_conv_ctl<M, CPLX><<<static_cast<unsigned>(a.ngroups) * a.batch, ctl_threads<M, CPLX>(),
                            smem_ctl(a.max_stage, a.G.d, table_bytes), s>>>(a);
  }
  // resident blocks per SM: banded waves (flow = false) or the dataflow kernel
  static int band_blocks_per_sm(bool flow) {
    int nb = 0;
    if (flow)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_conv_flow<M, CPLX>, kConvThreads, smem_flow());
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_conv_band<M, CPLX>, kConvThreads, smem_conv(kConvThreads));
    return nb > 0 ? nb : 1;
  }
  static void conv_prod(const SplitArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.njobs * a.T;
    if (n == 0) return;
    k_conv_prod<M, CPLX><<<static_cast<unsigned>((n + kConvThreads - 1) / kConvThreads), kConvThreads,
                           smem(kConvThreads), s>>>(a);
  }
  static void conv_accum(const SplitArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.njobs * ((a.G.d + 2) / 2);
    if (n == 0) return;
    k_conv_accum<M, CPLX><<<static_cast<unsigned>((n + kConvThreads - 1) / kConvThreads), kConvThreads,
                            smem(kConvThreads), s>>>(a);
  }
  static void add(const AddArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.njobs * (a.G.d + 1);
    if (n == 0) return;
    const size_t sh = smem(kAddThreads);
    k_add<M, CPLX><<<static_cast<unsigned>((n + kAddThreads - 1) / kAddThreads), kAddThreads, sh, s>>>(a);
  }
  static void scale(const ScaleArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.nitems * (a.G.d + 1);
    if (n == 0) return;
    const size_t sh = smem(kAddThreads);
    k_scale<M, CPLX><<<static_cast<unsigned>((n + kAddThreads - 1) / kAddThreads), kAddThreads, sh, s>>>(a);
  }
  static void extract(const ExtractArgs& a, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(a.batch) * a.nrows * (a.G.d + 1);
    if (n == 0) return;
    const size_t sh = smem(kAddThreads);
    k_extract<M, CPLX><<<static_cast<unsigned>((n + kAddThreads - 1) / kAddThreads), kAddThreads, sh, s>>>(a);
  }
  static void md(const MdArgs& a, cudaStream_t s) {
    if (a.count == 0) return;
    const size_t sh = smem(kAddThreads);
    k_md<M><<<static_cast<unsigned>((a.count + kAddThreads - 1) / kAddThreads), kAddThreads, sh, s>>>(a);
  }
  static void prepare() {
    const int c = static_cast<int>(smem(kConvThreads)), o = static_cast<int>(smem(kAddThreads));
    const int cc = static_cast<int>(smem_conv(kConvThreads));
    cudaFuncSetAttribute(k_conv<M, CPLX, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cc);
    cudaFuncSetAttribute(k_conv<M, CPLX, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, cc);
    cudaFuncSetAttribute(k_conv<M, CPLX, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, cc);
    cudaFuncSetAttribute(k_conv<M, CPLX, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, cc);
    cudaFuncSetAttribute(k_conv_band<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, cc);
    cudaFuncSetAttribute(k_conv_cta<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCtaSmemMax));
    cudaFuncSetAttribute(k_conv_ctl<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCtaSmemMax));
    cudaFuncSetAttribute(k_conv_flow<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_flow()));
    cudaFuncSetAttribute(k_conv_prod<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, c);
    cudaFuncSetAttribute(k_conv_accum<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, c);
    cudaFuncSetAttribute(k_add<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, o);
    cudaFuncSetAttribute(k_scale<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, o);
    cudaFuncSetAttribute(k_extract<M, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, o);
    cudaFuncSetAttribute(k_md<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, o);
  }
  static const Launchers* table() {
    static const Launchers L{&conv, &conv_band, &conv_flow, &band_blocks_per_sm, &conv_cta, &cta_fits, &conv_ctl, &ctl_fits, &conv_prod, &conv_accum, &add, &scale, &extract, &md, &prepare, MdTraits<M>::LANE, kLaneThreads};
    return &L;
  }
};

#define PSE_INSTANTIATE(M)                                                              \
  const Launchers* launchers_m##M(bool cplx) {                                           \
    return cplx ? Impl<M, true>::table() : Impl<M, false>::table();                      \
  }

#endif  // PSE_KERNELS_IMPL

const Launchers* launchers_m1(bool);
const Launchers* launchers_m2(bool);
const Launchers* launchers_m3(bool);
const Launchers* launchers_m4(bool);
const Launchers* launchers_m5(bool);
const Launchers* launchers_m8(bool);
const Launchers* launchers_m10(bool);

inline const Launchers* launchers_for(int m, bool cplx) {
  switch (m) {
    case 1: return launchers_m1(cplx);
    case 2: return launchers_m2(cplx);
    case 3: return launchers_m3(cplx);
    case 4: return launchers_m4(cplx);
    case 5: return launchers_m5(cplx);
    case 8: return launchers_m8(cplx);
    case 10: return launchers_m10(cplx);
    default: return nullptr;
  }
}

}  // namespace pse
