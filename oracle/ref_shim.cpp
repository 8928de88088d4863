// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference engine (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libpseval_ref.so). It lets the Python tests and the bench's
// cpu_baseline / --impl reference leg call the reference's own code:
//   gen_benchmark        proj/src/gen.cpp:50-71
//   build_jobgraph       proj/src/jobgraph.cpp:199-262
//   fold/stage/run_*     proj/src/executor.cpp:69-96, 168-231, 271-276
//   extract              proj/src/executor.cpp:254-269
//   eval_direct          proj/src/oracle_direct.cpp:41-78
//   exp_add/sub/mul      proj/include/pseval/expansion.hpp:142-211
//   instrumented/reporting_cost  proj/src/multidouble.cpp:60-75
//   flop_count*          proj/src/executor.cpp:233-252
//
// Packed array conventions shared with oracle/pse_oracle.c and the product:
//   P = 2 parts in complex mode (re, im), else 1
//   static block  [P][m][static_top][d+1], static_top = 1 + N + n
//                 (slot 0 = a0, 1+k = a_k, N+i = z_i; executor.cpp:163-165)
//   value/grad    [P][m][n+1][d+1]  row 0 = value, row 1+i = gradient i
//   md values     [count][m] (AoS, one MultiDouble per row)

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pseval/bench.hpp"
#include "pseval/executor.hpp"
#include "pseval/gen.hpp"
#include "pseval/multidouble.hpp"
#include "pseval/oracle.hpp"
#include "pseval/problem_io.hpp"

using namespace pseval;

namespace {

thread_local std::string g_err;

struct RefProblem {
  Problem p;
};

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

int parts(const Polynomial& poly) { return poly.a0.mode == Mode::cplx ? 2 : 1; }

void series_to_block(const Series& s, double* base, long rows, long row) {
  // base points at [P][m][rows][d+1]
  const int d1 = s.degree + 1;
  const int P = s.mode == Mode::cplx ? 2 : 1;
  for (int part = 0; part < P; ++part)
    for (int l = 0; l < s.m; ++l) {
      double* dst = base + ((static_cast<long>(part) * s.m + l) * rows + row) * d1;
      for (int j = 0; j < d1; ++j)
        dst[j] = part == 0 ? s.c[j].re.limb[l] : s.c[j].im.limb[l];
    }
}

Series block_to_series(const double* base, long rows, long row, int d, int m, Mode mode) {
  Series s = make_series(d, m, mode);
  const int P = mode == Mode::cplx ? 2 : 1;
  for (int part = 0; part < P; ++part)
    for (int l = 0; l < m; ++l) {
      const double* src = base + ((static_cast<long>(part) * m + l) * rows + row) * (d + 1);
      for (int j = 0; j <= d; ++j) {
        if (part == 0)
          s.c[j].re.limb[l] = src[j];
        else
          s.c[j].im.limb[l] = src[j];
      }
    }
  return s;
}

void write_vg(const Series& value, const std::vector<Series>& grad, double* out) {
  const long rows = static_cast<long>(grad.size()) + 1;
  series_to_block(value, out, rows, 0);
  for (size_t i = 0; i < grad.size(); ++i) series_to_block(grad[i], out, rows, static_cast<long>(i) + 1);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_problem_gen(const char* id, int d, int m, int cplx, uint64_t seed) {
  try {
    auto* r = new RefProblem;
    r->p = gen_benchmark(id, d, m, cplx ? Mode::cplx : Mode::real, seed);
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// nvars[N], idx[sum nvars] (1-based), exps[sum nvars] or nullptr; a monomial
// whose exponents are all 0 in exps is treated as "no exponents" (empty).
void* ref_problem_new(int n, int d, int m, int cplx, int N, const int* nvars, const int* idx,
                      const int* exps, const double* stat) {
  try {
    const Mode mode = cplx ? Mode::cplx : Mode::real;
    auto* r = new RefProblem;
    Problem& p = r->p;
    p.id = "file";
    p.poly.n = n;
    p.poly.d = d;
    const long top = 1L + N + n;
    p.poly.a0 = block_to_series(stat, top, 0, d, m, mode);
    long pos = 0;
    for (int k = 0; k < N; ++k) {
      Monomial mo;
      bool any = false;
      for (int j = 0; j < nvars[k]; ++j) {
        mo.indices.push_back(idx[pos + j]);
        if (exps && exps[pos + j] != 0) any = true;
      }
      if (any)
        for (int j = 0; j < nvars[k]; ++j) mo.exponents.push_back(exps[pos + j]);
      pos += nvars[k];
      mo.coeff = block_to_series(stat, top, 1 + k, d, m, mode);
      p.poly.monomials.push_back(std::move(mo));
    }
    for (int i = 1; i <= n; ++i) p.z.push_back(block_to_series(stat, top, N + i, d, m, mode));
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_problem_free(void* h) { delete static_cast<RefProblem*>(h); }

// info: n, N, d, m, cplx, total_slots, nconv, nadd, ncopy, nconv_layers,
//       nadd_layers, n_term_scales, shape_len (sum of nvars)
int ref_problem_info(void* h, int64_t* info) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    const JobGraph g = build_jobgraph(p.poly);
    long shape = 0;
    for (auto& mo : p.poly.monomials) shape += static_cast<long>(mo.indices.size());
    int64_t v[] = {p.poly.n, g.N, p.poly.d, p.poly.a0.m, p.poly.a0.mode == Mode::cplx ? 1 : 0,
                   g.total_slots, g.conv_job_count(), g.add_job_count(), g.copy_job_count(),
                   static_cast<int64_t>(g.conv_layers.size()),
                   static_cast<int64_t>(g.add_layers.size()),
                   static_cast<int64_t>(g.term_scales.size()), shape};
    std::memcpy(info, v, sizeof v);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_problem_shape(void* h, int* nvars, int* idx, int* exps) {
  const Problem& p = static_cast<RefProblem*>(h)->p;
  long pos = 0;
  for (size_t k = 0; k < p.poly.monomials.size(); ++k) {
    const Monomial& mo = p.poly.monomials[k];
    nvars[k] = static_cast<int>(mo.indices.size());
    for (size_t j = 0; j < mo.indices.size(); ++j) {
      idx[pos] = mo.indices[j];
      exps[pos] = mo.exponents.empty() ? 0 : mo.exponents[j];
      ++pos;
    }
  }
  return 0;
}

// unfolded static region exactly as the Problem holds it
int ref_problem_static(void* h, double* out) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    const int N = static_cast<int>(p.poly.monomials.size());
    const long top = 1L + N + p.poly.n;
    series_to_block(p.poly.a0, out, top, 0);
    for (int k = 0; k < N; ++k) series_to_block(p.poly.monomials[k].coeff, out, top, 1 + k);
    for (int i = 1; i <= p.poly.n; ++i) series_to_block(p.z[i - 1], out, top, N + i);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// conv: nconv rows of (layer, in1, in2, out, copy); add: nadd rows of
// (layer, src, dst); ts: rows of (slot, factor)
int ref_graph_export(void* h, int64_t* conv, int64_t* add, int64_t* value_slot,
                     int64_t* grad_slots, int64_t* mult, int64_t* ts) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    const JobGraph g = build_jobgraph(p.poly);
    long r = 0;
    for (size_t L = 0; L < g.conv_layers.size(); ++L)
      for (const ConvJob& j : g.conv_layers[L]) {
        int64_t row[] = {j.layer, j.in1, j.in2, j.out, j.copy ? 1 : 0};
        std::memcpy(conv + 5 * r++, row, sizeof row);
      }
    r = 0;
    for (size_t L = 0; L < g.add_layers.size(); ++L)
      for (const AddJob& j : g.add_layers[L]) {
        int64_t row[] = {j.layer, j.src, j.dst};
        std::memcpy(add + 3 * r++, row, sizeof row);
      }
    *value_slot = g.value_slot;
    for (int i = 0; i < g.n; ++i) {
      grad_slots[i] = g.gradient_slots[i];
      mult[i] = g.multipliers[i];
    }
    r = 0;
    for (const TermScale& t : g.term_scales) {
      ts[2 * r] = t.slot;
      ts[2 * r + 1] = t.factor;
      ++r;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// evaluate() (executor.cpp:271-276) with workers (0 = run_sequential).
// dyn_out, if given, receives the full arena [P][m][total_slots][d+1] after the run.
int ref_run(void* h, int workers, double* vg_out, double* dyn_out, double* times /*wall, conv, add*/,
            int64_t* double_ops) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    const JobGraph g = build_jobgraph(p.poly);
    const Polynomial folded = fold_polynomial(p.poly, p.z);
    DataArray a = stage(folded, p.z);
    RunReport rep = workers >= 1 ? run_parallel(g, a, workers) : run_sequential(g, a);
    if (vg_out) write_vg(rep.value, rep.gradient, vg_out);
    if (dyn_out) {
      const long slab = a.total_slots * (a.d + 1);
      for (int l = 0; l < a.m; ++l) std::memcpy(dyn_out + l * slab, a.re[l].data(), slab * sizeof(double));
      if (a.mode == Mode::cplx)
        for (int l = 0; l < a.m; ++l)
          std::memcpy(dyn_out + (a.m + l) * slab, a.im[l].data(), slab * sizeof(double));
    }
    if (times) {
      times[0] = rep.wall_ms;
      times[1] = rep.conv_ms();
      times[2] = rep.add_ms();
    }
    if (double_ops) *double_ops = rep.double_op_count;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_eval_direct(void* h, double* vg_out) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    Evaluation ev = eval_direct(p.poly, p.z);
    write_vg(ev.value, ev.gradient, vg_out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_within_oracle_guard(void* h) {
  return within_oracle_guard(static_cast<RefProblem*>(h)->p.poly) ? 1 : 0;
}

// op: 0 add, 1 sub, 2 mul ; x, y, out: [count][m]
int ref_md_op(int op, int m, int64_t count, const double* x, const double* y, double* out) {
  try {
    check_precision(m);
    for (int64_t c = 0; c < count; ++c) {
      MultiDouble a(m), b(m);
      for (int l = 0; l < m; ++l) {
        a.limb[l] = x[c * m + l];
        b.limb[l] = y[c * m + l];
      }
      MultiDouble r = op == 0 ? md_add(a, b) : op == 1 ? md_sub(a, b) : md_mul(a, b);
      for (int l = 0; l < m; ++l) out[c * m + l] = r.limb[l];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// count random_md values from Rng(seed) (multidouble.cpp:26-30), [count][m]
void ref_random_md(uint64_t seed, int m, int64_t count, double* out) {
  Rng rng(seed);
  for (int64_t c = 0; c < count; ++c) {
    MultiDouble v = random_md(rng, m);
    for (int l = 0; l < m; ++l) out[c * m + l] = v.limb[l];
  }
}

// renormalize (multidouble.cpp:9-24) of an n-term expansion to m limbs
int ref_renormalize(const double* t, int n, int m, double* out) {
  try {
    std::vector<double> v(t, t + n);
    MultiDouble r = renormalize(v, m);
    for (int l = 0; l < m; ++l) out[l] = r.limb[l];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

uint64_t ref_mix_seed(uint64_t base, uint64_t stream) { return mix_seed(base, stream); }

void ref_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
  Rng rng(seed);
  for (int64_t c = 0; c < count; ++c) out[c] = rng.u64();
}

int ref_cost(int m, int64_t* out /* inst_add, inst_mul, rep_add, rep_mul */) {
  try {
    OpCost a = instrumented_cost(m), b = reporting_cost(m);
    out[0] = a.add_cost;
    out[1] = a.mul_cost;
    out[2] = b.add_cost;
    out[3] = b.mul_cost;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// which: 0 total, 1 mul, 2 add  (executor.cpp:233-252)
int64_t ref_flop_count(void* h, int d, int cplx, int64_t add_cost, int64_t mul_cost, int which) {
  const Problem& p = static_cast<RefProblem*>(h)->p;
  const JobGraph g = build_jobgraph(p.poly);
  OpCost c{add_cost, mul_cost};
  Mode mode = cplx ? Mode::cplx : Mode::real;
  if (which == 1) return flop_count_mul(g, d, mode, c);
  if (which == 2) return flop_count_add(g, d, mode, c);
  return flop_count(g, d, mode, c);
}

// Bounded CPU timing sample for the bench's reference arm / cpu_baseline:
// the first `njobs` convolution jobs of conv layer 1 (all inputs static,
// full-precision data, so every job costs what any conv job of the graph
// costs) plus every addition layer, run through the reference's own
// run_parallel (workers >= 1) or run_sequential (workers == 0).
// times: [0] conv ms of the sample, [1] add ms, [2] wall ms
int ref_bench_sample(void* h, int workers, int64_t njobs, double* times) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    JobGraph g = build_jobgraph(p.poly);
    JobGraph s = g;
    s.conv_layers.assign(1, {});
    for (const ConvJob& j : g.conv_layers[0]) {
      if (static_cast<int64_t>(s.conv_layers[0].size()) >= njobs) break;
      if (!j.copy) s.conv_layers[0].push_back(j);
    }
    const Polynomial folded = fold_polynomial(p.poly, p.z);
    DataArray a = stage(folded, p.z);
    RunReport rep = workers >= 1 ? run_parallel(s, a, workers) : run_sequential(s, a);
    times[0] = rep.conv_ms();
    times[1] = rep.add_ms();
    times[2] = rep.wall_ms;
    return static_cast<int>(s.conv_layers[0].size());
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_bench (bench.cpp:17-50): median of `repeats` full runs
int ref_run_bench(void* h, int workers, int repeats, double* out /* conv, add, wall, gflops */) {
  try {
    const Problem& p = static_cast<RefProblem*>(h)->p;
    BenchRecord r = run_bench(p, workers, repeats);
    out[0] = r.conv_ms;
    out[1] = r.add_ms;
    out[2] = r.wall_ms;
    out[3] = r.gflops;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

// problem_to_text (problem_io.cpp:130-157): returns the full length, copies
// at most cap-1 bytes + NUL
int64_t ref_problem_to_text(void* h, char* buf, int64_t cap) {
  const std::string t = problem_to_text(static_cast<RefProblem*>(h)->p);
  if (buf && cap > 0) {
    const int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(t.size()));
    std::memcpy(buf, t.data(), n);
    buf[n] = 0;
  }
  return static_cast<int64_t>(t.size());
}

// problem_from_text (problem_io.cpp:159-245); nullptr + message on ParseError
void* ref_problem_from_text(const char* text) {
  try {
    auto* r = new RefProblem;
    r->p = problem_from_text(text);
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

}  // extern "C"
