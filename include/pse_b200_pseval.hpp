// Reference-side binding: the adapter a pseval maintainer adds to switch the
// engine behind evaluate() to the B200 device. Header-only; include it after
// the reference's own headers and link libpse_b200.so.
//
//   #include "pseval/executor.hpp"   // /root/reference/proj/include
//   #include "pse_b200_pseval.hpp"   // this file
//   ...
//   RunReport r = pseval::run_device(g, a);   // drop-in for run_sequential(g, a)
//
// run_device keeps run_sequential's contract (executor.hpp:49,
// executor.cpp:168-183): it reads the static region of the DataArray, writes
// the whole dynamic region back in place, and returns value + gradient
// (extract, executor.cpp:254-269) with the reporting-cost double_op_count.
// Failures surface as std::invalid_argument (PSE_EINVAL) like the reference,
// std::runtime_error otherwise.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pse_b200.h"
#include "pseval/bench.hpp"     // the reference's own headers (proj/include)
#include "pseval/executor.hpp"
#include "pseval/gen.hpp"

namespace pseval {

struct DeviceOptions {
  int device = 0;
};

namespace b200_detail {

inline void check(int rc) {
  if (rc == PSE_EINVAL) throw std::invalid_argument(pse_last_error());
  if (rc < 0) throw std::runtime_error(std::string("pse_b200: ") + pse_last_error());
}

// JobGraph (jobgraph.hpp:75-90) -> flat arrays that back a pse_graph_desc
struct FlatGraph {
  std::vector<int64_t> conv_off{0}, c1, c2, co, add_off{0}, as, ad, ts_s, ts_f;
  std::vector<uint8_t> cc;
  pse_graph_desc desc{};

  FlatGraph(const JobGraph& g, int m, Mode mode) {
    for (const auto& layer : g.conv_layers) {
      for (const ConvJob& j : layer) {
        c1.push_back(j.in1);
        c2.push_back(j.in2);
        co.push_back(j.out);
        cc.push_back(j.copy ? 1 : 0);
      }
      conv_off.push_back(static_cast<int64_t>(c1.size()));
    }
    for (const auto& layer : g.add_layers) {
      for (const AddJob& j : layer) {
        as.push_back(j.src);
        ad.push_back(j.dst);
      }
      add_off.push_back(static_cast<int64_t>(as.size()));
    }
    for (const TermScale& t : g.term_scales) {
      ts_s.push_back(t.slot);
      ts_f.push_back(t.factor);
    }
    desc.n = g.n;
    desc.N = g.N;
    desc.d = g.d;
    desc.m = m;
    desc.mode = mode == Mode::cplx ? PSE_MODE_COMPLEX : PSE_MODE_REAL;
    desc.total_slots = g.total_slots;
    desc.value_slot = g.value_slot;
    desc.gradient_slots = reinterpret_cast<const int64_t*>(g.gradient_slots.data());
    desc.multipliers = reinterpret_cast<const int64_t*>(g.multipliers.data());
    desc.n_conv_layers = static_cast<int32_t>(g.conv_layers.size());
    desc.conv_layer_off = conv_off.data();
    desc.conv_in1 = c1.data();
    desc.conv_in2 = c2.data();
    desc.conv_out = co.data();
    desc.conv_copy = cc.data();
    desc.n_add_layers = static_cast<int32_t>(g.add_layers.size());
    desc.add_layer_off = add_off.data();
    desc.add_src = as.data();
    desc.add_dst = ad.data();
    desc.n_term_scales = static_cast<int64_t>(ts_s.size());
    desc.ts_slot = ts_s.data();
    desc.ts_factor = ts_f.data();
  }
};

inline Series read_row(const std::vector<double>& vg, int rows, int row, int d, int m, Mode mode) {
  Series s = make_series(d, m, mode);
  const int P = mode == Mode::cplx ? 2 : 1;
  for (int part = 0; part < P; ++part)
    for (int l = 0; l < m; ++l)
      for (int j = 0; j <= d; ++j) {
        const double v = vg[((static_cast<size_t>(part) * m + l) * rows + row) * (d + 1) + j];
        if (part == 0)
          s.c[j].re.limb[l] = v;
        else
          s.c[j].im.limb[l] = v;
      }
  return s;
}

}  // namespace b200_detail

// drop-in for run_sequential / run_parallel (executor.hpp:49-52)
inline RunReport run_device(const JobGraph& g, DataArray& a, const DeviceOptions& opt = {}) {
  static_assert(sizeof(long) == sizeof(int64_t), "JobGraph slots are long");
  b200_detail::FlatGraph fg(g, a.m, a.mode);
  pse_plan* plan = nullptr;
  b200_detail::check(pse_plan_create(&fg.desc, opt.device, 1, &plan));
  const int P = a.mode == Mode::cplx ? 2 : 1;
  const int Q = P * a.m;
  const int rows = g.n + 1;
  std::vector<const double*> in(Q);
  std::vector<double*> dyn(Q), out(Q);
  std::vector<double> vg(static_cast<size_t>(Q) * rows * (a.d + 1));
  for (int q = 0; q < Q; ++q) {
    std::vector<double>& slab = q < a.m ? a.re[q] : a.im[q - a.m];
    in[q] = slab.data();
    dyn[q] = slab.data();  // the dynamic region is written back in place
    out[q] = vg.data() + static_cast<size_t>(q) * rows * (a.d + 1);
  }
  pse_report rep{};
  RunReport r;
  // per-phase times (executor.cpp:154-157): one entry per conv / add layer
  r.conv_layer_ms.assign(g.conv_layers.size(), 0.0);
  r.add_layer_ms.assign(g.add_layers.size(), 0.0);
  int rc = pse_plan_run(plan, 1, in.data(), a.total_slots * (a.d + 1), dyn.data(), out.data(), &rep);
  if (rc == PSE_OK)
    rc = pse_plan_layer_ms(plan, r.conv_layer_ms.data(), static_cast<int32_t>(r.conv_layer_ms.size()),
                           r.add_layer_ms.data(), static_cast<int32_t>(r.add_layer_ms.size()));
  pse_plan_destroy(plan);
  b200_detail::check(rc);
  r.value = b200_detail::read_row(vg, rows, 0, a.d, a.m, a.mode);
  for (int i = 0; i < g.n; ++i) r.gradient.push_back(b200_detail::read_row(vg, rows, 1 + i, a.d, a.m, a.mode));
  r.wall_ms = rep.wall_ms;
  r.double_op_count = rep.double_op_count;
  r.conv_jobs_executed = static_cast<long>(rep.conv_jobs_executed);
  r.add_jobs_executed = static_cast<long>(rep.add_jobs_executed);
  return r;
}

// run_bench (bench.cpp:17-50) with run_device in place of run_parallel /
// run_sequential -- the one-line engine switch INTEGRATION.md describes: same
// graph, fold, stage, median-of-repeats record, conv_ms / add_ms from the
// RunReport's per-layer lists
inline BenchRecord run_bench_device(const Problem& p, int repeats, const DeviceOptions& opt = {}) {
  if (repeats < 1) repeats = 1;
  const JobGraph g = build_jobgraph(p.poly);
  const Polynomial folded = fold_polynomial(p.poly, p.z);
  std::vector<RunReport> runs;
  for (int r = 0; r < repeats; ++r) {
    DataArray a = stage(folded, p.z);
    runs.push_back(run_device(g, a, opt));
  }
  std::vector<size_t> order(runs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return runs[x].wall_ms < runs[y].wall_ms; });
  const RunReport& mid = runs[order[(order.size() - 1) / 2]];
  BenchRecord rec;
  rec.id = p.id;
  rec.d = p.poly.d;
  rec.m = p.poly.a0.m;
  rec.mode = p.poly.a0.mode;
  rec.workers = 0;
  rec.conv_jobs = g.conv_job_count();
  rec.add_jobs = g.add_job_count();
  rec.conv_ms = mid.conv_ms();
  rec.add_ms = mid.add_ms();
  rec.sum_ms = rec.conv_ms + rec.add_ms;
  rec.wall_ms = mid.wall_ms;
  rec.double_ops = mid.double_op_count;
  rec.gflops = mid.wall_ms > 0 ? static_cast<double>(mid.double_op_count) / (mid.wall_ms * 1e6) : 0.0;
  return rec;
}

// evaluate (executor.cpp:271-276) with the device engine
inline RunReport evaluate_device(const Polynomial& poly, const std::vector<Series>& z, const DeviceOptions& opt = {}) {
  JobGraph g = build_jobgraph(poly);
  Polynomial folded = fold_polynomial(poly, z);
  DataArray a = stage(folded, z);
  return run_device(g, a, opt);
}

}  // namespace pseval
