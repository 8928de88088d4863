// pseval_b200: the reference CLI (proj/tools/pseval.cpp:128-282) over the
// B200 engine. Subcommands and options follow the reference:
//
//   pseval_b200 gen <p1|p2|p3> <out> [--degree D] [--precision M] [--mode real|complex] [--seed S]
//   pseval_b200 verify <id|file> [--degree D] [--precision M] [--mode ..] [--seed S] [--device G]
//                      [--oracle auto|on|off]
//   pseval_b200 bench [id|file] [--degree D ...] [--precision M ...] [--mode ..] [--seed S]
//                     [--repeats R] [--csv FILE] [--device G]
//   pseval_b200 graph-stats <id|file> [--degree D] [--precision M] [--mode ..] [--seed S]
//
// verify cross-checks the device engine's execution paths bit for bit
// (layered fused vs split convolutions, the dataflow and banded-wave
// schedules, a batch of points vs single evaluations) -- the device analogue
// of the reference's sequential-vs-parallel check (pseval.cpp:76-95) -- and
// the engine against an independent device evaluator (eval_direct,
// oracle_direct.cpp:41-78) within the reference's tolerance (pseval.cpp:97-118).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pse_b200.h"

namespace {

void check(int rc) {
  if (rc < 0) throw std::runtime_error(pse_last_error());
}

struct Args {
  std::string cmd;
  std::vector<std::string> pos;
  std::vector<int> degrees, precisions;
  std::string mode = "real", csv, oracle = "auto";
  uint64_t seed = 7;
  int repeats = 3, device = 0;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw std::invalid_argument("usage: pseval_b200 <gen|verify|bench|graph-stats> ...");
  a.cmd = argv[1];
  std::vector<int>* sweep = nullptr;  // bench: "--degree 8 15 31" extends the sweep
  for (int i = 2; i < argc; ++i) {
    const std::string s = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for " + s);
      return argv[++i];
    };
    if (sweep && a.cmd == "bench" && !s.empty() && std::isdigit(static_cast<unsigned char>(s[0]))) {
      sweep->push_back(std::stoi(s));
      continue;
    }
    sweep = nullptr;
    if (s == "--degree") {
      a.degrees.push_back(std::stoi(val()));
      sweep = &a.degrees;
    } else if (s == "--precision") {
      a.precisions.push_back(std::stoi(val()));
      sweep = &a.precisions;
    } else if (s == "--mode") {
      a.mode = val();
      if (a.mode != "real" && a.mode != "complex") throw std::invalid_argument("--mode must be real or complex");
    } else if (s == "--seed") {
      a.seed = std::stoull(val());
    } else if (s == "--repeats") {
      a.repeats = std::max(1, std::stoi(val()));
    } else if (s == "--csv") {
      a.csv = val();
    } else if (s == "--oracle") {
      a.oracle = val();
      if (a.oracle != "auto" && a.oracle != "on" && a.oracle != "off")
        throw std::invalid_argument("--oracle must be auto, on or off");
    } else if (s == "--device") {
      a.device = std::stoi(val());
    } else if (s.size() > 1 && s[0] == '-') {
      throw std::invalid_argument("unknown option " + s);
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

bool known_id(const std::string& t) { return t == "p1" || t == "p2" || t == "p3"; }

struct Prob {
  pse_problem* h = nullptr;
  ~Prob() { pse_problem_destroy(h); }
  int64_t info[7];
  const int32_t *nv, *ix, *ex;
  const double* st;
  std::string id;
  void load() {
    check(pse_problem_info(h, info));
    check(pse_problem_arrays(h, &nv, &ix, &ex, &st));
    char buf[128];
    check(pse_problem_id(h, buf, sizeof buf));
    id = buf;
  }
  int n() const { return static_cast<int>(info[0]); }
  int N() const { return static_cast<int>(info[1]); }
  int d() const { return static_cast<int>(info[2]); }
  int m() const { return static_cast<int>(info[3]); }
  int mode() const { return static_cast<int>(info[4]); }
  int Q() const { return (mode() ? 2 : 1) * m(); }
};

void load_target(Prob& p, const std::string& target, int d, int m, int mode, uint64_t seed) {
  if (known_id(target))
    check(pse_problem_gen(target.c_str(), d, m, mode, seed, &p.h));
  else
    check(pse_problem_read(target.c_str(), &p.h));
  p.load();
}

struct Graph {
  pse_graph* g = nullptr;
  pse_graph_desc desc{};
  ~Graph() { pse_graph_destroy(g); }
};

void build(const Prob& p, Graph& G) {
  check(pse_graph_build(p.n(), p.d(), p.N(), p.nv, p.ix, p.ex, &G.g));
  check(pse_graph_describe(G.g, p.m(), p.mode(), &G.desc));
}

// graph_stats_text (bench.cpp:52-75)
std::string graph_stats(const Prob& p, const Graph& G) {
  const pse_graph_desc& g = G.desc;
  std::string out = "problem " + p.id + ": n=" + std::to_string(g.n) + " N=" + std::to_string(g.N) +
                    " d=" + std::to_string(g.d) + " m=" + std::to_string(p.m()) +
                    " mode=" + (p.mode() ? "complex" : "real") + "\n";
  out += "slots: " + std::to_string(g.total_slots) + " (" + std::to_string(g.total_slots * (g.d + 1)) +
         " doubles per slab)\n";
  const int64_t nc = g.conv_layer_off[g.n_conv_layers], na = g.add_layer_off[g.n_add_layers];
  int64_t copies = 0;
  for (int64_t t = 0; t < nc; ++t) copies += g.conv_copy[t];
  out += "conv jobs: " + std::to_string(nc) + " in " + std::to_string(g.n_conv_layers) + " layers:";
  for (int L = 0; L < g.n_conv_layers; ++L) out += ' ' + std::to_string(g.conv_layer_off[L + 1] - g.conv_layer_off[L]);
  out += "\nadd jobs: " + std::to_string(na) + " in " + std::to_string(g.n_add_layers) + " layers:";
  for (int L = 0; L < g.n_add_layers; ++L) out += ' ' + std::to_string(g.add_layer_off[L + 1] - g.add_layer_off[L]);
  out += '\n';
  if (copies > 0) out += "copy jobs: " + std::to_string(copies) + " (included in the conv total)\n";
  if (p.id == "p3")
    out += "note: the conv total " + std::to_string(nc) + " counts 3 jobs per two-variable monomial and differs from the " +
           std::to_string(na) + " quoted for it in some references\n";
  return out;
}

// one device evaluation of `batch` copies-or-points; returns vg [Q][batch][n+1][d+1]
std::vector<double> eval(const Prob& p, const std::vector<double>& stat, int batch, int device, pse_report* rep) {
  std::vector<double> vg(static_cast<size_t>(p.Q()) * batch * (p.n() + 1) * (p.d() + 1));
  check(pse_evaluate(p.n(), p.d(), p.m(), p.mode(), p.N(), p.nv, p.ix, p.ex, batch, stat.data(), vg.data(), device, rep));
  return vg;
}

// one device evaluation with the conv path forced through the planner's knobs
// (PSE_CONV_MODE / PSE_SPLIT_THRESHOLD are read at plan creation)
std::vector<double> eval_path(const Prob& p, const std::vector<double>& stat, int batch, int device, const char* mode,
                              const char* split) {
  if (mode) setenv("PSE_CONV_MODE", mode, 1); else unsetenv("PSE_CONV_MODE");
  if (split) setenv("PSE_SPLIT_THRESHOLD", split, 1); else unsetenv("PSE_SPLIT_THRESHOLD");
  pse_report rep{};
  std::vector<double> vg = eval(p, stat, batch, device, &rep);
  unsetenv("PSE_CONV_MODE");
  unsetenv("PSE_SPLIT_THRESHOLD");
  return vg;
}

// PSE_VERIFY_PERTURB=<path> (testing verify itself): flip the lowest bit of
// the last limb of value coefficient 0 in that path's result -- "oracle"
// perturbs every path by a relative 1e-6 instead
void perturb(std::vector<double>& vg, const char* path, const Prob& p) {
  const char* e = getenv("PSE_VERIFY_PERTURB");
  if (!e) return;
  if (std::string(e) == "oracle") {
    vg[0] += std::fabs(vg[0]) * 1e-6 + 1e-300;
    return;
  }
  if (std::string(e) != path) return;
  const size_t at = static_cast<size_t>(p.m() - 1) * (p.n() + 1) * (p.d() + 1);  // limb m-1, value, coeff 0
  uint64_t b;
  std::memcpy(&b, &vg[at], 8);
  b ^= 1;
  std::memcpy(&vg[at], &b, 8);
}

// oracle_cost_estimate (pseval.cpp:55-66): the auto mode skips the oracle above 1e6
int64_t oracle_cost_estimate(const Prob& p) {
  int64_t q = 1, pos = 0;
  for (int k = 0; k < p.N(); ++k) {
    int64_t t = 0;
    bool has = false;
    if (p.ex)
      for (int j = 0; j < p.nv[k]; ++j) has = has || p.ex[pos + j] != 0;
    for (int j = 0; j < p.nv[k]; ++j) t += has ? p.ex[pos + j] : 1;
    q = std::max(q, t);
    pos += p.nv[k];
  }
  const int64_t len = p.d() + 1;
  return static_cast<int64_t>(p.N()) * q * q * len * len * p.m() * p.m();
}

double md_to_double(const double* limbs, int m, size_t stride) {  // multidouble.hpp:65-69
  double s = 0.0;
  for (int i = m - 1; i >= 0; --i) s += limbs[static_cast<size_t>(i) * stride];
  return s;
}

// do_verify (pseval.cpp:70-118) over the device engine. The reference
// compares its sequential and parallel engines bit for bit, then both with
// eval_direct; here the engine's distinct device paths are compared bit for
// bit -- layered fused vs layered split convolutions, the dataflow and the
// banded-wave schedules vs layered, the two CTA-local forms (band-task
// dataflow, layer walk) vs layered, the planner's own pick, a batch vs one
// point -- and the engine with the independent device evaluator
// (pse_eval_direct: direct product chains, literal md arithmetic) within the
// reference's tolerance 2^(32-52m) * max(1, |ref|).
int do_verify(const Prob& p, int device, const std::string& oracle_flag) {
  std::printf("problem %s: n=%d N=%d d=%d m=%d mode=%s\n", p.id.c_str(), p.n(), p.N(), p.d(), p.m(),
              p.mode() ? "complex" : "real");
  const size_t rows = 1 + static_cast<size_t>(p.N()) + p.n();
  const size_t pw = rows * (p.d() + 1);
  std::vector<double> one(p.st, p.st + static_cast<size_t>(p.Q()) * pw);
  const char* huge = "4611686018427387904";
  std::vector<double> fused = eval_path(p, one, 1, device, "layer", "0");
  std::vector<double> split = eval_path(p, one, 1, device, "layer", huge);
  std::vector<double> flow = eval_path(p, one, 1, device, "flow", nullptr);
  std::vector<double> waves = eval_path(p, one, 1, device, "band", nullptr);
  std::vector<double> cta = eval_path(p, one, 1, device, "cta", nullptr);
  std::vector<double> ctl = eval_path(p, one, 1, device, "ctl", nullptr);
  std::vector<double> autop = eval_path(p, one, 1, device, nullptr, nullptr);
  perturb(fused, "fused", p);
  perturb(cta, "cta", p);
  perturb(ctl, "ctl", p);
  perturb(split, "split", p);
  perturb(flow, "flow", p);
  perturb(waves, "band", p);
  perturb(autop, "auto", p);
  // batch of 3 identical points, [Q][3][rows][d+1]
  std::vector<double> three(static_cast<size_t>(p.Q()) * 3 * pw);
  for (int q = 0; q < p.Q(); ++q)
    for (int b = 0; b < 3; ++b) std::memcpy(&three[(q * 3 + b) * pw], &one[q * pw], pw * sizeof(double));
  const std::vector<double> batched = eval_path(p, three, 3, device, nullptr, nullptr);
  const size_t vw = static_cast<size_t>(p.n() + 1) * (p.d() + 1);
  auto same = [](const std::vector<double>& x, const std::vector<double>& y) {
    return x.size() == y.size() && std::memcmp(x.data(), y.data(), x.size() * sizeof(double)) == 0;
  };
  bool ok = true;
  auto report = [&](const char* what, bool eq) {
    std::printf("engines: %s: %s\n", what, eq ? "bitwise equal" : "MISMATCH");
    ok = ok && eq;
  };
  report("layered fused vs layered split convolutions", same(fused, split));
  report("dataflow (banded, one persistent launch) vs layered", same(flow, fused));
  report("banded waves vs layered", same(waves, fused));
  report("CTA-local dataflow vs layered", same(cta, fused));
  report("CTA-local layers vs layered", same(ctl, fused));
  report("planner's path vs layered", same(autop, fused));
  bool batch_ok = true;
  for (int q = 0; q < p.Q(); ++q)
    for (int b = 0; b < 3; ++b)
      batch_ok = batch_ok && std::memcmp(&batched[(q * 3 + b) * vw], &autop[q * vw], vw * sizeof(double)) == 0;
  report("batch of 3 points vs single point", batch_ok);

  bool oracle_ok = true;
  if (oracle_flag == "off") {
    std::printf("oracle: skipped (disabled)\n");
  } else if (oracle_flag == "auto" && oracle_cost_estimate(p) > 1000000) {
    std::printf("oracle: skipped (instance too large for auto mode; --oracle on forces it)\n");
  } else if (pse_within_oracle_guard(p.d(), p.N(), p.nv, p.ex) != 1) {
    std::printf("oracle: refused, instance exceeds the direct-evaluation size guard\n");
    return 2;
  } else {
    std::vector<double> ref(static_cast<size_t>(p.Q()) * vw);
    check(pse_eval_direct(p.n(), p.d(), p.m(), p.mode(), p.N(), p.nv, p.ix, p.ex, one.data(), ref.data(), device));
    // series_gap / series_norm (pseval.cpp:35-53): md_to_double(md_sub(x, y)),
    // the subtraction in the same md arithmetic (on the device)
    const int m = p.m(), P = p.mode() ? 2 : 1;
    const size_t cnt = static_cast<size_t>(P) * vw;
    std::vector<double> x(cnt * m), y(cnt * m), diff(cnt * m);
    for (int part = 0; part < P; ++part)
      for (size_t r = 0; r < vw; ++r)
        for (int l = 0; l < m; ++l) {
          const size_t src = (static_cast<size_t>(part) * m + l) * vw + r, dst = (part * vw + r) * m + l;
          x[dst] = autop[src];
          y[dst] = ref[src];
        }
    check(pse_md_apply(1, m, 1, static_cast<int64_t>(cnt), x.data(), y.data(), diff.data(), device));
    double norm = 1.0, gap = 0.0;
    for (size_t c = 0; c < cnt; ++c) {
      norm = std::max(norm, std::fabs(md_to_double(&y[c * m], m, 1)));
      gap = std::max(gap, std::fabs(md_to_double(&diff[c * m], m, 1)));
    }
    const double tol = std::ldexp(1.0, 32 - 52 * m);
    const double rel = gap / norm;
    oracle_ok = rel <= tol;
    std::printf("oracle: independent device evaluator (direct product chains, literal md arithmetic): max "
                "coefficient discrepancy %.3e relative (tolerance %.3e): %s\n",
                rel, tol, oracle_ok ? "ok" : "MISMATCH");
  }
  const bool pass = ok && oracle_ok;
  std::printf("verify: %s\n", pass ? "PASS" : "FAIL");
  return pass ? 0 : 1;
}

struct Row {
  std::string id;
  int d, m, mode;
  int64_t conv_jobs, add_jobs;
  double conv_ms, add_ms, wall_ms;
  int64_t ops;
  double gflops;
};

// run_bench (bench.cpp:17-50) on the device: median of `repeats` by wall time
Row bench_one(const Prob& p, int repeats, int device) {
  Graph G;
  build(p, G);
  pse_plan* plan = nullptr;
  check(pse_plan_create(&G.desc, device, 1, &plan));
  const size_t pw = (1 + static_cast<size_t>(p.N()) + p.n()) * (p.d() + 1);
  std::vector<const double*> slabs(p.Q());
  for (int q = 0; q < p.Q(); ++q) slabs[q] = p.st + q * pw;
  check(pse_plan_upload(plan, 1, slabs.data(), 0));
  std::vector<pse_report> reps(repeats);
  pse_report warm{};
  check(pse_plan_execute(plan, 1, 1, &warm));
  for (int r = 0; r < repeats; ++r) check(pse_plan_execute(plan, 1, 1, &reps[r]));
  pse_plan_destroy(plan);
  std::sort(reps.begin(), reps.end(), [](const pse_report& a, const pse_report& b) { return a.wall_ms < b.wall_ms; });
  const pse_report& mid = reps[(reps.size() - 1) / 2];
  Row row{p.id, p.d(), p.m(), p.mode(), mid.conv_jobs_executed, mid.add_jobs_executed, mid.conv_ms, mid.add_ms,
          mid.wall_ms, mid.double_op_count, 0.0};
  row.gflops = mid.wall_ms > 0 ? static_cast<double>(mid.double_op_count) / (mid.wall_ms * 1e6) : 0.0;
  return row;
}

// bench_markdown_row (bench.cpp:82-96); the workers column reports the device
std::string md_row(const Row& r, int device) {
  char buf[256];
  std::snprintf(buf, sizeof buf, "| %s | %d | %d | %s | gpu%d | %.3f | %.3f | %.3f | %.3f | %.3f |\n", r.id.c_str(), r.d,
                r.m, r.mode ? "complex" : "real", device, r.conv_ms, r.add_ms, r.conv_ms + r.add_ms, r.wall_ms,
                r.gflops);
  return buf;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    Args a = parse(argc, argv);
    const int mode = a.mode == "complex" ? PSE_MODE_COMPLEX : PSE_MODE_REAL;
    const int d0 = a.degrees.empty() ? 8 : a.degrees.front();
    const int m0 = a.precisions.empty() ? 2 : a.precisions.front();
    if (a.cmd == "gen") {
      if (a.pos.size() != 2) throw std::invalid_argument("usage: pseval_b200 gen <id> <out> [options]");
      if (!known_id(a.pos[0])) throw std::runtime_error("unknown benchmark id '" + a.pos[0] + "'");
      Prob p;
      load_target(p, a.pos[0], d0, m0, mode, a.seed);
      check(pse_problem_write(p.h, a.pos[1].c_str()));
      std::printf("wrote %s: %s n=%d N=%d d=%d m=%d mode=%s seed=%llu\n", a.pos[1].c_str(), p.id.c_str(), p.n(), p.N(),
                  p.d(), p.m(), a.mode.c_str(), static_cast<unsigned long long>(a.seed));
      return 0;
    }
    if (a.cmd == "verify") {
      if (a.pos.size() != 1) throw std::invalid_argument("usage: pseval_b200 verify <id|file> [options]");
      Prob p;
      load_target(p, a.pos[0], d0, m0, mode, a.seed);
      return do_verify(p, a.device, a.oracle);
    }
    if (a.cmd == "graph-stats") {
      if (a.pos.size() != 1) throw std::invalid_argument("usage: pseval_b200 graph-stats <id|file> [options]");
      Prob p;
      load_target(p, a.pos[0], d0, m0, mode, a.seed);
      Graph G;
      build(p, G);
      std::fputs(graph_stats(p, G).c_str(), stdout);
      return 0;
    }
    if (a.cmd == "bench") {
      const std::string target = a.pos.empty() ? "p1" : a.pos[0];
      const bool sweep_default = a.degrees.empty();
      std::vector<int> degrees = a.degrees;
      if (degrees.empty()) degrees = {0, 8, 15, 31, 63, 95, 127, 152, 159, 191};  // pseval.cpp:133
      std::vector<int> precisions = a.precisions.empty() ? std::vector<int>{2} : a.precisions;
      std::vector<Row> rows;
      const char* header =
          "| id | d | m | mode | workers | cnv ms | add ms | sum ms | wall ms | Gflop/s |\n"
          "|---|---:|---:|---|---:|---:|---:|---:|---:|---:|\n";
      if (known_id(target)) {
        {
          Prob p;
          load_target(p, target, degrees.front(), precisions.front(), mode, a.seed);
          Graph G;
          build(p, G);
          std::fputs(graph_stats(p, G).c_str(), stdout);
        }
        std::printf("\n%s", header);
        for (int m : precisions)
          for (int d : degrees) {
            if (sweep_default && m == 10 && d > 152) continue;  // pseval.cpp:255
            Prob p;
            load_target(p, target, d, m, mode, a.seed);
            rows.push_back(bench_one(p, a.repeats, a.device));
            std::fputs(md_row(rows.back(), a.device).c_str(), stdout);
            std::fflush(stdout);
          }
      } else {
        Prob p;
        load_target(p, target, 0, 1, mode, a.seed);
        Graph G;
        build(p, G);
        std::fputs(graph_stats(p, G).c_str(), stdout);
        std::printf("\n%s", header);
        rows.push_back(bench_one(p, a.repeats, a.device));
        std::fputs(md_row(rows.back(), a.device).c_str(), stdout);
      }
      if (!a.csv.empty()) {
        std::ofstream f(a.csv, std::ios::binary);
        if (!f) throw std::runtime_error("cannot open '" + a.csv + "' for writing");
        f << "id,d,m,mode,workers,conv_jobs,add_jobs,conv_ms,add_ms,sum_ms,wall_ms,double_ops,gflops\n";
        for (const Row& r : rows) {
          char buf[256];
          std::snprintf(buf, sizeof buf, "%s,%d,%d,%s,gpu%d,%lld,%lld,%.6f,%.6f,%.6f,%.6f,%lld,%.6f\n", r.id.c_str(), r.d,
                        r.m, r.mode ? "complex" : "real", a.device, static_cast<long long>(r.conv_jobs),
                        static_cast<long long>(r.add_jobs), r.conv_ms, r.add_ms, r.conv_ms + r.add_ms, r.wall_ms,
                        static_cast<long long>(r.ops), r.gflops);
          f << buf;
        }
        std::printf("wrote %zu rows to %s\n", rows.size(), a.csv.c_str());
      }
      return 0;
    }
    throw std::invalid_argument("unknown subcommand '" + a.cmd + "' (gen, verify, bench, graph-stats)");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
