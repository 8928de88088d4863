// TEST INFRASTRUCTURE ONLY. Drop-in check of the reference-side binding
// (include/pse_b200_pseval.hpp): the UNMODIFIED reference engine's own types
// and run_sequential next to run_device over the B200 C ABI, compared bit for
// bit on the reference's DataArray (value, every gradient, the whole arena).
// Built by oracle/Makefile into oracle/_ref/integration_check (needs the
// reference sources); run by tests/test_gpu_parity.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "pse_b200_pseval.hpp"
#include "pseval/executor.hpp"
#include "pseval/gen.hpp"

using namespace pseval;

static bool same(const std::vector<double>& x, const std::vector<double>& y) {
  return x.size() == y.size() && std::memcmp(x.data(), y.data(), x.size() * sizeof(double)) == 0;
}

int main(int argc, char** argv) {
  int bad = 0, runs = 0;
  struct Cfg {
    const char* id;
    int d, m;
    Mode mode;
  } cfgs[] = {{"p1", 15, 2, Mode::real}, {"p1", 8, 10, Mode::real}, {"p3", 3, 3, Mode::cplx}, {"p2", 2, 5, Mode::real}};
  for (const Cfg& c : cfgs) {
    const Problem p = gen_benchmark(c.id, c.d, c.m, c.mode, 7);
    const JobGraph g = build_jobgraph(p.poly);
    DataArray as = stage(p.poly, p.z), ad = stage(p.poly, p.z);
    const RunReport rs = run_sequential(g, as);
    const RunReport rd = run_device(g, ad);
    bool ok = series_bitwise_equal(rs.value, rd.value) && rs.double_op_count == rd.double_op_count;
    for (int i = 0; i < p.poly.n; ++i) ok = ok && series_bitwise_equal(rs.gradient[i], rd.gradient[i]);
    for (int l = 0; l < as.m; ++l) ok = ok && same(as.re[l], ad.re[l]);
    for (size_t l = 0; l < as.im.size(); ++l) ok = ok && same(as.im[l], ad.im[l]);
    std::printf("%s %s d=%d m=%d: run_device %s run_sequential (%.3f ms device)\n", c.id,
                c.mode == Mode::cplx ? "complex" : "real", c.d, c.m, ok ? "==" : "!=", rd.wall_ms);
    bad += ok ? 0 : 1;
    ++runs;
  }
  std::printf("%s: %d/%d configurations bitwise identical\n", bad ? "FAIL" : "OK", runs - bad, runs);

  // RunReport timings through the drop-in: the reference's run_bench
  // (bench.cpp:17-50) with run_device as its engine. conv_ms()/add_ms() sum
  // the per-layer lists (executor.cpp:154-157, one entry per layer) and,
  // with the (empty) scale phase, account for wall_ms.
  int tbad = 0;
  for (const Cfg& c : {Cfg{"p1", 15, 2, Mode::real}, Cfg{"p3", 40, 4, Mode::real}}) {
    const Problem p = gen_benchmark(c.id, c.d, c.m, c.mode, 7);
    const JobGraph g = build_jobgraph(p.poly);
    DataArray a = stage(p.poly, p.z);
    const RunReport r = run_device(g, a);
    const BenchRecord b = run_bench_device(p, 3);
    const bool lists = r.conv_layer_ms.size() == g.conv_layers.size() && r.add_layer_ms.size() == g.add_layers.size();
    const bool pos = b.conv_ms > 0 && b.add_ms > 0 && b.wall_ms > 0;
    const double gap = std::fabs(b.conv_ms + b.add_ms - b.wall_ms) / b.wall_ms;
    const bool ok = lists && pos && gap <= 0.01;
    std::printf("run_bench via run_device %s d=%d m=%d: conv %.4f ms + add %.4f ms vs wall %.4f ms (%zu + %zu layers) %s\n",
                c.id, c.d, c.m, b.conv_ms, b.add_ms, b.wall_ms, r.conv_layer_ms.size(), r.add_layer_ms.size(),
                ok ? "ok" : "BAD");
    tbad += ok ? 0 : 1;
  }
  std::printf("%s: RunReport per-layer timings\n", tbad ? "FAIL" : "OK");
  bad += tbad;
  (void)argc;
  (void)argv;
  return bad;
}
