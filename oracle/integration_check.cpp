// TEST INFRASTRUCTURE ONLY. Drop-in check of the reference-side binding
// (include/pse_b200_pseval.hpp): the UNMODIFIED reference engine's own types
// and run_sequential next to run_device over the B200 C ABI, compared bit for
// bit on the reference's DataArray (value, every gradient, the whole arena).
// Built by oracle/Makefile into oracle/_ref/integration_check (needs the
// reference sources); run by tests/test_gpu_parity.py on a GPU box.
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
  (void)argc;
  (void)argv;
  return bad;
}
