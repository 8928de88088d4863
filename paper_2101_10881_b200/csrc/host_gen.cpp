// Benchmark input generator, bit-identical to the reference gen_benchmark
// (proj/src/gen.cpp:13-71) with its seeded RNG (rng.hpp:11-36) and
// random_md / renormalize (multidouble.cpp:9-30).
//
// This is host-side input preparation (not timed, like the reference's
// staging), so it carries a small scalar renormalisation of its own. It MUST
// be compiled with -ffp-contract=off (see build.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host_graph.hpp"

namespace pse {
namespace {

// splitmix64 stream derivation (rng.hpp:31-36)
uint64_t mix_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// [-1, 1) with the explicit 53-bit mapping (rng.hpp:22)
double pm1(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1p-52 - 1.0; }

void two_sum(double a, double b, double& s, double& e) {
  const double ss = a + b;
  const double bv = ss - a;
  e = (a - (ss - bv)) + (b - bv);
  s = ss;
}

bool normalized(const double* v, int m) {
  int last = -1;
  bool zero_seen = false;
  for (int i = 0; i < m; ++i) {
    if (v[i] == 0.0) {
      zero_seen = true;
      continue;
    }
    if (zero_seen || !std::isfinite(v[i])) return false;
    if (last >= 0) {
      const int e = std::ilogb(v[last]);
      if (std::fabs(v[i]) > 0.5 * std::ldexp(1.0, std::max(e - 52, -1074))) return false;
    }
    last = i;
  }
  return true;
}

// renormalize of an m-term expansion to m limbs (multidouble.cpp:9-24)
void renorm(double* t, int m, double* out) {
  if (normalized(t, m)) {
    std::memcpy(out, t, sizeof(double) * m);
    return;
  }
  for (int pass = 0; pass < 2; ++pass) {
    double s = t[m - 1];
    for (int i = m - 2; i >= 0; --i) {
      double e;
      two_sum(t[i], s, s, e);
      t[i + 1] = e;
    }
    t[0] = s;
  }
  int j = 0;
  double eps = t[0];
  bool full = false;
  for (int i = 1; i < m && !full; ++i) {
    const double r = eps + t[i];
    const double tt = t[i] - (r - eps);
    if (tt != 0.0) {
      out[j++] = r;
      if (j == m) full = true;
      eps = tt;
    } else {
      eps = r;
    }
  }
  if (!full) {
    out[j++] = eps;
    while (j < m) out[j++] = 0.0;
  }
  for (int pass = 0; pass < m; ++pass) {
    bool changed = false;
    for (int i = 0; i + 1 < m; ++i) {
      double s, e;
      two_sum(out[i], out[i + 1], s, e);
      uint64_t a, b, c, d;
      std::memcpy(&a, &s, 8);
      std::memcpy(&b, &out[i], 8);
      std::memcpy(&c, &e, 8);
      std::memcpy(&d, &out[i + 1], 8);
      if (a != b || c != d) {
        out[i] = s;
        out[i + 1] = e;
        changed = true;
      }
    }
    if (!changed) break;
  }
}

// random_series (pseries.cpp:95-103) into row `row` of a [Q][rows][d+1] block
void fill_series(uint64_t seed, int d, int m, int P, double* stat, int64_t rows, int64_t row) {
  std::mt19937_64 r(seed);
  double t[16], v[16];
  for (int k = 0; k <= d; ++k)
    for (int part = 0; part < P; ++part) {
      for (int l = 0; l < m; ++l) t[l] = pm1(r) * std::ldexp(1.0, -53 * l);
      renorm(t, m, v);
      for (int l = 0; l < m; ++l) stat[((static_cast<int64_t>(part) * m + l) * rows + row) * (d + 1) + k] = v[l];
    }
}

void shape_of(const std::string& id, int32_t& n, int32_t& N, int32_t& len) {
  if (id == "p1") {
    n = 16, N = 1820, len = 1820 * 4;
  } else if (id == "p2") {
    n = 128, N = 128, len = 128 * 64;
  } else if (id == "p3") {
    n = 128, N = 8128, len = 8128 * 2;
  } else {
    throw std::invalid_argument("unknown benchmark polynomial id: " + id);
  }
}

// all r-subsets of {1..n} in lexicographic order (gen.cpp:13-26)
void subsets(int n, int r, int32_t* nvars, int32_t* idx) {
  std::vector<int32_t> c(r);
  for (int i = 0; i < r; ++i) c[i] = i + 1;
  int64_t k = 0;
  while (true) {
    nvars[k] = r;
    std::copy(c.begin(), c.end(), idx + k * r);
    ++k;
    int i = r - 1;
    while (i >= 0 && c[i] == n - (r - 1 - i)) --i;
    if (i < 0) break;
    ++c[i];
    for (int j = i + 1; j < r; ++j) c[j] = c[j - 1] + 1;
  }
}

}  // namespace
}  // namespace pse

extern "C" {

int pse_gen_benchmark_size(const char* id, int32_t* n, int32_t* N, int32_t* shape_len) {
  try {
    pse::shape_of(id ? id : "", *n, *N, *shape_len);
    return PSE_OK;
  } catch (const std::invalid_argument& e) {
    pse::set_error(e.what());
    return PSE_EINVAL;
  }
}

int pse_gen_benchmark(const char* id, int32_t d, int32_t m, int32_t mode, uint64_t seed, int32_t* nvars,
                      int32_t* indices, double* stat) {
  try {
    int32_t n, N, len;
    pse::shape_of(id ? id : "", n, N, len);
    if (!pse::valid_precision(m)) throw std::invalid_argument("unsupported precision level");
    if (d < 0) throw std::invalid_argument("negative truncation degree");
    const std::string sid(id);
    if (sid == "p1") {
      pse::subsets(16, 4, nvars, indices);
    } else if (sid == "p3") {
      pse::subsets(128, 2, nvars, indices);
    } else {  // p2: 128 cyclic windows of 64 variables, sorted (gen.cpp:31-40)
      for (int k = 0; k < 128; ++k) {
        nvars[k] = 64;
        for (int j = 0; j < 64; ++j) indices[k * 64 + j] = (k + j) % 128 + 1;
        std::sort(indices + k * 64, indices + k * 64 + 64);
      }
    }
    if (!stat) return PSE_OK;
    const int P = mode == PSE_MODE_COMPLEX ? 2 : 1;
    const int64_t rows = 1 + static_cast<int64_t>(N) + n;
    // stream seeds (gen.cpp:58-68): a0 <- (1<<32), a_k <- (2<<32)+k, z_i <- (3<<32)+i
    std::vector<std::pair<uint64_t, int64_t>> jobs;
    jobs.reserve(rows);
    jobs.emplace_back(pse::mix_seed(seed, 1ULL << 32), 0);
    for (int k = 0; k < N; ++k) jobs.emplace_back(pse::mix_seed(seed, (2ULL << 32) + k), 1 + k);
    for (int i = 0; i < n; ++i) jobs.emplace_back(pse::mix_seed(seed, (3ULL << 32) + i), N + 1 + i);
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < hw; ++w)
      pool.emplace_back([&, w] {
        for (size_t t = w; t < jobs.size(); t += hw)
          pse::fill_series(jobs[t].first, d, m, P, stat, rows, jobs[t].second);
      });
    for (auto& th : pool) th.join();
    return PSE_OK;
  } catch (const std::invalid_argument& e) {
    pse::set_error(e.what());
    return PSE_EINVAL;
  }
}

}  // extern "C"
