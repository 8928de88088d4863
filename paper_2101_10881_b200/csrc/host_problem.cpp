// Problem files: the reference's line-oriented text format
// (proj/src/problem_io.cpp:11-24, :130-245) -- hexfloat limbs so a write/read
// cycle reproduces every bit, decimal accepted on input, parse errors carry
// the 1-based line number ("line N: ..."), returned as PSE_EINVAL.
//
//   pseval 1
//   problem <id> <n> <N> <d> <m> <real|complex> <seed>
//   constant            + d+1 coefficient lines
//   monomial <nk> / indices i1..ink / [exponents e1..enk] / d+1 coefficient lines
//   input <i>           + d+1 coefficient lines, i = 1..n
//   end
// A coefficient line holds the m limbs (2m in complex mode: real then imaginary).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_graph.hpp"

namespace pse {
namespace {

struct LineError : std::invalid_argument {
  LineError(int line, const std::string& what) : std::invalid_argument("line " + std::to_string(line) + ": " + what) {}
};

}  // namespace

struct Problem {
  std::string id = "file";
  uint64_t seed = 0;
  int32_t n = 0, d = 0, m = 1, mode = PSE_MODE_REAL;
  std::vector<int32_t> nvars, indices, exponents;  // exponents: 0 = none for that monomial
  std::vector<double> stat;                        // [Q][1+N+n][d+1]
  int32_t N() const { return static_cast<int32_t>(nvars.size()); }
  int Q() const { return (mode == PSE_MODE_COMPLEX ? 2 : 1) * m; }
  int64_t rows() const { return 1 + static_cast<int64_t>(N()) + n; }
  double& at(int q, int64_t row, int k) { return stat[(static_cast<int64_t>(q) * rows() + row) * (d + 1) + k]; }
  double at(int q, int64_t row, int k) const {
    return stat[(static_cast<int64_t>(q) * rows() + row) * (d + 1) + k];
  }
};

namespace {

class Lines {
 public:
  explicit Lines(const std::string& text) : in_(text) {}
  int line = 0;
  // next non-blank line, split into tokens
  std::vector<std::string> want(const std::string& what) {
    std::vector<std::string> t;
    if (pending_) {
      pending_ = false;
      return cur_;
    }
    std::string s;
    while (std::getline(in_, s)) {
      ++line;
      std::istringstream ss(s);
      std::string w;
      t.clear();
      while (ss >> w) t.push_back(w);
      if (!t.empty()) {
        cur_ = t;
        return t;
      }
    }
    throw LineError(line, "unexpected end of file, expected " + what);
  }
  void unread() { pending_ = true; }

 private:
  std::istringstream in_;
  std::vector<std::string> cur_;
  bool pending_ = false;
};

double to_double(const std::string& s, int line) {
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size()) throw LineError(line, "malformed number '" + s + "'");
  return v;
}

long to_long(const std::string& s, int line) {
  char* end = nullptr;
  const long v = std::strtol(s.c_str(), &end, 10);
  if (s.empty() || end != s.c_str() + s.size()) throw LineError(line, "malformed integer '" + s + "'");
  return v;
}

void read_coeffs(Lines& r, Problem& p, int64_t row, const std::string& what) {
  const size_t per = static_cast<size_t>(p.Q());
  for (int k = 0; k <= p.d; ++k) {
    const auto t = r.want(what + " coefficient line");
    if (t.size() != per)
      throw LineError(r.line, what + ": expected " + std::to_string(per) + " values, got " + std::to_string(t.size()));
    for (size_t q = 0; q < per; ++q) p.at(static_cast<int>(q), row, k) = to_double(t[q], r.line);
  }
}

Problem parse(const std::string& text) {
  Lines r(text);
  auto t = r.want("the format header");
  if (t.size() != 2 || t[0] != "pseval" || t[1] != "1")
    throw LineError(r.line, "not a pseval problem file (expected 'pseval 1')");
  t = r.want("the problem header");
  if (t.size() != 8 || t[0] != "problem") throw LineError(r.line, "malformed problem header");
  Problem p;
  p.id = t[1];
  const long n = to_long(t[2], r.line), N = to_long(t[3], r.line), d = to_long(t[4], r.line),
             m = to_long(t[5], r.line);
  if (n < 1) throw LineError(r.line, "variable count must be positive");
  if (N < 1) throw LineError(r.line, "monomial count must be positive");
  if (d < 0) throw LineError(r.line, "negative truncation degree");
  if (!valid_precision(static_cast<int>(m))) throw LineError(r.line, "unsupported precision level " + t[5]);
  if (t[6] == "real")
    p.mode = PSE_MODE_REAL;
  else if (t[6] == "complex")
    p.mode = PSE_MODE_COMPLEX;
  else
    throw LineError(r.line, "unknown mode '" + t[6] + "'");
  {
    char* end = nullptr;
    p.seed = std::strtoull(t[7].c_str(), &end, 10);
    if (t[7].empty() || t[7][0] == '-' || end != t[7].c_str() + t[7].size())
      throw LineError(r.line, "malformed seed '" + t[7] + "'");
  }
  p.n = static_cast<int32_t>(n);
  p.d = static_cast<int32_t>(d);
  p.m = static_cast<int32_t>(m);
  p.nvars.resize(N);
  p.stat.assign(static_cast<size_t>(p.Q()) * (1 + N + n) * (d + 1), 0.0);

  t = r.want("the constant record");
  if (t.size() != 1 || t[0] != "constant") throw LineError(r.line, "expected the constant record");
  read_coeffs(r, p, 0, "constant");

  bool any_exp = false;
  std::vector<int32_t> exps;
  for (long k = 0; k < N; ++k) {
    t = r.want("a monomial record");
    if (t.size() != 2 || t[0] != "monomial") throw LineError(r.line, "expected 'monomial <count>'");
    const long nk = to_long(t[1], r.line);
    if (nk < 1) throw LineError(r.line, "monomial needs at least one variable");
    p.nvars[k] = static_cast<int32_t>(nk);
    t = r.want("the indices line");
    if (t.empty() || t[0] != "indices") throw LineError(r.line, "expected the indices line");
    if (static_cast<long>(t.size()) - 1 != nk) throw LineError(r.line, "expected " + std::to_string(nk) + " indices");
    long prev = 0;
    for (size_t j = 1; j < t.size(); ++j) {
      const long ix = to_long(t[j], r.line);
      if (ix < 1 || ix > n) throw LineError(r.line, "variable index out of range");
      if (ix == prev) throw LineError(r.line, "duplicate variable index");
      if (ix < prev) throw LineError(r.line, "indices must be strictly increasing");
      prev = ix;
      p.indices.push_back(static_cast<int32_t>(ix));
    }
    t = r.want("a coefficient or exponents line");
    if (t[0] == "exponents") {
      if (static_cast<long>(t.size()) - 1 != nk)
        throw LineError(r.line, "expected " + std::to_string(nk) + " exponents");
      for (size_t j = 1; j < t.size(); ++j) {
        const long e = to_long(t[j], r.line);
        if (e < 1) throw LineError(r.line, "exponents must be positive");
        exps.push_back(static_cast<int32_t>(e));
      }
      any_exp = true;
    } else {
      r.unread();
      exps.insert(exps.end(), static_cast<size_t>(nk), 0);
    }
    read_coeffs(r, p, 1 + k, "monomial coefficient");
  }
  if (any_exp) p.exponents = exps;
  for (long i = 1; i <= n; ++i) {
    t = r.want("an input record");
    if (t.size() != 2 || t[0] != "input" || to_long(t[1], r.line) != i)
      throw LineError(r.line, "expected 'input " + std::to_string(i) + "'");
    read_coeffs(r, p, N + i, "input");
  }
  t = r.want("the end marker");
  if (t.size() != 1 || t[0] != "end") throw LineError(r.line, "expected the end marker");
  return p;
}

void append_coeffs(std::string& out, const Problem& p, int64_t row) {
  char buf[40];
  for (int k = 0; k <= p.d; ++k) {
    for (int q = 0; q < p.Q(); ++q) {
      std::snprintf(buf, sizeof buf, "%a", p.at(q, row, k));
      if (q) out += ' ';
      out += buf;
    }
    out += '\n';
  }
}

std::string to_text(const Problem& p) {
  std::string out = "pseval 1\n";
  out += "problem " + p.id + ' ' + std::to_string(p.n) + ' ' + std::to_string(p.N()) + ' ' + std::to_string(p.d) +
         ' ' + std::to_string(p.m) + ' ' + (p.mode == PSE_MODE_COMPLEX ? "complex" : "real") + ' ' +
         std::to_string(p.seed) + '\n';
  out += "constant\n";
  append_coeffs(out, p, 0);
  size_t pos = 0;
  for (int k = 0; k < p.N(); ++k) {
    const int nk = p.nvars[k];
    out += "monomial " + std::to_string(nk) + "\nindices";
    for (int j = 0; j < nk; ++j) out += ' ' + std::to_string(p.indices[pos + j]);
    out += '\n';
    bool has = false;
    for (int j = 0; j < nk && !p.exponents.empty(); ++j) has |= p.exponents[pos + j] != 0;
    if (has) {
      out += "exponents";
      for (int j = 0; j < nk; ++j) out += ' ' + std::to_string(p.exponents[pos + j]);
      out += '\n';
    }
    append_coeffs(out, p, 1 + k);
    pos += nk;
  }
  for (int i = 1; i <= p.n; ++i) {
    out += "input " + std::to_string(i) + '\n';
    append_coeffs(out, p, p.N() + i);
  }
  out += "end\n";
  return out;
}

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return PSE_EINVAL;
  } catch (const std::exception& e) {
    set_error(e.what());
    return PSE_ESTATE;
  }
}

}  // namespace
}  // namespace pse

struct pse_problem {
  pse::Problem p;
};

extern "C" {

int pse_problem_parse(const char* text, pse_problem** out) {
  return pse::guard([&] {
    if (!text || !out) throw std::invalid_argument("null argument");
    auto* h = new pse_problem;
    try {
      h->p = pse::parse(text);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return PSE_OK;
  });
}

int pse_problem_read(const char* path, pse_problem** out) {
  return pse::guard([&] {
    if (!path || !out) throw std::invalid_argument("null argument");
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("cannot open '") + path + "'");
    std::ostringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    return pse_problem_parse(text.c_str(), out);
  });
}

int pse_problem_text(const pse_problem* h, char* buf, size_t cap, size_t* len) {
  return pse::guard([&] {
    if (!h) throw std::invalid_argument("null problem");
    const std::string t = pse::to_text(h->p);
    if (len) *len = t.size();
    if (buf && cap) {
      std::memcpy(buf, t.data(), std::min(cap - 1, t.size()));
      buf[std::min(cap - 1, t.size())] = 0;
    }
    return PSE_OK;
  });
}

int pse_problem_write(const pse_problem* h, const char* path) {
  return pse::guard([&] {
    if (!h || !path) throw std::invalid_argument("null argument");
    const std::string t = pse::to_text(h->p);
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("cannot open '") + path + "' for writing");
    f.write(t.data(), static_cast<std::streamsize>(t.size()));
    if (!f) throw std::runtime_error(std::string("write to '") + path + "' failed");
    return PSE_OK;
  });
}

int pse_problem_create(const char* id, uint64_t seed, int32_t n, int32_t d, int32_t m, int32_t mode, int32_t N,
                       const int32_t* nvars, const int32_t* indices, const int32_t* exponents, const double* stat,
                       pse_problem** out) {
  return pse::guard([&] {
    if (!nvars || !indices || !stat || !out) throw std::invalid_argument("null argument");
    pse::build_graph(n, d, N, nvars, indices, exponents);  // shape checks (check_polynomial)
    if (!pse::valid_precision(m)) throw std::invalid_argument("unsupported precision level");
    auto* h = new pse_problem;
    pse::Problem& p = h->p;
    p.id = id ? id : "file";
    p.seed = seed;
    p.n = n;
    p.d = d;
    p.m = m;
    p.mode = mode;
    p.nvars.assign(nvars, nvars + N);
    int64_t len = 0;
    for (int k = 0; k < N; ++k) len += nvars[k];
    p.indices.assign(indices, indices + len);
    if (exponents) {
      bool any = false;
      for (int64_t q = 0; q < len; ++q) any |= exponents[q] != 0;
      if (any) p.exponents.assign(exponents, exponents + len);
    }
    p.stat.assign(stat, stat + static_cast<size_t>(p.Q()) * p.rows() * (d + 1));
    *out = h;
    return PSE_OK;
  });
}

int pse_problem_gen(const char* id, int32_t d, int32_t m, int32_t mode, uint64_t seed, pse_problem** out) {
  return pse::guard([&] {
    int32_t n, N, len;
    if (pse_gen_benchmark_size(id, &n, &N, &len) != PSE_OK) throw std::invalid_argument(pse_last_error());
    std::vector<int32_t> nv(N), ix(len);
    const int Q = (mode == PSE_MODE_COMPLEX ? 2 : 1) * m;
    std::vector<double> st(static_cast<size_t>(Q) * (1 + N + n) * (d + 1));
    if (pse_gen_benchmark(id, d, m, mode, seed, nv.data(), ix.data(), st.data()) != PSE_OK)
      throw std::invalid_argument(pse_last_error());
    return pse_problem_create(id, seed, n, d, m, mode, N, nv.data(), ix.data(), nullptr, st.data(), out);
  });
}

// out[7] = n, N, d, m, mode, seed, shape length
int pse_problem_info(const pse_problem* h, int64_t* out) {
  if (!h || !out) return PSE_EINVAL;
  const pse::Problem& p = h->p;
  int64_t v[7] = {p.n, p.N(), p.d, p.m, p.mode, static_cast<int64_t>(p.seed), static_cast<int64_t>(p.indices.size())};
  std::memcpy(out, v, sizeof v);
  return PSE_OK;
}

int pse_problem_id(const pse_problem* h, char* buf, size_t cap) {
  if (!h || !buf || !cap) return PSE_EINVAL;
  std::strncpy(buf, h->p.id.c_str(), cap - 1);
  buf[cap - 1] = 0;
  return PSE_OK;
}

// pointers stay valid until pse_problem_destroy; exponents is NULL when the
// problem has none; stat is [Q][1+N+n][d+1]
int pse_problem_arrays(const pse_problem* h, const int32_t** nvars, const int32_t** indices,
                       const int32_t** exponents, const double** stat) {
  if (!h) return PSE_EINVAL;
  if (nvars) *nvars = h->p.nvars.data();
  if (indices) *indices = h->p.indices.data();
  if (exponents) *exponents = h->p.exponents.empty() ? nullptr : h->p.exponents.data();
  if (stat) *stat = h->p.stat.data();
  return PSE_OK;
}

void pse_problem_destroy(pse_problem* h) { delete h; }

}  // extern "C"
