// Host graph compiler: polynomial shape -> layered convolution / addition job
// lists, job-for-job identical to the reference build_jobgraph
// (proj/src/jobgraph.cpp:199-262), plus validation, FLOP models and the C-ABI
// entry points for them.
//
// Slot layout (Eq. 6 of the paper; jobgraph.hpp:58-73): a0 = 0, a_k = 1+k,
// z_i = N+i, then all forward blocks (n_k slots per monomial), all backward
// blocks (max(1, n_k-2)), all cross blocks (max(0, n_k-2)).
#include <algorithm>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>

#include "host_graph.hpp"

namespace pse {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

bool HostGraph::has_exponents(int k) const {
  if (exponents.empty()) return false;
  for (int64_t p = mono_start[k]; p < mono_start[k + 1]; ++p)
    if (exponents[p] != 0) return true;
  return false;
}

namespace {

void fail(const char* msg) { throw std::invalid_argument(msg); }

// Slot arithmetic of one compiled shape.
struct SlotMap {
  int32_t n, N;
  std::vector<int64_t> fwd, bwd, crs;  // per-monomial block starts (absolute slots)
  int64_t total;

  SlotMap(int32_t n_, const std::vector<int32_t>& nv) : n(n_), N(static_cast<int32_t>(nv.size())) {
    const int64_t base = 1 + N + n;
    int64_t f = 0, b = 0, c = 0;
    fwd.resize(N + 1);
    bwd.resize(N + 1);
    crs.resize(N + 1);
    for (int32_t k = 0; k < N; ++k) {
      fwd[k] = f;
      bwd[k] = b;
      crs[k] = c;
      f += nv[k];
      b += std::max<int64_t>(1, nv[k] - 2);
      c += std::max<int64_t>(0, nv[k] - 2);
    }
    fwd[N] = f;
    bwd[N] = b;
    crs[N] = c;
    for (int32_t k = 0; k <= N; ++k) {
      fwd[k] += base;
      bwd[k] += base + f;
      crs[k] += base + f + b;
    }
    total = crs[N];
  }
  int64_t a(int k) const { return 1 + k; }
  int64_t z(int i) const { return N + i; }
  int64_t F(int k, int l) const { return fwd[k] + l - 1; }
  int64_t B(int k, int l) const { return bwd[k] + l - 1; }
  int64_t Cx(int k, int j) const { return crs[k] + j - 1; }
};

struct Row {
  int32_t layer;
  int64_t in1, in2, out;
  uint8_t copy;
};

// Reverse-mode products of one monomial (jobgraph.cpp:90-124): forward
// chain f, backward chain b with the coefficient folded into its last link,
// and cross products c; 3 n_k - 3 jobs for n_k >= 3.
void monomial_rows(int k, const int32_t* ix, int nk, const SlotMap& S, std::vector<Row>& rows) {
  auto Z = [&](int pos) { return S.z(ix[pos - 1]); };
  rows.push_back({1, S.a(k), Z(1), S.F(k, 1), 0});
  for (int l = 2; l <= nk; ++l) rows.push_back({l, S.F(k, l - 1), Z(l), S.F(k, l), 0});
  switch (nk) {
    case 1:
      rows.push_back({1, S.a(k), 0, S.B(k, 1), 1});  // derivative = a_k, as a copy
      return;
    case 2:
      rows.push_back({1, Z(2), S.a(k), S.B(k, 1), 0});
      return;
    default:
      break;
  }
  rows.push_back({1, Z(nk), Z(nk - 1), S.B(k, 1), 0});
  for (int l = 2; l <= nk - 2; ++l) rows.push_back({l, S.B(k, l - 1), Z(nk - l), S.B(k, l), 0});
  rows.push_back({nk - 1, S.B(k, nk - 2), S.a(k), S.B(k, nk - 2), 0});  // in-place fold
  for (int j = 1; j <= nk - 3; ++j)
    rows.push_back({std::max(j, nk - 2 - j) + 1, S.F(k, j), S.B(k, nk - 2 - j), S.Cx(k, j), 0});
  rows.push_back({nk - 1, S.F(k, nk - 2), Z(nk), S.Cx(k, nk - 2), 0});
}

// slot holding monomial k's derivative term for its j-th variable
// (gradient_term_map, jobgraph.cpp:149-166)
int64_t derivative_slot(int k, int j, int nk, const SlotMap& S) {
  if (nk >= 2 && j == nk) return S.F(k, nk - 1);
  if (j == 1) return S.B(k, nk >= 3 ? nk - 2 : 1);
  return S.Cx(k, j - 1);
}

}  // namespace

HostGraph build_graph(int32_t n, int32_t d, int32_t N, const int32_t* nvars, const int32_t* indices,
                      const int32_t* exponents) {
  // check_polynomial (jobgraph.cpp:41-63)
  if (n < 1) fail("polynomial needs at least one variable");
  if (N < 1) fail("polynomial needs at least one monomial");
  if (d < 0) fail("negative truncation degree");
  HostGraph g;
  g.n = n;
  g.N = N;
  g.d = d;
  g.nvars.assign(nvars, nvars + N);
  g.mono_start.resize(N + 1, 0);
  for (int32_t k = 0; k < N; ++k) {
    if (nvars[k] < 1) fail("monomial without variables");
    g.mono_start[k + 1] = g.mono_start[k] + nvars[k];
  }
  const int64_t len = g.mono_start[N];
  g.indices.assign(indices, indices + len);
  bool any_exp = false;
  if (exponents) {
    g.exponents.assign(exponents, exponents + len);
    for (int64_t p = 0; p < len; ++p) any_exp |= exponents[p] != 0;
    if (!any_exp) g.exponents.clear();
  }
  for (int32_t k = 0; k < N; ++k) {
    int prev = 0;
    const bool has = g.has_exponents(k);
    for (int64_t p = g.mono_start[k]; p < g.mono_start[k + 1]; ++p) {
      if (indices[p] <= prev) fail("monomial indices must be strictly increasing");
      if (indices[p] > n) fail("monomial index out of range");
      prev = indices[p];
      if (has && g.exponents[p] < 1) fail("exponents must be positive");
    }
  }

  const SlotMap S(n, g.nvars);
  g.total_slots = S.total;

  // conv jobs, grouped by layer in monomial order (stable bucket by layer)
  std::vector<Row> rows;
  rows.reserve(static_cast<size_t>(3 * len));
  for (int32_t k = 0; k < N; ++k) monomial_rows(k, g.indices.data() + g.mono_start[k], g.nvars[k], S, rows);
  int32_t nlayers = 0;
  for (const Row& r : rows) nlayers = std::max(nlayers, r.layer);
  std::vector<int64_t> cnt(nlayers + 1, 0);
  for (const Row& r : rows) ++cnt[r.layer];
  g.conv_layer_off.assign(nlayers + 1, 0);
  for (int32_t L = 1; L <= nlayers; ++L) g.conv_layer_off[L] = g.conv_layer_off[L - 1] + cnt[L];
  std::vector<int64_t> fill(g.conv_layer_off.begin(), g.conv_layer_off.end() - 1);
  const size_t nc = rows.size();
  g.conv_in1.resize(nc);
  g.conv_in2.resize(nc);
  g.conv_out.resize(nc);
  g.conv_copy.resize(nc);
  for (const Row& r : rows) {
    const int64_t at = fill[r.layer - 1]++;
    g.conv_in1[at] = r.in1;
    g.conv_in2[at] = r.in2;
    g.conv_out[at] = r.out;
    g.conv_copy[at] = r.copy;
  }

  // term lists: value list (a0, then each monomial's full product), then the
  // non-empty per-variable derivative lists in variable order
  std::vector<std::vector<int64_t>> lists(1);
  lists[0].push_back(0);
  for (int32_t k = 0; k < N; ++k) lists[0].push_back(S.F(k, g.nvars[k]));
  std::vector<std::vector<int64_t>> per_var(n);
  for (int32_t k = 0; k < N; ++k) {
    const int nk = g.nvars[k];
    for (int j = 1; j <= nk; ++j)
      per_var[g.indices[g.mono_start[k] + j - 1] - 1].push_back(derivative_slot(k, j, nk, S));
  }
  for (auto& v : per_var)
    if (!v.empty()) lists.push_back(v);

  // pairwise tree per list (addition_schedule, jobgraph.cpp:126-147):
  // level L pairs consecutive survivors (dst = the later one); an odd tail
  // passes through; level-L jobs of all lists form add layer L
  std::vector<std::vector<std::pair<int64_t, int64_t>>> levels;
  for (const auto& list : lists) {
    std::vector<int64_t> live = list;
    for (size_t level = 0; live.size() > 1; ++level) {
      if (levels.size() <= level) levels.emplace_back();
      std::vector<int64_t> keep;
      keep.reserve(live.size() / 2 + 1);
      size_t t = 0;
      for (; t + 1 < live.size(); t += 2) {
        levels[level].emplace_back(live[t], live[t + 1]);
        keep.push_back(live[t + 1]);
      }
      if (t < live.size()) keep.push_back(live[t]);
      live.swap(keep);
    }
  }
  g.add_layer_off.assign(levels.size() + 1, 0);
  for (size_t L = 0; L < levels.size(); ++L) {
    g.add_layer_off[L + 1] = g.add_layer_off[L] + static_cast<int64_t>(levels[L].size());
    for (auto& [src, dst] : levels[L]) {
      g.add_src.push_back(src);
      g.add_dst.push_back(dst);
    }
  }

  g.value_slot = lists[0].back();
  g.gradient_slots.assign(n, -1);
  for (int32_t i = 0; i < n; ++i)
    if (!per_var[i].empty()) g.gradient_slots[i] = per_var[i].back();

  // chain-rule exponent factors (jobgraph.cpp:232-261): a variable with one
  // exponent value everywhere gets an extraction multiplier; mixed exponents
  // scale the individual term slots instead
  std::vector<std::set<int64_t>> seen(n);
  for (int32_t k = 0; k < N; ++k) {
    const bool has = g.has_exponents(k);
    for (int64_t p = g.mono_start[k]; p < g.mono_start[k + 1]; ++p)
      seen[g.indices[p] - 1].insert(has ? g.exponents[p] : 1);
  }
  g.multipliers.assign(n, 1);
  std::vector<char> mixed(n, 0);
  for (int32_t i = 0; i < n; ++i) {
    if (seen[i].size() == 1) g.multipliers[i] = *seen[i].begin();
    if (seen[i].size() > 1) mixed[i] = 1;
  }
  std::vector<size_t> cursor(n, 0);
  for (int32_t k = 0; k < N; ++k) {
    const bool has = g.has_exponents(k);
    for (int64_t p = g.mono_start[k]; p < g.mono_start[k + 1]; ++p) {
      const int var = g.indices[p] - 1;
      const int64_t slot = per_var[var][cursor[var]++];
      const int64_t e = has ? g.exponents[p] : 1;
      if (mixed[var] && e != 1) {
        g.ts_slot.push_back(slot);
        g.ts_factor.push_back(e);
      }
    }
  }
  return g;
}

pse_graph_desc describe(const HostGraph& g, int32_t m, int32_t mode) {
  pse_graph_desc d{};
  d.n = g.n;
  d.N = g.N;
  d.d = g.d;
  d.m = m;
  d.mode = mode;
  d.total_slots = g.total_slots;
  d.value_slot = g.value_slot;
  d.gradient_slots = g.gradient_slots.data();
  d.multipliers = g.multipliers.data();
  d.n_conv_layers = static_cast<int32_t>(g.conv_layer_off.size()) - 1;
  d.conv_layer_off = g.conv_layer_off.data();
  d.conv_in1 = g.conv_in1.data();
  d.conv_in2 = g.conv_in2.data();
  d.conv_out = g.conv_out.data();
  d.conv_copy = g.conv_copy.data();
  d.n_add_layers = static_cast<int32_t>(g.add_layer_off.size()) - 1;
  d.add_layer_off = g.add_layer_off.data();
  d.add_src = g.add_src.data();
  d.add_dst = g.add_dst.data();
  d.n_term_scales = static_cast<int64_t>(g.ts_slot.size());
  d.ts_slot = g.ts_slot.data();
  d.ts_factor = g.ts_factor.data();
  return d;
}

// validate (jobgraph.cpp:273-336): layer dependencies, disjoint writes per
// layer, no output aliasing the second input, add inputs produced by the
// conv stage, accumulation only into dynamic slots, full slot coverage.
std::string validate_desc(const pse_graph_desc& g) {
  if (g.n < 1 || g.N < 1 || g.d < 0) return "bad graph dimensions";
  const int64_t top = 1 + static_cast<int64_t>(g.N) + g.n;
  const int64_t T = g.total_slots;
  if (T < top) return "total_slots below the static region";
  std::vector<int32_t> first_write(static_cast<size_t>(T), -1);
  std::vector<int32_t> stamp(static_cast<size_t>(T), -1);
  auto name = [](const char* stage, int L, int64_t t) {
    return std::string(stage) + " layer " + std::to_string(L + 1) + " job " + std::to_string(t);
  };
  for (int32_t L = 0; L < g.n_conv_layers; ++L) {
    const int64_t b = g.conv_layer_off[L], e = g.conv_layer_off[L + 1];
    for (int64_t t = b; t < e; ++t) {
      const int64_t o = g.conv_out[t];
      if (o < top || o >= T) return name("conv", L, t - b) + ": writes outside the dynamic region";
      if (stamp[o] == L) return name("conv", L, t - b) + ": duplicate write in one layer";
      stamp[o] = L;
      if (!g.conv_copy[t] && o == g.conv_in2[t]) return name("conv", L, t - b) + ": output aliases second input";
    }
    for (int64_t t = b; t < e; ++t) {
      const int64_t ins[2] = {g.conv_in1[t], g.conv_copy[t] ? g.conv_in1[t] : g.conv_in2[t]};
      for (int64_t s : ins) {
        if (s < 0 || s >= T) return name("conv", L, t - b) + ": input slot out of range";
        if (s < top) continue;
        if (!(first_write[s] >= 0 && first_write[s] < L))
          return name("conv", L, t - b) + ": reads slot " + std::to_string(s) + " not written in an earlier layer";
        if (stamp[s] == L && s != g.conv_out[t])
          return name("conv", L, t - b) + ": reads slot " + std::to_string(s) +
                 " written by another job in the same layer";
      }
    }
    for (int64_t t = b; t < e; ++t)
      if (first_write[g.conv_out[t]] < 0) first_write[g.conv_out[t]] = L;
  }
  std::fill(stamp.begin(), stamp.end(), -1);
  for (int32_t L = 0; L < g.n_add_layers; ++L) {
    const int64_t b = g.add_layer_off[L], e = g.add_layer_off[L + 1];
    for (int64_t t = b; t < e; ++t) {
      const int64_t src = g.add_src[t], dst = g.add_dst[t];
      if (src == dst) return name("add", L, t - b) + ": source equals destination";
      for (int64_t s : {src, dst}) {
        if (s < 0 || s >= T) return name("add", L, t - b) + ": slot out of range";
        if (s >= top && first_write[s] < 0)
          return name("add", L, t - b) + ": slot " + std::to_string(s) + " never written by a conv job";
      }
      if (dst < top) return name("add", L, t - b) + ": accumulates into a static slot";
      if (stamp[dst] == L) return name("add", L, t - b) + ": duplicate write in one layer";
      stamp[dst] = L;
    }
  }
  for (int64_t s = top; s < T; ++s)
    if (first_write[s] < 0) return "slot " + std::to_string(s) + " is never written";
  if (g.value_slot < 0 || g.value_slot >= T) return "value slot out of range";
  for (int32_t i = 0; i < g.n; ++i)
    if (g.gradient_slots[i] >= T) return "gradient slot out of range";
  for (int64_t t = 0; t < g.n_term_scales; ++t)
    if (g.ts_slot[t] < top || g.ts_slot[t] >= T) return "term scale slot outside the dynamic region";
  return "";
}

namespace {
int64_t copy_jobs(const pse_graph_desc& g) {
  const int64_t nc = g.conv_layer_off[g.n_conv_layers];
  int64_t c = 0;
  for (int64_t t = 0; t < nc; ++t) c += g.conv_copy[t] ? 1 : 0;
  return c;
}
}  // namespace

// flop_count* (executor.cpp:233-252): (d+1)^2 products and d(d+1) sums per
// convolution (the paper's zero-insertion model), d+1 sums per addition job
int64_t flop_count(const pse_graph_desc& g, int which, int64_t add_cost, int64_t mul_cost) {
  const int64_t C = g.conv_layer_off[g.n_conv_layers] - copy_jobs(g);
  const int64_t A = g.add_layer_off[g.n_add_layers];
  const int64_t d1 = g.d + 1;
  const bool cx = g.mode == PSE_MODE_COMPLEX;
  const int64_t mul = C * d1 * d1 * (cx ? 4 : 1) * mul_cost;
  int64_t conv_adds = C * g.d * d1;
  if (cx) conv_adds = conv_adds * 2 + C * d1 * d1 * 2;
  const int64_t add = (conv_adds + A * d1 * (cx ? 2 : 1)) * add_cost;
  return which == 1 ? mul : which == 2 ? add : mul + add;
}

bool valid_precision(int m) { return m == 1 || m == 2 || m == 3 || m == 4 || m == 5 || m == 8 || m == 10; }

// instrumented_cost (multidouble.cpp:36-68) is the maximum op count of the
// counting build over a fixed deterministic 64-pair sample; these are its
// values (pinned against the reference library by tests/test_graph.py).
// reporting_cost (multidouble.cpp:70-75) swaps in (1,1) at m=1 and the
// paper's deca-double constants (397, 3089) at m=10.
Costs costs(int m) {
  switch (m) {
    case 1: return {1, 1, 1, 1};
    case 2: return {39, 94, 39, 94};
    case 3: return {69, 203, 69, 203};
    case 4: return {99, 360, 99, 360};
    case 5: return {129, 544, 129, 544};
    case 8: return {219, 1285, 219, 1285};
    case 10: return {279, 1944, 397, 3089};
    default: fail("unsupported precision level");
  }
  return {};
}

int64_t alg_op_count(const pse_graph_desc& g) {
  const Costs c = costs(g.m);
  const int64_t C = g.conv_layer_off[g.n_conv_layers] - copy_jobs(g);
  const int64_t A = g.add_layer_off[g.n_add_layers];
  const int64_t d1 = g.d + 1;
  const int64_t prods = d1 * (d1 + 1) / 2, accs = static_cast<int64_t>(g.d) * d1 / 2;
  if (g.mode == PSE_MODE_COMPLEX)
    return C * (prods * (4 * c.inst_mul + 2 * c.inst_add) + accs * 2 * c.inst_add) + A * d1 * 2 * c.inst_add +
           g.n_term_scales * d1 * 2 * c.inst_mul;
  return C * (prods * c.inst_mul + accs * c.inst_add) + A * d1 * c.inst_add + g.n_term_scales * d1 * c.inst_mul;
}

}  // namespace pse

// ------------------------------------------------------------------ C ABI
struct pse_graph {
  pse::HostGraph g;
};

extern "C" {

const char* pse_last_error(void) { return pse::g_error.c_str(); }
const char* pse_version(void) { return "pse_b200 0.1 (sm_100a)"; }

int pse_graph_build(int32_t n, int32_t d, int32_t N, const int32_t* nvars, const int32_t* indices,
                    const int32_t* exponents, pse_graph** out) {
  if (!out || !nvars || !indices) {
    pse::set_error("null argument");
    return PSE_EINVAL;
  }
  try {
    auto* h = new pse_graph;
    h->g = pse::build_graph(n, d, N, nvars, indices, exponents);
    *out = h;
    return PSE_OK;
  } catch (const std::invalid_argument& e) {
    pse::set_error(e.what());
    return PSE_EINVAL;
  } catch (const std::bad_alloc&) {
    pse::set_error("out of host memory");
    return PSE_ENOMEM;
  }
}

int pse_graph_describe(const pse_graph* g, int32_t m, int32_t mode, pse_graph_desc* desc) {
  if (!g || !desc) {
    pse::set_error("null argument");
    return PSE_EINVAL;
  }
  if (!pse::valid_precision(m) || (mode != PSE_MODE_REAL && mode != PSE_MODE_COMPLEX)) {
    pse::set_error("unsupported precision level");
    return PSE_EINVAL;
  }
  *desc = pse::describe(g->g, m, mode);
  return PSE_OK;
}

void pse_graph_destroy(pse_graph* g) { delete g; }

int pse_graph_validate(const pse_graph_desc* desc, char* msg, size_t cap) {
  if (!desc) {
    pse::set_error("null argument");
    return PSE_EINVAL;
  }
  const std::string why = pse::validate_desc(*desc);
  if (msg && cap) {
    std::strncpy(msg, why.c_str(), cap - 1);
    msg[cap - 1] = 0;
  }
  return why.empty() ? 1 : 0;
}

int64_t pse_flop_count(const pse_graph_desc* desc, int32_t which, int64_t add_cost, int64_t mul_cost) {
  if (!desc) return PSE_EINVAL;
  return pse::flop_count(*desc, which, add_cost, mul_cost);
}

int pse_cost(int32_t m, int64_t* out) {
  if (!pse::valid_precision(m)) {
    pse::set_error("unsupported precision level");
    return PSE_EINVAL;
  }
  const pse::Costs c = pse::costs(m);
  out[0] = c.inst_add;
  out[1] = c.inst_mul;
  out[2] = c.rep_add;
  out[3] = c.rep_mul;
  return PSE_OK;
}

}  // extern "C"
