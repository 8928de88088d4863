// Host-side graph compiler shared by the C ABI and the device planner.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pse_b200.h"

namespace pse {

void set_error(const std::string& msg);

// Compiled polynomial shape: the reference JobGraph (jobgraph.hpp:75-90) in
// flat, layer-sorted arrays, plus the shape itself (needed for device-side
// exponent folding, jobgraph.cpp:168-197).
struct HostGraph {
  int32_t n = 0, N = 0, d = 0;
  int64_t total_slots = 0, value_slot = -1;
  std::vector<int64_t> gradient_slots, multipliers;
  std::vector<int64_t> conv_layer_off, conv_in1, conv_in2, conv_out;
  std::vector<uint8_t> conv_copy;
  std::vector<int64_t> add_layer_off, add_src, add_dst;
  std::vector<int64_t> ts_slot, ts_factor;
  // shape
  std::vector<int32_t> nvars, indices, exponents;  // exponents empty = none anywhere
  std::vector<int64_t> mono_start;                 // [N+1]
  bool has_exponents(int k) const;
};

// build_jobgraph (jobgraph.cpp:199-262); throws std::invalid_argument
HostGraph build_graph(int32_t n, int32_t d, int32_t N, const int32_t* nvars, const int32_t* indices,
                      const int32_t* exponents);

pse_graph_desc describe(const HostGraph& g, int32_t m, int32_t mode);

// validate (jobgraph.cpp:273-336): empty string when valid
std::string validate_desc(const pse_graph_desc& g);

int64_t flop_count(const pse_graph_desc& g, int which, int64_t add_cost, int64_t mul_cost);

struct Costs {
  int64_t inst_add, inst_mul, rep_add, rep_mul;
};
bool valid_precision(int m);
Costs costs(int m);  // throws for unsupported m

// executed binary64 ops of one evaluation at the instrumented costs: the
// roofline numerator (triangular convolutions)
int64_t alg_op_count(const pse_graph_desc& g);

}  // namespace pse
