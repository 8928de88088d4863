/* TEST INFRASTRUCTURE ONLY -- the checker, never the product.
 *
 * Plain-C restatement of the reference CPU path (arXiv 2101.10881 artifact
 * `pseval`, /root/reference/proj). Each function cites the reference
 * file:line it restates. Parity of this restatement is pinned two ways:
 *   - against the reference engine itself, compiled from its sources into
 *     oracle/_ref/libpseval_ref.so (tests/test_oracle_pins.py), and
 *   - against committed golden vectors generated from that library
 *     (tests/golden/, made by tests/golden/make_golden.py).
 *
 * Packed conventions (shared with oracle/ref_shim.cpp and the product C ABI):
 *   P = 2 in complex mode (re, im), else 1
 *   static block  [P][m][static_top][d+1], static_top = 1 + N + n
 *   value/grad    [P][m][n+1][d+1] (row 0 value, row 1+i gradient i)
 *   md values     [count][m]
 */
#ifndef PSE_ORACLE_H
#define PSE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* expansion arithmetic (expansion.hpp:31-211); op 0 add, 1 sub, 2 mul */
int pso_md_op(int op, int m, int64_t count, const double* x, const double* y, double* out);
/* instrumented / reporting op costs (multidouble.cpp:36-75): out = {ia, im, ra, rm} */
int pso_cost(int m, int64_t* out);
/* Rng + splitmix (rng.hpp:11-36) */
uint64_t pso_mix_seed(uint64_t base, uint64_t stream);
void pso_rng_u64(uint64_t seed, int64_t count, uint64_t* out);
/* count random_md values from Rng(seed) (multidouble.cpp:26-30) */
void pso_random_md(uint64_t seed, int m, int64_t count, double* out);
int pso_renormalize(const double* t, int n, int m, double* out);

/* Graph (jobgraph.cpp:65-262). Shape: nvars[N], idx[sum] 1-based, exps[sum]
 * (all-zero row = no exponents) or NULL. */
typedef struct pso_graph pso_graph;
pso_graph* pso_graph_build(int n, int d, int N, const int* nvars, const int* idx, const int* exps);
void pso_graph_free(pso_graph* g);
/* info: n, N, d, total_slots, nconv, nadd, ncopy, nconv_layers, nadd_layers, n_term_scales */
void pso_graph_info(const pso_graph* g, int64_t* info);
/* same row formats as ref_graph_export */
void pso_graph_export(const pso_graph* g, int64_t* conv, int64_t* add, int64_t* value_slot,
                      int64_t* grad_slots, int64_t* mult, int64_t* ts);
/* 1 valid, 0 invalid (message into msg) -- validate(), jobgraph.cpp:273-336 */
int pso_graph_validate(const pso_graph* g, char* msg, int cap);
/* flop_count* (executor.cpp:233-252); which 0 total, 1 mul, 2 add */
int64_t pso_flop_count(const pso_graph* g, int d, int cplx, int64_t add_cost, int64_t mul_cost, int which);

/* gen_benchmark (gen.cpp:50-71): shape sizes, then shape + static block */
int pso_gen_shape_size(const char* id, int* n, int* N, int* shape_len);
int pso_gen_benchmark(const char* id, int d, int m, int cplx, uint64_t seed, int* nvars, int* idx,
                      double* stat);

/* evaluate() with the sequential engine (executor.cpp:271-276): fold, stage,
 * run_sequential, extract. dyn_out (nullable) receives [P][m][total_slots][d+1]. */
int pso_evaluate(int n, int d, int m, int cplx, int N, const int* nvars, const int* idx,
                 const int* exps, const double* stat, double* vg_out, double* dyn_out);
/* eval_direct (oracle_direct.cpp:41-78); returns -2 when beyond the guard */
int pso_eval_direct(int n, int d, int m, int cplx, int N, const int* nvars, const int* idx,
                    const int* exps, const double* stat, double* vg_out);
/* series conv (pseries.cpp:37-64); x, y, out: [P][m][d+1] */
int pso_series_conv(int d, int m, int cplx, const double* x, const double* y, double* out);

const char* pso_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
