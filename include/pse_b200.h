/* pse_b200 -- B200-native evaluate-and-differentiate engine for polynomials at
 * truncated power series in multiple-double precision (arXiv 2101.10881).
 *
 * C ABI: plain pointers and sizes, no C++ or torch types. Every entry point
 * returns 0 (PSE_OK) or a negative code and never throws; pse_last_error()
 * gives the thread-local message. The reference reports the same failures as
 * std::invalid_argument (jobgraph.cpp:41-63, executor.cpp:69-80, :186,
 * multidouble.hpp:28-30).
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   pse_graph_build / pse_graph_describe  <- JobGraph build_jobgraph(const Polynomial&)
 *                                            include/pseval/jobgraph.hpp:117, src/jobgraph.cpp:199-262
 *   pse_graph_validate                    <- Validation validate(const JobGraph&)
 *                                            jobgraph.hpp:126, src/jobgraph.cpp:273-336
 *   pse_flop_count                        <- flop_count / flop_count_mul / flop_count_add
 *                                            include/pseval/executor.hpp:59-61, src/executor.cpp:233-252
 *   pse_cost                              <- instrumented_cost / reporting_cost
 *                                            include/pseval/multidouble.hpp:125-131, src/multidouble.cpp:60-75
 *   pse_plan_create + pse_plan_run        <- RunReport run_sequential(const JobGraph&, DataArray&)
 *                                            RunReport run_parallel(const JobGraph&, DataArray&, int)
 *                                            include/pseval/executor.hpp:49-52, src/executor.cpp:168-231
 *                                            (+ extract, executor.cpp:254-269)
 *   pse_evaluate                          <- RunReport evaluate(const Polynomial&, const std::vector<Series>&, int)
 *                                            include/pseval/executor.hpp:69, src/executor.cpp:271-276
 *   pse_gen_benchmark                     <- Problem gen_benchmark(id, d, m, mode, seed)
 *                                            include/pseval/gen.hpp:28, src/gen.cpp:50-71
 *   pse_md_apply                          <- md_add / md_sub / md_mul (multidouble.hpp:75-94 ->
 *                                            expansion.hpp:142-211), elementwise on arrays
 *   pse_series_conv                       <- Series conv(const Series&, const Series&)  src/pseries.cpp:37-64
 *   pse_series_add                        <- Series series_add(const Series&, const Series&)  src/pseries.cpp:66-74
 *   pse_series_scale_int                  <- Series series_scale_int(const Series&, long)  src/pseries.cpp:85-93
 *   pse_eval_direct                       <- Evaluation eval_direct(const Polynomial&, const std::vector<Series>&)
 *                                            include/pseval/oracle.hpp, src/oracle_direct.cpp:41-78
 *   pse_plan_layer_ms                     <- RunReport::conv_layer_ms / add_layer_ms  executor.hpp:31-43
 *
 * Array conventions (P = 2 parts re/im in complex mode, else 1; Q = P*m slabs;
 * slab q = part*m + limb, exactly the reference DataArray's re[0..m-1] then
 * im[0..m-1], executor.hpp:17-29):
 *   static slabs   q-th pointer: point b, slot s < static_top, coefficient j at
 *                  b*point_stride + s*(d+1) + j; static_top = 1 + N + n
 *                  (slot 0 = a0, 1+k = a_k, N+i = z_i, executor.cpp:163-165).
 *                  A reference DataArray's re[l].data() is a valid slab with
 *                  batch = 1.
 *   value/gradient q-th pointer: point b, row r, coefficient j at
 *                  (b*(n+1) + r)*(d+1) + j; row 0 = value, row 1+i = gradient
 *                  of variable i+1 with its multiplier applied, zero series
 *                  for absent variables (extract, executor.cpp:254-269).
 *   dynamic slabs  q-th pointer: point b, slot s < total_slots at
 *                  (b*total_slots + s)*(d+1) + j -- the whole arena exactly as
 *                  run_sequential leaves the DataArray.
 */
#ifndef PSE_B200_H
#define PSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSE_OK 0
#define PSE_EINVAL (-1) /* std::invalid_argument in the reference */
#define PSE_ECUDA (-2)
#define PSE_ENOMEM (-3)
#define PSE_ESTATE (-4)

#define PSE_MODE_REAL 0
#define PSE_MODE_COMPLEX 1

typedef struct pse_graph pse_graph; /* host-side compiled JobGraph */
typedef struct pse_plan pse_plan;   /* device-resident plan for one GPU */

/* Flattened JobGraph (jobgraph.hpp:75-90), job-for-job identical to
 * build_jobgraph. Layer l of the conv stage is rows
 * [conv_layer_off[l], conv_layer_off[l+1]) of the conv_* arrays, and likewise
 * for additions. All arrays are owned by the caller (or by the pse_graph that
 * filled the descriptor). */
typedef struct {
  int32_t n, N, d, m, mode;
  int64_t total_slots, value_slot;
  const int64_t* gradient_slots; /* [n], -1 = variable absent everywhere */
  const int64_t* multipliers;    /* [n] */
  int32_t n_conv_layers;
  const int64_t* conv_layer_off; /* [n_conv_layers + 1] */
  const int64_t *conv_in1, *conv_in2, *conv_out;
  const uint8_t* conv_copy;
  int32_t n_add_layers;
  const int64_t* add_layer_off; /* [n_add_layers + 1] */
  const int64_t *add_src, *add_dst;
  int64_t n_term_scales;
  const int64_t *ts_slot, *ts_factor;
} pse_graph_desc;

/* RunReport (executor.hpp:31-43) plus device timings, in milliseconds.
 * wall/conv/scale/add come from the kernels' own %globaltimer stamps of the
 * run (a phase ends when all of its jobs and those of the earlier phases are
 * done; executor.cpp:154-157 records the same per-phase split); per-layer
 * times: pse_plan_layer_ms. The other times are CUDA events on the plan's
 * stream. */
typedef struct {
  double wall_ms;  /* conv + scale + add phases (the paper's "wall") */
  double conv_ms, scale_ms, add_ms;
  double h2d_ms, d2h_ms, e2e_ms; /* pse_plan_run only: upload, download, whole call */
  int64_t double_op_count;       /* flop_count with reporting_cost(m), per point */
  int64_t alg_op_count;          /* executed-work model (instrumented_cost), per point */
  int64_t conv_jobs_executed, add_jobs_executed, copy_jobs_executed; /* all points */
  int32_t batch;
  int32_t kernel_launches; /* device kernels launched by the call */
  double device_ms;        /* events around the whole device evaluation (CUDA-graph replay) */
  double exchange_ms;      /* sharded plans (pse_plan_finish): conv end -> addition-stage start */
} pse_report;

const char* pse_last_error(void);
const char* pse_version(void);

/* ---- host graph compiler ---------------------------------------------- */
/* nvars[N]; indices[sum nvars] 1-based strictly increasing; exponents
 * [sum nvars] or NULL (a monomial whose exponents are all 0 has none) */
int pse_graph_build(int32_t n, int32_t d, int32_t N, const int32_t* nvars, const int32_t* indices,
                    const int32_t* exponents, pse_graph** out);
/* fills desc with pointers owned by g (valid until pse_graph_destroy) */
int pse_graph_describe(const pse_graph* g, int32_t m, int32_t mode, pse_graph_desc* desc);
void pse_graph_destroy(pse_graph* g);
/* 1 valid, 0 invalid (first violation in msg), <0 error */
int pse_graph_validate(const pse_graph_desc* desc, char* msg, size_t cap);
/* which: 0 total, 1 mul, 2 add; add_cost/mul_cost per md op */
int64_t pse_flop_count(const pse_graph_desc* desc, int32_t which, int64_t add_cost, int64_t mul_cost);
/* out[4] = instrumented add, instrumented mul, reporting add, reporting mul */
int pse_cost(int32_t m, int64_t* out);

/* ---- benchmark generator (gen.cpp:13-71, rng.hpp, multidouble.cpp:26-30) -- */
int pse_gen_benchmark_size(const char* id, int32_t* n, int32_t* N, int32_t* shape_len);
/* stat: [Q][1+N+n][d+1] (nullable: shape only) */
int pse_gen_benchmark(const char* id, int32_t d, int32_t m, int32_t mode, uint64_t seed, int32_t* nvars,
                      int32_t* indices, double* stat);

/* ---- problem files (problem_io.cpp:130-245; Problem, gen.hpp:14-19) ------- */
/* The reference's text format: hexfloat limbs (bit-exact round trip),
 * decimals accepted on input; parse errors return PSE_EINVAL with
 * "line N: ..." in pse_last_error() (ParseError, problem_io.hpp:15-24). */
typedef struct pse_problem pse_problem;
int pse_problem_parse(const char* text, pse_problem** out);
int pse_problem_read(const char* path, pse_problem** out);
int pse_problem_write(const pse_problem* p, const char* path);
/* text into buf (NUL-terminated, truncated to cap); *len = full length */
int pse_problem_text(const pse_problem* p, char* buf, size_t cap, size_t* len);
int pse_problem_create(const char* id, uint64_t seed, int32_t n, int32_t d, int32_t m, int32_t mode, int32_t N,
                       const int32_t* nvars, const int32_t* indices, const int32_t* exponents, const double* stat,
                       pse_problem** out);
int pse_problem_gen(const char* id, int32_t d, int32_t m, int32_t mode, uint64_t seed, pse_problem** out);
/* out[7] = n, N, d, m, mode, seed, shape length */
int pse_problem_info(const pse_problem* p, int64_t* out);
int pse_problem_id(const pse_problem* p, char* buf, size_t cap);
/* arrays owned by p; exponents NULL when none; stat [Q][1+N+n][d+1] */
int pse_problem_arrays(const pse_problem* p, const int32_t** nvars, const int32_t** indices,
                       const int32_t** exponents, const double** stat);
void pse_problem_destroy(pse_problem* p);

/* ---- device plan -------------------------------------------------------- */
/* Validates desc (as validate()), uploads the graph and allocates an arena
 * for up to max_batch points on `device`. */
int pse_plan_create(const pse_graph_desc* desc, int32_t device, int32_t max_batch, pse_plan** out);
void pse_plan_destroy(pse_plan* p);
/* upload `batch` points' static regions (copy + layout transform). The slab
 * pointers may be host memory or device memory already resident in HBM (a
 * D2D copy then). point_stride in doubles between consecutive points inside
 * each slab; 0 means static_top*(d+1) (packed). */
int pse_plan_upload(pse_plan* p, int32_t batch, const double* const* static_slabs, int64_t point_stride);
/* run all phases on the resident arena (device only); detail != 0 times every
 * phase with events, detail == 0 replays a captured CUDA graph */
int pse_plan_execute(pse_plan* p, int32_t batch, int32_t detail, pse_report* rep);
/* download value/gradient series and/or the dynamic arena (either nullable) */
int pse_plan_download(pse_plan* p, int32_t batch, double* const* value_grad_out, double* const* dyn_slabs_out);
/* one call = upload + execute + download, timed end to end: the run_sequential
 * contract over a DataArray (batch = 1) or a batch of points */
int pse_plan_run(pse_plan* p, int32_t batch, const double* const* static_slabs, int64_t point_stride,
                 double* const* dyn_slabs_out, double* const* value_grad_out, pse_report* rep);
/* per-layer phase times of the plan's last run (RunReport::conv_layer_ms /
 * add_layer_ms, executor.hpp:31-43, filled per phase at executor.cpp:154-157):
 * n_conv / n_add must equal the graph's conv / add layer counts */
int pse_plan_layer_ms(const pse_plan* p, double* conv_layer_ms, int32_t n_conv, double* add_layer_ms, int32_t n_add);
/* ---- one polynomial sharded over devices (one plan per GPU) --------------
 * Rank r's plan executes only the convolution jobs of its share of the
 * independent job groups (whole monomials, contiguous and balanced by job
 * count). The addition stage needs every term: each rank packs the dynamic
 * slots it produced (pse_plan_pack), the blocks are exchanged (e.g. NCCL
 * all-gather or peer copies over NVLink -- plain data movement, never an NCCL
 * sum, which would add limbs as plain doubles), every plan unpacks the
 * others' blocks and pse_plan_finish runs the term scales, the reference's
 * exact addition tree and the extraction with device md_adds. The result is
 * bit-identical to one device. pse_plan_execute on a sharded plan runs the
 * conv stage only. Buffers are device pointers. */
int pse_plan_create_sharded(const pse_graph_desc* desc, int32_t device, int32_t max_batch, int32_t rank,
                            int32_t nranks, pse_plan** out);
/* doubles in rank `rank`'s exchange block for `batch` points */
int pse_plan_exchange_words(const pse_plan* p, int32_t rank, int32_t batch, int64_t* words);
int pse_plan_pack(pse_plan* p, int32_t batch, double* dst);
int pse_plan_unpack(pse_plan* p, int32_t batch, int32_t src_rank, const double* src);
int pse_plan_finish(pse_plan* p, int32_t batch, int32_t detail, pse_report* rep);
/* The same exchange without staging buffers or a collective: each rank maps
 * the other ranks' arenas (CUDA IPC across processes -- NVLink peer memory on
 * one node -- or a plan of the same process) and, once every rank's conv
 * stage has finished (the caller's barrier), pse_plan_gather_peers copies the
 * slots each peer produced straight from the peer's arena into its own (one
 * kernel, peer loads). Then pse_plan_finish as above. */
#define PSE_IPC_HANDLE_BYTES 64
int pse_plan_arena_ipc_handle(const pse_plan* p, void* handle /* PSE_IPC_HANDLE_BYTES */);
int pse_plan_open_peer(pse_plan* p, int32_t rank, const void* handle);
int pse_plan_set_peer_arena(pse_plan* p, int32_t rank, const pse_plan* peer);
int pse_plan_gather_peers(pse_plan* p, int32_t batch);

/* plan geometry: out[8] = n, N, d, m, mode, total_slots, static_top, max_batch */
int pse_plan_info(const pse_plan* p, int64_t* out);
/* the plan's CUDA stream (cudaStream_t), for callers that time or order
 * their own work against the engine's */
int pse_plan_stream(const pse_plan* p, void** stream);
/* which convolution path a run of `batch` points takes (no reference
 * counterpart; for reporting): PSE_CONV_LAYERED (one launch per dependency
 * level, concurrent monomial groups, split chains for small layers),
 * PSE_CONV_WAVES (band x segment tasks, one launch per scheduled wave),
 * PSE_CONV_DATAFLOW (the same tasks in one persistent launch) or
 * PSE_CONV_HYBRID (layered for the large layers, then one dataflow launch
 * for the trailing small ones) or PSE_CONV_CTA (one block per independent job
 * group and point, the group's band tasks synchronised in shared memory) or
 * PSE_CONV_CTA_LAYERS (one block per independent job group and point, the
 * group's conv layers in order with a block barrier between them) */
enum {
  PSE_CONV_LAYERED = 1,
  PSE_CONV_WAVES = 2,
  PSE_CONV_DATAFLOW = 3,
  PSE_CONV_HYBRID = 4,
  PSE_CONV_CTA = 5,
  PSE_CONV_CTA_LAYERS = 6
};
int pse_plan_conv_path(const pse_plan* p, int32_t batch, int32_t* path);
/* host only (no device): the banded task schedule of a whole graph with band
 * width W (16 or 32), in dataflow order (flow != 0) or waves of `procs` warps;
 * the scheduler checks that every descriptor's dependencies precede it.
 * out[7] = {conv jobs, tasks, warp descriptors, waves, dependency entries,
 * occupied 8-lane slots, makespan estimate in steps} */
int pse_band_schedule_stats(const pse_graph_desc* desc, int32_t W, int32_t flow, int64_t procs, double slack,
                            int64_t* out);

/* evaluate() (executor.cpp:271-276): build graph, fold exponents (on the
 * device), stage, run, extract, for `batch` points sharing one polynomial
 * shape. stat: [Q][batch][1+N+n][d+1] (unfolded coefficients); vg_out:
 * [Q][batch][n+1][d+1]. */
int pse_evaluate(int32_t n, int32_t d, int32_t m, int32_t mode, int32_t N, const int32_t* nvars,
                 const int32_t* indices, const int32_t* exponents, int32_t batch, const double* stat,
                 double* vg_out, int32_t device, pse_report* rep);

/* eval_direct (oracle_direct.cpp:41-78) on the device: the INDEPENDENT
 * evaluator `verify` checks the engine against (proj/tools/pseval.cpp:97-118).
 * No job graph (each monomial's value and derivative terms are their own
 * left-to-right product chains, summed in monomial order) and the literal md
 * arithmetic (expansion.hpp restated over local arrays), not the engine's
 * register-streamed one. Refuses instances outside within_oracle_guard
 * (PSE_EINVAL, as the reference). stat: [Q][1+N+n][d+1] (one point, unfolded
 * coefficients); vg_out: [Q][n+1][d+1]. */
int pse_eval_direct(int32_t n, int32_t d, int32_t m, int32_t mode, int32_t N, const int32_t* nvars,
                    const int32_t* indices, const int32_t* exponents, const double* stat, double* vg_out,
                    int32_t device);
/* within_oracle_guard (oracle_direct.cpp:32-39): 1 inside, 0 outside, <0 error */
int pse_within_oracle_guard(int32_t d, int32_t N, const int32_t* nvars, const int32_t* exponents);

/* ---- primitives (host buffers; for tests and callers of the series ops) --- */
/* op: 0 add, 1 sub, 2 mul; impl: 0 register-streamed engine path, 1 literal;
 * x, y, out: [count][m] */
int pse_md_apply(int32_t op, int32_t m, int32_t impl, int64_t count, const double* x, const double* y,
                 double* out, int32_t device);
/* z = conv(x, y) for `count` independent pairs; x, y, z: [count][Q][d+1] */
int pse_series_conv(int32_t d, int32_t m, int32_t mode, int64_t count, const double* x, const double* y,
                    double* z, int32_t device);
/* z = series_add(x, y) (pseries.cpp:66-74: md_add per coefficient, x first)
 * and z = series_scale_int(x, factor) (pseries.cpp:85-93: md_mul by
 * md_from_double(factor); |factor| < 2^31) for `count` independent items;
 * x, y, z: [count][Q][d+1] */
int pse_series_add(int32_t d, int32_t m, int32_t mode, int64_t count, const double* x, const double* y,
                   double* z, int32_t device);
int pse_series_scale_int(int32_t d, int32_t m, int32_t mode, int64_t count, const double* x, int64_t factor,
                         double* z, int32_t device);

/* pinned host memory for end-to-end transfers */
void* pse_host_alloc(size_t bytes);
void pse_host_free(void* p);
/* out[4] = SM count, SM clock kHz, compute capability major*10+minor, device count */
int pse_device_info(int32_t device, int64_t* out);
/* measured FP64 issue rate (the conv roofline denominator): out[4] = DADD
 * lane-ops/s, DFMA lane-ops/s, blocks, ms of the DADD run */
int pse_fp64_peak(int32_t device, double* out);

#ifdef __cplusplus
}
#endif
#endif /* PSE_B200_H */
