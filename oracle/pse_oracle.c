/* TEST INFRASTRUCTURE ONLY -- the checker, never the product.
 *
 * Plain-C restatement of the reference CPU path of arXiv 2101.10881's artifact
 * (`pseval`, /root/reference/proj). Compiled with the reference's semantic
 * flags (-O3 -mfma -ffp-contract=off, proj/CMakeLists.txt:12-15) so every
 * +, *, fma rounds exactly as the reference's. Pinned against the reference
 * library (oracle/_ref) and the committed golden vectors in tests/golden/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 */
#include "pse_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXM 10
#define MAXNT (MAXM * (MAXM + 1) + (MAXM - 1))

static _Thread_local char g_err[256];
static int set_err(const char* m) {
  snprintf(g_err, sizeof g_err, "%s", m);
  return -1;
}
const char* pso_last_error(void) { return g_err; }

/* ---- op counting policy (expansion.hpp:18-29) ---- */
static _Thread_local long long g_ops;
static _Thread_local int g_count;
#define CNT(k)             \
  do {                     \
    if (g_count) g_ops += (k); \
  } while (0)

/* ---- error-free transforms (expansion.hpp:31-55) ---- */
static inline void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  double bv = ss - a;
  *e = (a - (ss - bv)) + (b - bv);
  *s = ss;
  CNT(6);
}
static inline void fast_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
  CNT(3);
}
static inline void two_prod(double a, double b, double* p, double* e) {
  double pp = a * b;
  *e = fma(a, b, -pp);
  *p = pp;
  CNT(3);
}

/* vec_sum (expansion.hpp:57-69): backward in-place error-free cascade */
static void vec_sum(double* x, int n) {
  double s = x[n - 1];
  for (int i = n - 2; i >= 0; --i) {
    double e;
    two_sum(x[i], s, &s, &e);
    x[i + 1] = e;
  }
  x[0] = s;
}

/* vec_sum_err_branch (expansion.hpp:71-90) */
static void vec_sum_err_branch(const double* e, int n, double* out, int m) {
  int j = 0;
  double eps = e[0];
  for (int i = 1; i < n; ++i) {
    double r, t;
    fast_two_sum(eps, e[i], &r, &t);
    if (t != 0.0) {
      out[j++] = r;
      if (j == m) return;
      eps = t;
    } else {
      eps = r;
    }
  }
  out[j++] = eps;
  while (j < m) out[j++] = 0.0;
}

/* tighten (expansion.hpp:92-114): bitwise fixed point of adjacent two_sums */
static void tighten(double* w, int m) {
  for (int pass = 0; pass < m; ++pass) {
    int changed = 0;
    for (int i = 0; i + 1 < m; ++i) {
      double s, e;
      two_sum(w[i], w[i + 1], &s, &e);
      uint64_t bs, bw0, be, bw1;
      memcpy(&bs, &s, 8);
      memcpy(&bw0, &w[i], 8);
      memcpy(&be, &e, 8);
      memcpy(&bw1, &w[i + 1], 8);
      if (bs != bw0 || be != bw1) {
        w[i] = s;
        w[i + 1] = e;
        changed = 1;
      }
    }
    if (!changed) return;
  }
}

/* exp_add (expansion.hpp:142-158) */
static void exp_add(int M, const double* x, const double* y, double* out) {
  if (M == 1) {
    out[0] = x[0] + y[0];
    CNT(1);
    return;
  }
  double t[2 * MAXM];
  int i = 0, j = 0, p = 0;
  while (i < M && j < M) t[p++] = fabs(x[i]) >= fabs(y[j]) ? x[i++] : y[j++];
  while (i < M) t[p++] = x[i++];
  while (j < M) t[p++] = y[j++];
  vec_sum(t, 2 * M);
  vec_sum_err_branch(t, 2 * M, out, M);
  tighten(out, M);
}

/* exp_sub (expansion.hpp:160-170) */
static void exp_sub(int M, const double* x, const double* y, double* out) {
  if (M == 1) {
    out[0] = x[0] - y[0];
    CNT(1);
    return;
  }
  double ny[MAXM];
  for (int k = 0; k < M; ++k) ny[k] = -y[k];
  exp_add(M, x, ny, out);
}

/* exp_mul (expansion.hpp:177-211): diagonal-grouped partial products with
 * each diagonal's two_prod errors deferred to the next diagonal */
static void exp_mul(int M, const double* x, const double* y, double* out) {
  if (M == 1) {
    out[0] = x[0] * y[0];
    CNT(1);
    return;
  }
  const int NT = M * (M + 1) + (M - 1);
  double t[MAXNT], carry[MAXM], next[MAXM];
  int pos = 0, ncarry = 0;
  for (int k = 0; k <= M; ++k) {
    int nn = 0;
    int ilo = k - (M - 1) > 0 ? k - (M - 1) : 0;
    int ihi = k < M - 1 ? k : M - 1;
    for (int i = ilo; i <= ihi; ++i) {
      if (k < M) {
        double pr, er;
        two_prod(x[i], y[k - i], &pr, &er);
        t[pos++] = pr;
        next[nn++] = er;
      } else {
        t[pos++] = x[i] * y[k - i];
        CNT(1);
      }
    }
    for (int c = 0; c < ncarry; ++c) t[pos++] = carry[c];
    for (int c = 0; c < nn; ++c) carry[c] = next[c];
    ncarry = nn;
  }
  vec_sum(t, NT);
  vec_sum(t, NT);
  vec_sum_err_branch(t, NT, out, M);
  tighten(out, M);
}

static int valid_m(int m) {
  return m == 1 || m == 2 || m == 3 || m == 4 || m == 5 || m == 8 || m == 10;
}

int pso_md_op(int op, int m, int64_t count, const double* x, const double* y, double* out) {
  if (!valid_m(m)) return set_err("unsupported precision level");
  double r[MAXM];
  for (int64_t c = 0; c < count; ++c) {
    const double* a = x + c * m;
    const double* b = y + c * m;
    if (op == 0)
      exp_add(m, a, b, r);
    else if (op == 1)
      exp_sub(m, a, b, r);
    else
      exp_mul(m, a, b, r);
    memcpy(out + c * m, r, sizeof(double) * (size_t)m);
  }
  return 0;
}

/* ---- Rng: std::mt19937_64 + explicit bit mappings (rng.hpp:11-36) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt_seed(mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt_next(mt64* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

static double rng_pm1(mt64* r) { return (double)(mt_next(r) >> 11) * 0x1p-52 - 1.0; }

uint64_t pso_mix_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void pso_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
  mt64 r;
  mt_seed(&r, seed);
  for (int64_t c = 0; c < count; ++c) out[c] = mt_next(&r);
}

static int is_normalized(const double* limb, int m) {
  int last = -1, seen_zero = 0;
  for (int i = 0; i < m; ++i) {
    if (limb[i] == 0.0) {
      seen_zero = 1;
      continue;
    }
    if (seen_zero || !isfinite(limb[i])) return 0;
    if (last >= 0) {
      int e = ilogb(limb[last]);
      double ulp = ldexp(1.0, e - 52 < -1074 ? -1074 : e - 52);
      if (fabs(limb[i]) > 0.5 * ulp) return 0;
    }
    last = i;
  }
  return 1;
}

/* renormalize (multidouble.cpp:9-24) */
static void renormalize(const double* in, int n, int m, double* out) {
  for (int l = 0; l < m; ++l) out[l] = 0.0;
  if (n == 0) return;
  if (n == m && is_normalized(in, m)) {
    memcpy(out, in, sizeof(double) * (size_t)m);
    return;
  }
  double t[MAXNT + 8];
  memcpy(t, in, sizeof(double) * (size_t)n);
  vec_sum(t, n);
  vec_sum(t, n);
  vec_sum_err_branch(t, n, out, m);
  tighten(out, m);
}

int pso_renormalize(const double* t, int n, int m, double* out) {
  if (!valid_m(m) || n > MAXNT) return set_err("bad renormalize arguments");
  renormalize(t, n, m, out);
  return 0;
}

/* random_md (multidouble.cpp:26-30) */
static void random_md(mt64* r, int m, double* out) {
  double t[MAXM];
  for (int k = 0; k < m; ++k) t[k] = rng_pm1(r) * ldexp(1.0, -53 * k);
  renormalize(t, m, m, out);
}

void pso_random_md(uint64_t seed, int m, int64_t count, double* out) {
  mt64 r;
  mt_seed(&r, seed);
  for (int64_t c = 0; c < count; ++c) random_md(&r, m, out + c * m);
}

/* instrumented_cost measure() (multidouble.cpp:36-56) and reporting_cost (:70-75) */
int pso_cost(int m, int64_t* out) {
  if (!valid_m(m)) return set_err("unsupported precision level");
  mt64 r;
  mt_seed(&r, pso_mix_seed(0x705e5a1cULL, (uint64_t)m));
  long long wa = 0, wm = 0;
  double x[MAXM], y[MAXM], z[MAXM];
  for (int s = 0; s < 64; ++s) {
    random_md(&r, m, x);
    random_md(&r, m, y);
    g_count = 1;
    g_ops = 0;
    exp_add(m, x, y, z);
    if (g_ops > wa) wa = g_ops;
    g_ops = 0;
    exp_mul(m, x, y, z);
    if (g_ops > wm) wm = g_ops;
    g_count = 0;
  }
  out[0] = wa;
  out[1] = wm;
  if (m == 1) {
    out[2] = 1;
    out[3] = 1;
  } else if (m == 10) {
    out[2] = 397;
    out[3] = 3089;
  } else {
    out[2] = wa;
    out[3] = wm;
  }
  return 0;
}

/* ---- series (pseries.cpp) : AoS series s[(k*P + part)*m + l] ---- */
typedef struct {
  int d, m, P;
} sdim;

static inline double* co(double* s, sdim D, int k, int part) { return s + ((size_t)k * D.P + part) * D.m; }
static inline const double* cco(const double* s, sdim D, int k, int part) {
  return s + ((size_t)k * D.P + part) * D.m;
}
static size_t slen(sdim D) { return (size_t)(D.d + 1) * D.P * D.m; }

/* conv (pseries.cpp:37-64) */
static void conv(sdim D, const double* x, const double* y, double* z) {
  const int M = D.m;
  double acc_re[MAXM], acc_im[MAXM], a[MAXM], b[MAXM], c[MAXM], e[MAXM], pre[MAXM], pim[MAXM];
  for (int k = 0; k <= D.d; ++k) {
    for (int i = 0; i <= k; ++i) {
      const double* xr = cco(x, D, i, 0);
      const double* yr = cco(y, D, k - i, 0);
      if (D.P == 1) {
        exp_mul(M, xr, yr, pre);
        if (i == 0)
          memcpy(acc_re, pre, sizeof(double) * (size_t)M);
        else
          exp_add(M, acc_re, pre, acc_re);
      } else {
        const double* xi = cco(x, D, i, 1);
        const double* yi = cco(y, D, k - i, 1);
        exp_mul(M, xr, yr, a);
        exp_mul(M, xi, yi, b);
        exp_sub(M, a, b, pre);
        exp_mul(M, xr, yi, c);
        exp_mul(M, xi, yr, e);
        exp_add(M, c, e, pim);
        if (i == 0) {
          memcpy(acc_re, pre, sizeof(double) * (size_t)M);
          memcpy(acc_im, pim, sizeof(double) * (size_t)M);
        } else {
          exp_add(M, acc_re, pre, acc_re);
          exp_add(M, acc_im, pim, acc_im);
        }
      }
    }
    memcpy(co(z, D, k, 0), acc_re, sizeof(double) * (size_t)M);
    if (D.P == 2) memcpy(co(z, D, k, 1), acc_im, sizeof(double) * (size_t)M);
  }
}

int pso_series_conv(int d, int m, int cplx, const double* x, const double* y, double* out) {
  if (!valid_m(m) || d < 0) return set_err("bad series arguments");
  sdim D = {d, m, cplx ? 2 : 1};
  size_t L = slen(D);
  double* xs = malloc(L * 8);
  double* ys = malloc(L * 8);
  double* zs = malloc(L * 8);
  /* [P][m][d+1] -> AoS */
  for (int p = 0; p < D.P; ++p)
    for (int l = 0; l < m; ++l)
      for (int k = 0; k <= d; ++k) {
        co(xs, D, k, p)[l] = x[((size_t)p * m + l) * (d + 1) + k];
        co(ys, D, k, p)[l] = y[((size_t)p * m + l) * (d + 1) + k];
      }
  conv(D, xs, ys, zs);
  for (int p = 0; p < D.P; ++p)
    for (int l = 0; l < m; ++l)
      for (int k = 0; k <= d; ++k) out[((size_t)p * m + l) * (d + 1) + k] = co(zs, D, k, p)[l];
  free(xs);
  free(ys);
  free(zs);
  return 0;
}

/* series_add (pseries.cpp:66-74) */
static void series_add(sdim D, const double* x, const double* y, double* z) {
  for (int k = 0; k <= D.d; ++k)
    for (int p = 0; p < D.P; ++p) exp_add(D.m, cco(x, D, k, p), cco(y, D, k, p), co(z, D, k, p));
}

/* series_scale_int (pseries.cpp:85-93) */
static void series_scale_int(sdim D, const double* x, long c, double* z) {
  double cm[MAXM] = {0};
  cm[0] = (double)c;
  for (int k = 0; k <= D.d; ++k)
    for (int p = 0; p < D.P; ++p) exp_mul(D.m, cco(x, D, k, p), cm, co(z, D, k, p));
}

/* ---- job graph (jobgraph.cpp) ---- */
struct pso_graph {
  int n, N, d;
  long total_slots;
  int nconv_layers, nadd_layers;
  long nconv, nadd, nts;
  long* conv; /* rows: layer, in1, in2, out, copy (sorted by layer, stable) */
  long* add;  /* rows: layer, src, dst */
  long value_slot;
  long* grad_slots;
  long* mult;
  long* ts; /* rows: slot, factor */
};

typedef struct {
  int n, N;
  long *alpha, *beta, *gamma;
  long total_slots;
} offs;

static long f_base(const offs* o) { return 1 + o->N + o->n; }
static long f_slot(const offs* o, int k, int l) { return f_base(o) + o->alpha[k] + (l - 1); }
static long b_slot(const offs* o, int k, int l) { return f_base(o) + o->beta[k] + (l - 1); }
static long c_slot(const offs* o, int k, int j) { return f_base(o) + o->gamma[k] + (j - 1); }
static long z_slot(const offs* o, int i) { return o->N + i; }
static long a_slot(int k) { return 1 + k; }

static void push(long** arr, long* n, long* cap, const long* row, int w) {
  if (*n >= *cap) {
    *cap = *cap ? *cap * 2 : 1024;
    *arr = realloc(*arr, sizeof(long) * (size_t)(*cap) * (size_t)w);
  }
  memcpy(*arr + (*n) * w, row, sizeof(long) * (size_t)w);
  ++*n;
}

/* stable counting sort of rows by column 0 (layer, 1-based) */
static void sort_by_layer(long* rows, long n, int w, int nlayers) {
  long* cnt = calloc((size_t)nlayers + 2, sizeof(long));
  for (long r = 0; r < n; ++r) cnt[rows[r * w]]++;
  long acc = 0;
  for (int L = 0; L <= nlayers + 1; ++L) {
    long c = cnt[L];
    cnt[L] = acc;
    acc += c;
  }
  long* tmp = malloc(sizeof(long) * (size_t)(n * w + 1));
  for (long r = 0; r < n; ++r) memcpy(tmp + (cnt[rows[r * w]]++) * w, rows + r * w, sizeof(long) * (size_t)w);
  memcpy(rows, tmp, sizeof(long) * (size_t)(n * w));
  free(tmp);
  free(cnt);
}

pso_graph* pso_graph_build(int n, int d, int N, const int* nvars, const int* idx, const int* exps) {
  /* check_polynomial (jobgraph.cpp:41-63) */
  if (n < 1) return set_err("polynomial needs at least one variable"), NULL;
  if (N < 1) return set_err("polynomial needs at least one monomial"), NULL;
  long* start = malloc(sizeof(long) * (size_t)(N + 1));
  start[0] = 0;
  for (int k = 0; k < N; ++k) {
    if (nvars[k] < 1) return free(start), set_err("monomial without variables"), NULL;
    start[k + 1] = start[k] + nvars[k];
    int prev = 0;
    for (int j = 0; j < nvars[k]; ++j) {
      int i = idx[start[k] + j];
      if (i <= prev) return free(start), set_err("monomial indices must be strictly increasing"), NULL;
      if (i > n) return free(start), set_err("monomial index out of range"), NULL;
      prev = i;
      if (exps && exps[start[k] + j] < 0) return free(start), set_err("exponents must be positive"), NULL;
    }
  }
  /* offsets (jobgraph.cpp:65-88) */
  offs o;
  o.n = n;
  o.N = N;
  o.alpha = calloc((size_t)N + 1, sizeof(long));
  o.beta = calloc((size_t)N + 1, sizeof(long));
  o.gamma = calloc((size_t)N + 1, sizeof(long));
  for (int k = 0; k < N; ++k) {
    long nk = nvars[k];
    o.alpha[k + 1] = o.alpha[k] + nk;
    o.beta[k + 1] = o.beta[k] + (nk - 2 > 1 ? nk - 2 : 1);
    o.gamma[k + 1] = o.gamma[k] + (nk - 2 > 0 ? nk - 2 : 0);
  }
  long fext = o.alpha[N], bext = o.beta[N];
  for (int k = 0; k <= N; ++k) {
    o.beta[k] += fext;
    o.gamma[k] += fext + bext;
  }
  o.total_slots = f_base(&o) + o.gamma[N];

  pso_graph* g = calloc(1, sizeof *g);
  g->n = n;
  g->N = N;
  g->d = d;
  g->total_slots = o.total_slots;
  long cap = 0;
  int maxlayer = 0;
  /* monomial_conv_jobs (jobgraph.cpp:90-124) */
  for (int k = 0; k < N; ++k) {
    const int nk = nvars[k];
    const int* ix = idx + start[k];
#define Z(pos) z_slot(&o, ix[(pos)-1])
#define JOB(i1, i2, ou, lay, cp)                        \
  do {                                                   \
    long row[5] = {(lay), (i1), (i2), (ou), (cp)};       \
    push(&g->conv, &g->nconv, &cap, row, 5);             \
    if ((lay) > maxlayer) maxlayer = (lay);              \
  } while (0)
    JOB(a_slot(k), Z(1), f_slot(&o, k, 1), 1, 0);
    for (int l = 2; l <= nk; ++l) JOB(f_slot(&o, k, l - 1), Z(l), f_slot(&o, k, l), l, 0);
    if (nk == 1) {
      JOB(a_slot(k), 0, b_slot(&o, k, 1), 1, 1);
      continue;
    }
    if (nk == 2) {
      JOB(Z(2), a_slot(k), b_slot(&o, k, 1), 1, 0);
      continue;
    }
    JOB(Z(nk), Z(nk - 1), b_slot(&o, k, 1), 1, 0);
    for (int l = 2; l <= nk - 2; ++l) JOB(b_slot(&o, k, l - 1), Z(nk - l), b_slot(&o, k, l), l, 0);
    JOB(b_slot(&o, k, nk - 2), a_slot(k), b_slot(&o, k, nk - 2), nk - 1, 0);
    for (int j = 1; j <= nk - 3; ++j) {
      int layer = (j > nk - 2 - j ? j : nk - 2 - j) + 1;
      JOB(f_slot(&o, k, j), b_slot(&o, k, nk - 2 - j), c_slot(&o, k, j), layer, 0);
    }
    JOB(f_slot(&o, k, nk - 2), Z(nk), c_slot(&o, k, nk - 2), nk - 1, 0);
#undef JOB
#undef Z
  }
  g->nconv_layers = maxlayer;
  sort_by_layer(g->conv, g->nconv, 5, maxlayer);

  /* gradient_term_map (jobgraph.cpp:149-166): per-variable lists in monomial order */
  long* gcnt = calloc((size_t)n, sizeof(long));
  for (int k = 0; k < N; ++k)
    for (int j = 0; j < nvars[k]; ++j) gcnt[idx[start[k] + j] - 1]++;
  long** glist = calloc((size_t)n, sizeof(long*));
  long* gfill = calloc((size_t)n, sizeof(long));
  for (int i = 0; i < n; ++i) glist[i] = malloc(sizeof(long) * (size_t)(gcnt[i] + 1));
  for (int k = 0; k < N; ++k) {
    const int nk = nvars[k];
    for (int j = 1; j <= nk; ++j) {
      long slot;
      if (j == nk && nk >= 2)
        slot = f_slot(&o, k, nk - 1);
      else if (j == 1)
        slot = nk >= 3 ? b_slot(&o, k, nk - 2) : b_slot(&o, k, 1);
      else
        slot = c_slot(&o, k, j - 1);
      int var = idx[start[k] + j - 1] - 1;
      glist[var][gfill[var]++] = slot;
    }
  }

  /* addition_schedule (jobgraph.cpp:126-147) over [value list] + non-empty gradient lists */
  long acap = 0;
  int maxadd = 0;
  long* surv = malloc(sizeof(long) * (size_t)(N + 2));
  long* nxt = malloc(sizeof(long) * (size_t)(N + 2));
  for (int li = -1; li < n; ++li) {
    long cnt;
    if (li < 0) {
      cnt = N + 1;
      surv[0] = 0;
      for (int k = 0; k < N; ++k) surv[k + 1] = f_slot(&o, k, nvars[k]);
    } else {
      cnt = gfill[li];
      if (cnt == 0) continue;
      memcpy(surv, glist[li], sizeof(long) * (size_t)cnt);
    }
    int level = 1;
    while (cnt > 1) {
      long nn = 0, t = 0;
      for (; t + 1 < cnt; t += 2) {
        long row[3] = {level, surv[t], surv[t + 1]};
        push(&g->add, &g->nadd, &acap, row, 3);
        nxt[nn++] = surv[t + 1];
      }
      if (t < cnt) nxt[nn++] = surv[t];
      memcpy(surv, nxt, sizeof(long) * (size_t)nn);
      cnt = nn;
      if (level > maxadd) maxadd = level;
      ++level;
    }
  }
  g->nadd_layers = maxadd;
  sort_by_layer(g->add, g->nadd, 3, maxadd);
  free(surv);
  free(nxt);

  /* value / gradient slots, multipliers, term scales (jobgraph.cpp:226-261) */
  g->value_slot = f_slot(&o, N - 1, nvars[N - 1]);
  g->grad_slots = malloc(sizeof(long) * (size_t)n);
  g->mult = malloc(sizeof(long) * (size_t)n);
  /* seen exponent set per variable: track the first value and whether a second differs */
  long* first = malloc(sizeof(long) * (size_t)n);
  int* state = calloc((size_t)n, sizeof(int)); /* 0 none, 1 uniform, 2 mixed */
  for (int k = 0; k < N; ++k) {
    int any = 0;
    if (exps)
      for (int j = 0; j < nvars[k]; ++j) any |= exps[start[k] + j] != 0;
    for (int j = 0; j < nvars[k]; ++j) {
      long e = any ? exps[start[k] + j] : 1;
      int var = idx[start[k] + j] - 1;
      if (state[var] == 0) {
        state[var] = 1;
        first[var] = e;
      } else if (state[var] == 1 && first[var] != e) {
        state[var] = 2;
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    g->grad_slots[i] = gfill[i] ? glist[i][gfill[i] - 1] : -1;
    g->mult[i] = state[i] == 1 ? first[i] : 1;
  }
  long tcap = 0;
  long* cursor = calloc((size_t)n, sizeof(long));
  for (int k = 0; k < N; ++k) {
    int any = 0;
    if (exps)
      for (int j = 0; j < nvars[k]; ++j) any |= exps[start[k] + j] != 0;
    for (int j = 0; j < nvars[k]; ++j) {
      int var = idx[start[k] + j] - 1;
      long slot = glist[var][cursor[var]++];
      long e = any ? exps[start[k] + j] : 1;
      if (state[var] == 2 && e != 1) {
        long row[2] = {slot, e};
        push(&g->ts, &g->nts, &tcap, row, 2);
      }
    }
  }
  free(cursor);
  free(first);
  free(state);
  for (int i = 0; i < n; ++i) free(glist[i]);
  free(glist);
  free(gfill);
  free(gcnt);
  free(start);
  free(o.alpha);
  free(o.beta);
  free(o.gamma);
  return g;
}

void pso_graph_free(pso_graph* g) {
  if (!g) return;
  free(g->conv);
  free(g->add);
  free(g->grad_slots);
  free(g->mult);
  free(g->ts);
  free(g);
}

void pso_graph_info(const pso_graph* g, int64_t* info) {
  long ncopy = 0;
  for (long r = 0; r < g->nconv; ++r) ncopy += g->conv[r * 5 + 4];
  int64_t v[] = {g->n, g->N, g->d, g->total_slots, g->nconv, g->nadd, ncopy,
                 g->nconv_layers, g->nadd_layers, g->nts};
  memcpy(info, v, sizeof v);
}

void pso_graph_export(const pso_graph* g, int64_t* conv, int64_t* add, int64_t* value_slot,
                      int64_t* grad_slots, int64_t* mult, int64_t* ts) {
  for (long r = 0; r < g->nconv * 5; ++r) conv[r] = g->conv[r];
  for (long r = 0; r < g->nadd * 3; ++r) add[r] = g->add[r];
  *value_slot = g->value_slot;
  for (int i = 0; i < g->n; ++i) {
    grad_slots[i] = g->grad_slots[i];
    mult[i] = g->mult[i];
  }
  for (long r = 0; r < g->nts * 2; ++r) ts[r] = g->ts[r];
}

/* validate (jobgraph.cpp:273-336) */
int pso_graph_validate(const pso_graph* g, char* msg, int cap) {
  const long top = 1 + g->N + g->n;
  int* first_write = malloc(sizeof(int) * (size_t)g->total_slots);
  int* wlayer = malloc(sizeof(int) * (size_t)g->total_slots); /* layer of write in current layer */
  for (long s = 0; s < g->total_slots; ++s) first_write[s] = -1, wlayer[s] = -1;
  int ok = 1;
#define BAD(...)                          \
  do {                                    \
    if (msg) snprintf(msg, (size_t)cap, __VA_ARGS__); \
    ok = 0;                               \
    goto done;                            \
  } while (0)
  long r = 0;
  for (int L = 0; L < g->nconv_layers; ++L) {
    long r0 = r;
    while (r < g->nconv && g->conv[r * 5] == L + 1) {
      const long* j = g->conv + r * 5;
      if (j[3] < top || j[3] >= g->total_slots) BAD("conv layer %d: writes outside the dynamic region", L + 1);
      if (wlayer[j[3]] == L) BAD("conv layer %d: duplicate write in one layer", L + 1);
      wlayer[j[3]] = L;
      if (!j[4] && j[3] == j[2]) BAD("conv layer %d: output aliases second input", L + 1);
      ++r;
    }
    for (long q = r0; q < r; ++q) {
      const long* j = g->conv + q * 5;
      long ins[2] = {j[1], j[4] ? j[1] : j[2]};
      for (int t = 0; t < 2; ++t) {
        long s = ins[t];
        if (s < 0 || s >= g->total_slots) BAD("conv layer %d: input slot out of range", L + 1);
        if (s < top) continue;
        if (!(first_write[s] >= 0 && first_write[s] < L))
          BAD("conv layer %d: reads slot %ld not written in an earlier layer", L + 1, s);
        if (wlayer[s] == L && s != j[3])
          BAD("conv layer %d: reads slot %ld written by another job in the same layer", L + 1, s);
      }
    }
    for (long q = r0; q < r; ++q) {
      long o = g->conv[q * 5 + 3];
      if (first_write[o] < 0) first_write[o] = L;
    }
  }
  r = 0;
  for (int L = 0; L < g->nadd_layers; ++L) {
    while (r < g->nadd && g->add[r * 3] == L + 1) {
      const long* j = g->add + r * 3;
      if (j[1] == j[2]) BAD("add layer %d: source equals destination", L + 1);
      for (int t = 1; t <= 2; ++t) {
        long s = j[t];
        if (s < 0 || s >= g->total_slots) BAD("add layer %d: slot out of range", L + 1);
        if (s >= top && first_write[s] < 0) BAD("add layer %d: slot %ld never written by a conv job", L + 1, s);
      }
      if (j[2] < top) BAD("add layer %d: accumulates into a static slot", L + 1);
      if (wlayer[j[2]] == 1000000 + L) BAD("add layer %d: duplicate write in one layer", L + 1);
      wlayer[j[2]] = 1000000 + L;
      ++r;
    }
  }
  for (long s = top; s < g->total_slots; ++s)
    if (first_write[s] < 0) BAD("slot %ld is never written", s);
done:
#undef BAD
  free(first_write);
  free(wlayer);
  return ok;
}

/* flop_count* (executor.cpp:233-252) */
int64_t pso_flop_count(const pso_graph* g, int d, int cplx, int64_t add_cost, int64_t mul_cost, int which) {
  long ncopy = 0;
  for (long r = 0; r < g->nconv; ++r) ncopy += g->conv[r * 5 + 4];
  const long long C = g->nconv - ncopy, A = g->nadd, d1 = d + 1;
  const long long mul = C * d1 * d1 * (cplx ? 4 : 1) * mul_cost;
  long long conv_adds = C * d * d1;
  if (cplx) conv_adds = conv_adds * 2 + C * d1 * d1 * 2;
  const long long add = (conv_adds + A * d1 * (cplx ? 2 : 1)) * add_cost;
  return which == 1 ? mul : which == 2 ? add : mul + add;
}

/* ---- gen_benchmark (gen.cpp:13-71) ---- */
static int shape_dims(const char* id, int* n, int* N, int* len) {
  if (!strcmp(id, "p1")) *n = 16, *N = 1820, *len = 1820 * 4;
  else if (!strcmp(id, "p2")) *n = 128, *N = 128, *len = 128 * 64;
  else if (!strcmp(id, "p3")) *n = 128, *N = 8128, *len = 8128 * 2;
  else return set_err("unknown benchmark polynomial id");
  return 0;
}

int pso_gen_shape_size(const char* id, int* n, int* N, int* shape_len) { return shape_dims(id, n, N, shape_len); }

static int cmp_int(const void* a, const void* b) { return *(const int*)a - *(const int*)b; }

/* combinations (gen.cpp:13-26): lexicographic r-subsets of 1..n */
static void combinations(int n, int r, int* nvars, int* idx) {
  int c[8];
  for (int i = 0; i < r; ++i) c[i] = i + 1;
  long k = 0;
  for (;;) {
    nvars[k] = r;
    memcpy(idx + k * r, c, sizeof(int) * (size_t)r);
    ++k;
    int i = r - 1;
    while (i >= 0 && c[i] == n - (r - 1 - i)) --i;
    if (i < 0) break;
    ++c[i];
    for (int j = i + 1; j < r; ++j) c[j] = c[j - 1] + 1;
  }
}

static void random_series_block(uint64_t seed, int d, int m, int P, double* stat, long top, long row) {
  mt64 r;
  mt_seed(&r, seed);
  double v[MAXM];
  /* random_series (pseries.cpp:95-103): per coefficient re then im */
  for (int k = 0; k <= d; ++k)
    for (int p = 0; p < P; ++p) {
      random_md(&r, m, v);
      for (int l = 0; l < m; ++l) stat[(((size_t)p * m + l) * top + row) * (d + 1) + k] = v[l];
    }
}

int pso_gen_benchmark(const char* id, int d, int m, int cplx, uint64_t seed, int* nvars, int* idx, double* stat) {
  int n, N, len;
  if (shape_dims(id, &n, &N, &len)) return -1;
  if (!valid_m(m)) return set_err("unsupported precision level");
  if (!strcmp(id, "p1"))
    combinations(16, 4, nvars, idx);
  else if (!strcmp(id, "p3"))
    combinations(128, 2, nvars, idx);
  else
    for (int k = 0; k < 128; ++k) {
      nvars[k] = 64;
      for (int j = 0; j < 64; ++j) idx[k * 64 + j] = (k + j) % 128 + 1;
      qsort(idx + k * 64, 64, sizeof(int), cmp_int);
    }
  if (!stat) return 0;
  const int P = cplx ? 2 : 1;
  const long top = 1L + N + n;
  random_series_block(pso_mix_seed(seed, 1ULL << 32), d, m, P, stat, top, 0);
  for (int k = 0; k < N; ++k) random_series_block(pso_mix_seed(seed, (2ULL << 32) + (uint64_t)k), d, m, P, stat, top, 1 + k);
  for (int i = 0; i < n; ++i) random_series_block(pso_mix_seed(seed, (3ULL << 32) + (uint64_t)i), d, m, P, stat, top, N + 1 + i);
  return 0;
}

/* ---- engine: stage + run_sequential + extract (executor.cpp:69-269) ---- */
/* arena: limb-major slabs [P][m][total_slots][d+1] like DataArray (executor.hpp:17-29) */
static void read_slot(const double* arena, sdim D, long TS, long slot, double* s) {
  for (int p = 0; p < D.P; ++p)
    for (int l = 0; l < D.m; ++l) {
      const double* src = arena + (((size_t)p * D.m + l) * TS + slot) * (D.d + 1);
      for (int k = 0; k <= D.d; ++k) co(s, D, k, p)[l] = src[k];
    }
}
static void write_slot(double* arena, sdim D, long TS, long slot, const double* s) {
  for (int p = 0; p < D.P; ++p)
    for (int l = 0; l < D.m; ++l) {
      double* dst = arena + (((size_t)p * D.m + l) * TS + slot) * (D.d + 1);
      for (int k = 0; k <= D.d; ++k) dst[k] = cco(s, D, k, p)[l];
    }
}
static void read_block(const double* stat, sdim D, long top, long row, double* s) {
  for (int p = 0; p < D.P; ++p)
    for (int l = 0; l < D.m; ++l)
      for (int k = 0; k <= D.d; ++k) co(s, D, k, p)[l] = stat[(((size_t)p * D.m + l) * top + row) * (D.d + 1) + k];
}
static void write_block(double* out, sdim D, long rows, long row, const double* s) {
  for (int p = 0; p < D.P; ++p)
    for (int l = 0; l < D.m; ++l)
      for (int k = 0; k <= D.d; ++k) out[(((size_t)p * D.m + l) * rows + row) * (D.d + 1) + k] = cco(s, D, k, p)[l];
}

/* fold_exponents (jobgraph.cpp:168-187): a' = a * prod z^(e-1) with a power table */
static void fold(sdim D, const double* coeff, int nk, const int* ix, const int* ex, const double* stat, long top,
                 int N, double* out) {
  size_t L = slen(D);
  double* power = malloc(L * 8);
  double* zi = malloc(L * 8);
  double* tmp = malloc(L * 8);
  memcpy(out, coeff, L * 8);
  for (int j = 0; j < nk; ++j) {
    int e = ex[j];
    if (e <= 1) continue;
    read_block(stat, D, top, N + ix[j], zi);
    memcpy(power, zi, L * 8);
    for (int q = 2; q <= e - 1; ++q) {
      conv(D, power, zi, tmp);
      memcpy(power, tmp, L * 8);
    }
    conv(D, out, power, tmp);
    memcpy(out, tmp, L * 8);
  }
  free(power);
  free(zi);
  free(tmp);
}

int pso_evaluate(int n, int d, int m, int cplx, int N, const int* nvars, const int* idx, const int* exps,
                 const double* stat, double* vg_out, double* dyn_out) {
  if (!valid_m(m)) return set_err("unsupported precision level");
  pso_graph* g = pso_graph_build(n, d, N, nvars, idx, exps);
  if (!g) return -1;
  sdim D = {d, m, cplx ? 2 : 1};
  const long TS = g->total_slots, top = 1L + N + n;
  size_t L = slen(D);
  double* arena = calloc((size_t)D.P * m * (size_t)TS * (size_t)(d + 1), sizeof(double));
  double* x = malloc(L * 8);
  double* y = malloc(L * 8);
  double* z = malloc(L * 8);
  /* fold_polynomial + stage (executor.cpp:69-96) */
  long pos = 0;
  read_block(stat, D, top, 0, x);
  write_slot(arena, D, TS, 0, x);
  for (int k = 0; k < N; ++k) {
    read_block(stat, D, top, 1 + k, x);
    int any = 0;
    if (exps)
      for (int j = 0; j < nvars[k]; ++j) any |= exps[pos + j] > 1;
    if (any) {
      fold(D, x, nvars[k], idx + pos, exps + pos, stat, top, N, y);
      write_slot(arena, D, TS, 1 + k, y);
    } else {
      write_slot(arena, D, TS, 1 + k, x);
    }
    pos += nvars[k];
  }
  for (int i = 1; i <= n; ++i) {
    read_block(stat, D, top, N + i, x);
    write_slot(arena, D, TS, N + i, x);
  }
  /* run_sequential: conv layers, scale phase, add layers (executor.cpp:100-183) */
  for (long r = 0; r < g->nconv; ++r) {
    const long* j = g->conv + r * 5;
    read_slot(arena, D, TS, j[1], x);
    if (j[4]) {
      write_slot(arena, D, TS, j[3], x);
      continue;
    }
    read_slot(arena, D, TS, j[2], y);
    conv(D, x, y, z);
    write_slot(arena, D, TS, j[3], z);
  }
  for (long r = 0; r < g->nts; ++r) {
    read_slot(arena, D, TS, g->ts[2 * r], x);
    series_scale_int(D, x, g->ts[2 * r + 1], z);
    write_slot(arena, D, TS, g->ts[2 * r], z);
  }
  for (long r = 0; r < g->nadd; ++r) {
    const long* j = g->add + r * 3;
    read_slot(arena, D, TS, j[2], x);
    read_slot(arena, D, TS, j[1], y);
    series_add(D, x, y, z);
    write_slot(arena, D, TS, j[2], z);
  }
  /* extract (executor.cpp:254-269) */
  if (vg_out) {
    read_slot(arena, D, TS, g->value_slot, x);
    write_block(vg_out, D, n + 1, 0, x);
    for (int i = 0; i < n; ++i) {
      if (g->grad_slots[i] < 0) {
        memset(x, 0, L * 8);
      } else {
        read_slot(arena, D, TS, g->grad_slots[i], x);
        if (g->mult[i] != 1) {
          series_scale_int(D, x, g->mult[i], z);
          memcpy(x, z, L * 8);
        }
      }
      write_block(vg_out, D, n + 1, 1 + i, x);
    }
  }
  if (dyn_out) memcpy(dyn_out, arena, (size_t)D.P * m * (size_t)TS * (size_t)(d + 1) * sizeof(double));
  free(arena);
  free(x);
  free(y);
  free(z);
  pso_graph_free(g);
  return 0;
}

/* eval_direct (oracle_direct.cpp:41-78) */
int pso_eval_direct(int n, int d, int m, int cplx, int N, const int* nvars, const int* idx, const int* exps,
                    const double* stat, double* vg_out) {
  if (!valid_m(m)) return set_err("unsupported precision level");
  sdim D = {d, m, cplx ? 2 : 1};
  const long top = 1L + N + n;
  long long worst = 1;
  long pos = 0;
  for (int k = 0; k < N; ++k) {
    long long q = 0;
    int any = 0;
    if (exps)
      for (int j = 0; j < nvars[k]; ++j) any |= exps[pos + j] != 0;
    for (int j = 0; j < nvars[k]; ++j) q += any ? exps[pos + j] : 1;
    if (q > worst) worst = q;
    pos += nvars[k];
  }
  if ((long long)N * worst * (d + 1) * (d + 1) > 10000000LL) {
    set_err("instance exceeds the direct-evaluation size guard");
    return -2;
  }
  size_t L = slen(D);
  double* value = malloc(L * 8);
  double* grad = calloc((size_t)n * L, 8);
  int* touched = calloc((size_t)n, sizeof(int));
  double* v = malloc(L * 8);
  double* t = malloc(L * 8);
  double* zz = malloc(L * 8);
  double* tmp = malloc(L * 8);
  read_block(stat, D, top, 0, value);
  pos = 0;
  for (int k = 0; k < N; ++k) {
    const int nk = nvars[k];
    const int* ix = idx + pos;
    int any = 0;
    if (exps)
      for (int j = 0; j < nk; ++j) any |= exps[pos + j] != 0;
#define EXP(j) (any ? exps[pos + (j)] : 1)
    read_block(stat, D, top, 1 + k, v);
    for (int j = 0; j < nk; ++j) {
      read_block(stat, D, top, N + ix[j], zz);
      for (int q = 0; q < EXP(j); ++q) {
        conv(D, v, zz, tmp);
        memcpy(v, tmp, L * 8);
      }
    }
    series_add(D, value, v, tmp);
    memcpy(value, tmp, L * 8);
    for (int j = 0; j < nk; ++j) {
      read_block(stat, D, top, 1 + k, t);
      for (int l = 0; l < nk; ++l) {
        const int reps = EXP(l) - (l == j ? 1 : 0);
        read_block(stat, D, top, N + ix[l], zz);
        for (int q = 0; q < reps; ++q) {
          conv(D, t, zz, tmp);
          memcpy(t, tmp, L * 8);
        }
      }
      if (EXP(j) != 1) {
        series_scale_int(D, t, EXP(j), tmp);
        memcpy(t, tmp, L * 8);
      }
      const int var = ix[j] - 1;
      if (touched[var]) {
        series_add(D, grad + (size_t)var * L, t, tmp);
        memcpy(grad + (size_t)var * L, tmp, L * 8);
      } else {
        memcpy(grad + (size_t)var * L, t, L * 8);
      }
      touched[var] = 1;
    }
#undef EXP
    pos += nk;
  }
  write_block(vg_out, D, n + 1, 0, value);
  for (int i = 0; i < n; ++i) write_block(vg_out, D, n + 1, 1 + i, grad + (size_t)i * L);
  free(value);
  free(grad);
  free(touched);
  free(v);
  free(t);
  free(zz);
  free(tmp);
  return 0;
}
