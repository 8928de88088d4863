/* Data-dependent behaviour of the md operations on convolution chains (CPU,
 * analysis only): tighten passes, vec_sum_err_branch trip counts, nonzero
 * pass-2 terms, magnitude order of the exp_add merge inputs. Follows
 * expansion.hpp:31-211 (same algorithms as oracle/pse_oracle.c).
 * Build: gcc -O2 -ffp-contract=off -o /tmp/md_stats tools/md_stats.c -lm
 * Run:   /tmp/md_stats M D  (one conv of degree D on random_md-like inputs) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXM 10
#define MAXNT (MAXM * (MAXM + 1) + MAXM)
static uint64_t st = 0x12345678abcdefULL;
static double rnd(void) { /* [-1, 1) */
  st ^= st << 13; st ^= st >> 7; st ^= st << 17;
  return (double)(st >> 11) * 0x1p-52 - 1.0;
}
static void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b, bv = ss - a, av = ss - bv;
  *e = (a - av) + (b - bv); *s = ss;
}
static void fast_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b; *e = b - (ss - a); *s = ss;
}
static long n_ts, n_ts_fastok;  /* two_sums in vec_sum, and how many had exp(a) >= exp(b) or b == 0 */
static void vec_sum(double* x, int n) {
  double s = x[n - 1];
  for (int i = n - 2; i >= 0; --i) {
    double e;
    n_ts++;
    if (fabs(x[i]) >= fabs(s)) n_ts_fastok++;
    two_sum(x[i], s, &s, &e);
    x[i + 1] = e;
  }
  x[0] = s;
}
static int last_steps;  /* loop trips of the last err_branch */
static int last_nzpops; /* nonzero terms consumed by the last err_branch */
static void err_branch(const double* e, int n, double* out, int m) {
  int j = 0; double eps = e[0]; last_steps = 0; last_nzpops = 0;
  for (int i = 1; i < n; ++i) {
    double r, t; last_steps++; last_nzpops += e[i] != 0.0;
    fast_two_sum(eps, e[i], &r, &t);
    if (t != 0.0) { out[j++] = r; if (j == m) return; eps = t; } else eps = r;
  }
  out[j++] = eps;
  while (j < m) out[j++] = 0.0;
}
static int tighten(double* w, int m) {  /* returns passes that changed something */
  int changed_passes = 0;
  for (int pass = 0; pass < m; ++pass) {
    int changed = 0;
    for (int i = 0; i + 1 < m; ++i) {
      double s, e; two_sum(w[i], w[i + 1], &s, &e);
      if (memcmp(&s, &w[i], 8) || memcmp(&e, &w[i + 1], 8)) { w[i] = s; w[i + 1] = e; changed = 1; }
    }
    if (!changed) break;
    changed_passes++;
  }
  return changed_passes;
}
static long hist_tm[12], hist_ta[12], hist_stm[130], hist_sta[40], hist_nz[130];
static long nz_total, nz_popped, nz_left_hist[64];
static long unsorted_x, unsorted_y, nadds;
static int sorted(const double* v, int m) {
  for (int i = 0; i + 1 < m; ++i) if (fabs(v[i]) < fabs(v[i + 1])) return 0;
  return 1;
}
static void exp_add(int m, const double* x, const double* y, double* out) {
  double t[2 * MAXM]; int i = 0, j = 0, p = 0;
  nadds++;
  if (!sorted(x, m)) unsorted_x++;
  if (!sorted(y, m)) unsorted_y++;
  while (i < m && j < m) t[p++] = fabs(x[i]) >= fabs(y[j]) ? x[i++] : y[j++];
  while (i < m) t[p++] = x[i++];
  while (j < m) t[p++] = y[j++];
  vec_sum(t, 2 * m);
  err_branch(t, 2 * m, out, m);
  hist_sta[last_steps]++;
  hist_ta[tighten(out, m)]++;
}
static void exp_mul(int m, const double* x, const double* y, double* out) {
  double t[MAXNT], carry[MAXM], next[MAXM]; int pos = 0, nc = 0;
  for (int k = 0; k <= m; ++k) {
    int nn = 0, ilo = k - (m - 1) > 0 ? k - (m - 1) : 0, ihi = k < m - 1 ? k : m - 1;
    for (int i = ilo; i <= ihi; ++i) {
      if (k < m) { double p = x[i] * y[k - i]; t[pos++] = p; next[nn++] = fma(x[i], y[k - i], -p); }
      else t[pos++] = x[i] * y[k - i];
    }
    for (int c = 0; c < nc; ++c) t[pos++] = carry[c];
    for (int c = 0; c < nn; ++c) carry[c] = next[c];
    nc = nn;
  }
  vec_sum(t, pos);
  vec_sum(t, pos);
  int nz = 0; for (int i = 1; i < pos; ++i) nz += t[i] != 0.0;
  hist_nz[nz]++;
  err_branch(t, pos, out, m);
  nz_total += nz; nz_popped += last_nzpops; nz_left_hist[nz - last_nzpops]++;
  hist_stm[last_steps]++;
  hist_tm[tighten(out, m)]++;
}
static void renorm(double* v, int m) {  /* random md: limbs at 2^-53k, then vec_sum + err_branch + tighten */
  double t[MAXM]; for (int k = 0; k < m; ++k) t[k] = rnd() * ldexp(1.0, -53 * k);
  vec_sum(t, m); err_branch(t, m, v, m); tighten(v, m);
}
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 10, d = argc > 2 ? atoi(argv[2]) : 152, reps = argc > 3 ? atoi(argv[3]) : 4;
  static double X[1024][MAXM], Y[1024][MAXM];
  for (int r = 0; r < reps; ++r) {
    for (int k = 0; k <= d; ++k) { renorm(X[k], m); renorm(Y[k], m); }
    n_ts = n_ts_fastok = 0;
    for (int k = 0; k <= d; ++k) {
      double acc[MAXM], p[MAXM], o[MAXM];
      exp_mul(m, X[0], Y[k], acc);
      for (int i = 1; i <= k; ++i) { exp_mul(m, X[i], Y[k - i], p); exp_add(m, acc, p, o); memcpy(acc, o, sizeof o); }
    }
  }
  long tot = 0; for (int i = 0; i < 12; ++i) tot += hist_tm[i];
  printf("M=%d d=%d: %ld md_mul, %ld md_add\n", m, d, tot, nadds);
  printf("tighten passes (changed) md_mul:"); for (int i = 0; i < 12; ++i) if (hist_tm[i]) printf(" %d:%.4f", i, hist_tm[i] / (double)tot); printf("\n");
  printf("tighten passes (changed) md_add:"); for (int i = 0; i < 12; ++i) if (hist_ta[i]) printf(" %d:%.4f", i, hist_ta[i] / (double)nadds); printf("\n");
  printf("err_branch trips md_mul:"); for (int i = 0; i < 130; ++i) if (hist_stm[i]) printf(" %d:%.3f", i, hist_stm[i] / (double)tot); printf("\n");
  printf("err_branch trips md_add:"); for (int i = 0; i < 40; ++i) if (hist_sta[i]) printf(" %d:%.3f", i, hist_sta[i] / (double)nadds); printf("\n");
  printf("nonzero pass-2 terms md_mul:"); for (int i = 0; i < 130; ++i) if (hist_nz[i]) printf(" %d:%.4f", i, hist_nz[i] / (double)tot); printf("\n");
  printf("md_mul nonzero terms popped before the M-th emission: %.3f of %.3f; left over:", nz_popped / (double)tot, nz_total / (double)tot);
  for (int i = 0; i < 64; ++i) if (nz_left_hist[i]) printf(" %d:%.3f", i, nz_left_hist[i] / (double)tot); printf("\n");
  printf("merge inputs unsorted: acc %.5f, product %.5f\n", unsorted_x / (double)nadds, unsorted_y / (double)nadds);
  printf("vec_sum steps with |t| >= |s| (last rep): %.4f\n", n_ts_fastok / (double)n_ts);
  return 0;
}
