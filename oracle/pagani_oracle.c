/*
 * TEST INFRASTRUCTURE ONLY (oracle) -- never linked into or called by the
 * product; loaded only by tests/ (and optionally bench.py's CPU baseline).
 *
 * Plain-C restatement of the reference PAGANI hot path, serial, for checking:
 *   rule construction    /root/reference/proj/src/rule.cpp:14-349
 *   evaluate_batch       rule.cpp:351-430
 *   integrands f1..f8    integrands.cpp:14-79 (platform libm exp/cos/sqrt)
 *   two_level_refine     errorest.cpp:10-37
 *   rel_err_classify / apply_threshold / threshold_classify / filter
 *                        classify.cpp:11-129
 *   block sums, counts   reduce.cpp:10-82
 *   uniform_split / bisect / initial_subdivisions  geometry.cpp:54-143
 *   integrate loop       driver.cpp:28-215
 * Compiled with -ffp-contract=off and no -march, like the reference.
 * Parity: pinned bit-for-bit against oracle/_ref by tests/test_oracle.py.
 */
#include "pagani_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXDIM 16
#define BLOCK 2048

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rule ---- */
typedef long double ld;
enum { CENTER, NEAR, FAR, PAIRS, CORNERS, NORB };

typedef struct {
  int k;
  int e[3];
} Mono;

typedef struct {
  ld mag[NORB];
  int64_t size[NORB];
} Geom;

typedef struct {
  int n;
  int64_t N;
  double w[5][NORB]; /* [weight set][orbit] */
  double gen[4];     /* l2 l3 l4 l5 */
} Rule;

static Geom geometry(int n) { /* rule.cpp:119-125, 14-17 */
  Geom g;
  g.mag[CENTER] = 0.0L;
  g.mag[NEAR] = sqrtl(9.0L / 70.0L);
  g.mag[FAR] = sqrtl(9.0L / 10.0L);
  g.mag[PAIRS] = sqrtl(9.0L / 10.0L);
  g.mag[CORNERS] = sqrtl(9.0L / 19.0L);
  g.size[CENTER] = 1;
  g.size[NEAR] = 2 * n;
  g.size[FAR] = 2 * n;
  g.size[PAIRS] = (int64_t)2 * n * (n - 1);
  g.size[CORNERS] = (int64_t)1 << n;
  return g;
}

static ld orbit_sum(int o, ld mag, int n, const Mono* p) { /* rule.cpp:38-57 */
  switch (o) {
    case CENTER:
      return p->k == 0 ? 1.0L : 0.0L;
    case NEAR:
    case FAR:
      if (p->k == 0) return 2.0L * n;
      if (p->k == 1) return 2.0L * powl(mag, (ld)p->e[0]);
      return 0.0L;
    case PAIRS:
      if (p->k == 0) return 2.0L * n * (n - 1);
      if (p->k == 1) return 4.0L * (n - 1) * powl(mag, (ld)p->e[0]);
      if (p->k == 2) return 4.0L * powl(mag, (ld)(p->e[0] + p->e[1]));
      return 0.0L;
    default:
      return powl(2.0L, (ld)n) * powl(mag, (ld)(p->e[0] + p->e[1] + p->e[2]));
  }
}

static ld moment_target(const Mono* p) { /* rule.cpp:60-64 */
  ld t = 1.0L;
  for (int i = 0; i < p->k; ++i) t /= (ld)(p->e[i] + 1);
  return t;
}

static int patterns_upto(int n, int max_deg, Mono* ps) { /* rule.cpp:177-191 */
  int c = 0;
  ps[c++] = (Mono){0, {0, 0, 0}};
  if (max_deg >= 2) ps[c++] = (Mono){1, {2, 0, 0}};
  if (max_deg >= 4) {
    ps[c++] = (Mono){1, {4, 0, 0}};
    if (n >= 2) ps[c++] = (Mono){2, {2, 2, 0}};
  }
  if (max_deg >= 6) {
    ps[c++] = (Mono){1, {6, 0, 0}};
    if (n >= 2) ps[c++] = (Mono){2, {4, 2, 0}};
    if (n >= 3) ps[c++] = (Mono){3, {2, 2, 2}};
  }
  return c;
}

/* rule.cpp:68-111 -- normal equations, partial pivoting, residual check */
static int solve_moments(ld rows[][NORB], const ld* rhs, int nrows, const int* cols, int k,
                         ld x[NORB]) {
  ld ata[NORB][NORB] = {{0}};
  ld atb[NORB] = {0};
  for (int r = 0; r < nrows; ++r)
    for (int i = 0; i < k; ++i) {
      atb[i] += rows[r][cols[i]] * rhs[r];
      for (int j = 0; j < k; ++j) ata[i][j] += rows[r][cols[i]] * rows[r][cols[j]];
    }
  for (int c = 0; c < k; ++c) {
    int piv = c;
    for (int r = c + 1; r < k; ++r)
      if (fabsl(ata[r][c]) > fabsl(ata[piv][c])) piv = r;
    if (piv != c) {
      for (int j = 0; j < k; ++j) {
        ld t = ata[c][j];
        ata[c][j] = ata[piv][j];
        ata[piv][j] = t;
      }
      ld t = atb[c];
      atb[c] = atb[piv];
      atb[piv] = t;
    }
    if (ata[c][c] == 0.0L) return fail(-3, "rule moments: singular system");
    for (int r = c + 1; r < k; ++r) {
      const ld m = ata[r][c] / ata[c][c];
      for (int j = c; j < k; ++j) ata[r][j] -= m * ata[c][j];
      atb[r] -= m * atb[c];
    }
  }
  for (int o = 0; o < NORB; ++o) x[o] = 0.0L;
  for (int c = k - 1; c >= 0; --c) {
    ld s = atb[c];
    for (int j = c + 1; j < k; ++j) s -= ata[c][j] * x[cols[j]];
    x[cols[c]] = s / ata[c][c];
  }
  for (int r = 0; r < nrows; ++r) {
    ld resid = -rhs[r];
    for (int i = 0; i < k; ++i) resid += rows[r][cols[i]] * x[cols[i]];
    if (fabsl(resid) > 1e-12L) return fail(-3, "rule moments: inconsistent system");
  }
  return 0;
}

static ld wdot(const ld* u, const ld* v, const Geom* g) { /* rule.cpp:127-132 */
  ld s = 0.0L;
  for (int o = 0; o < NORB; ++o) s += (ld)g->size[o] * u[o] * v[o];
  return s;
}

typedef struct {
  const Geom* g;
  int count;
  ld b[12][NORB];
} Ortho; /* rule.cpp:135-158 */

static int ortho_residual(const Ortho* O, const ld* vin, ld* out) {
  ld v[NORB];
  memcpy(v, vin, sizeof v);
  for (int q = 0; q < O->count; ++q) {
    const ld c = wdot(v, O->b[q], O->g);
    for (int o = 0; o < NORB; ++o) v[o] -= c * O->b[q][o];
  }
  const ld norm2 = wdot(v, v, O->g);
  if (norm2 < 1e-18L) return 0;
  const ld inv = 1.0L / sqrtl(norm2);
  for (int o = 0; o < NORB; ++o) out[o] = v[o] * inv;
  return 1;
}

static int ortho_add(Ortho* O, const ld* v) {
  ld r[NORB];
  if (!ortho_residual(O, v, r)) return 0;
  memcpy(O->b[O->count++], r, sizeof r);
  return 1;
}

static void wspace_row(const Geom* g, int n, const Mono* p, ld* v) { /* rule.cpp:216-222 */
  for (int o = 0; o < NORB; ++o)
    v[o] = g->size[o] ? orbit_sum(o, g->mag[o], n, p) / (ld)g->size[o] : 0.0L;
}

/* rule.cpp:224-242 */
static int null_rules_below(const Geom* g, int n, const Mono* anni, int nanni, ld priors[][NORB],
                            int npriors, int want, ld found[][NORB]) {
  Ortho O;
  O.g = g;
  O.count = 0;
  for (int i = 0; i < nanni; ++i) {
    ld v[NORB];
    wspace_row(g, n, &anni[i], v);
    ortho_add(&O, v);
  }
  for (int i = 0; i < npriors; ++i) ortho_add(&O, priors[i]);
  int nf = 0;
  for (int o = 0; o < NORB && nf < want; ++o) {
    if (!g->size[o]) continue;
    ld seed[NORB] = {0};
    seed[o] = 1.0L;
    ld r[NORB];
    if (ortho_residual(&O, seed, r)) {
      memcpy(found[nf++], r, sizeof r);
      ortho_add(&O, r);
    }
  }
  return nf;
}

static int build_rule(int n, Rule* R) { /* rule.cpp:166-349 */
  if (n < 1 || n > MAXDIM) return fail(-1, "build_rule: dimension out of range");
  const Geom g = geometry(n);
  int cols7[NORB], cols5[NORB], k7 = 0, k5 = 0;
  for (int o = 0; o < NORB; ++o)
    if (g.size[o] > 0) cols7[k7++] = o;
  for (int o = 0; o < NORB - 1; ++o)
    if (g.size[o] > 0) cols5[k5++] = o;
  Mono p7[8], p5[8];
  const int n7 = patterns_upto(n, 6, p7), n5 = patterns_upto(n, 4, p5);
  ld rows7[8][NORB], rhs7[8], rows5[8][NORB], rhs5[8];
  for (int r = 0; r < n7; ++r) {
    for (int o = 0; o < NORB; ++o) rows7[r][o] = g.size[o] ? orbit_sum(o, g.mag[o], n, &p7[r]) : 0.0L;
    rhs7[r] = moment_target(&p7[r]);
  }
  for (int r = 0; r < n5; ++r) {
    for (int o = 0; o < NORB; ++o) rows5[r][o] = g.size[o] ? orbit_sum(o, g.mag[o], n, &p5[r]) : 0.0L;
    rhs5[r] = moment_target(&p5[r]);
  }
  ld w7[NORB], w5[NORB];
  int rc = solve_moments(rows7, rhs7, n7, cols7, k7, w7);
  if (rc) return rc;
  rc = solve_moments(rows5, rhs5, n5, cols5, k5, w5);
  if (rc) return rc;
  ld u1[NORB];
  for (int o = 0; o < NORB; ++o) u1[o] = w7[o] - w5[o];
  const ld u1_norm = sqrtl(wdot(u1, u1, &g));

  const Mono deg1[1] = {{0, {0, 0, 0}}};
  const Mono deg3[2] = {{0, {0, 0, 0}}, {1, {2, 0, 0}}};
  ld pri[4][NORB], d3[2][NORB], d1[1][NORB];
  memcpy(pri[0], u1, sizeof u1);
  const int nd3 = null_rules_below(&g, n, deg3, 2, pri, 1, 2, d3);
  for (int i = 0; i < nd3; ++i) memcpy(pri[1 + i], d3[i], sizeof u1);
  const int nd1 = null_rules_below(&g, n, deg1, 1, pri, 1 + nd3, 1, d1);
  if (nd1 == 0) return fail(-3, "build_rule: degree-1 null rule not found");

  ld nulls[4][NORB];
  int nn = 0;
  memcpy(nulls[nn++], u1, sizeof u1);
  for (int i = 0; i < nd3; ++i) {
    for (int o = 0; o < NORB; ++o) d3[i][o] *= u1_norm * (ld)1e-2; /* kNullScaleDeg3 (double) */
    memcpy(nulls[nn++], d3[i], sizeof u1);
  }
  for (int o = 0; o < NORB; ++o) d1[0][o] *= u1_norm * (ld)1e-4; /* kNullScaleDeg1 (double) */
  memcpy(nulls[nn++], d1[0], sizeof u1);
  while (nn < 4) {
    memcpy(nulls[nn], nulls[nn - 1], sizeof u1);
    ++nn;
  }
  /* annihilation check, rule.cpp:267-279 */
  for (int k = 0; k < 4; ++k) {
    const Mono* an = k == 0 ? p5 : (k <= nd3 ? deg3 : deg1);
    const int na = k == 0 ? n5 : (k <= nd3 ? 2 : 1);
    for (int i = 0; i < na; ++i) {
      ld s = 0.0L;
      for (int o = 0; o < NORB; ++o)
        if (g.size[o]) s += nulls[k][o] * orbit_sum(o, g.mag[o], n, &an[i]);
      if (fabsl(s) > 1e-13L) return fail(-3, "build_rule: null rule fails annihilation");
    }
  }
  R->n = n;
  R->N = ((int64_t)1 << n) + (int64_t)2 * n * (n - 1) + 4 * n + 1;
  for (int o = 0; o < NORB; ++o) {
    R->w[0][o] = (double)w7[o];
    for (int k = 1; k < 5; ++k) R->w[k][o] = (double)nulls[k - 1][o];
  }
  R->gen[0] = (double)g.mag[NEAR];
  R->gen[1] = (double)g.mag[FAR];
  R->gen[2] = (double)g.mag[PAIRS];
  R->gen[3] = (double)g.mag[CORNERS];
  return 0;
}

/* point p of the rule in generator coordinates + its orbit (rule.cpp:297-337) */
static int rule_point(const Rule* R, int64_t p, double* g) {
  const int n = R->n;
  for (int a = 0; a < n; ++a) g[a] = 0.0;
  if (p == 0) return CENTER;
  p -= 1;
  if (p < 4 * n) {
    const int orbit = p < 2 * n ? NEAR : FAR;
    const int64_t q = p % (2 * n);
    const double l = R->gen[orbit - 1];
    g[q / 2] = (q & 1) ? l : -l;
    return orbit;
  }
  p -= 4 * n;
  if (p < (int64_t)2 * n * (n - 1)) {
    int64_t idx = p / 4;
    const int sa = (int)((p / 2) & 1), sb = (int)(p & 1);
    for (int a = 0; a < n; ++a)
      for (int b = a + 1; b < n; ++b) {
        if (idx-- == 0) {
          g[a] = sa ? R->gen[2] : -R->gen[2];
          g[b] = sb ? R->gen[2] : -R->gen[2];
          return PAIRS;
        }
      }
  }
  p -= (int64_t)2 * n * (n - 1);
  for (int a = 0; a < n; ++a) g[a] = ((p >> a) & 1) ? R->gen[3] : -R->gen[3];
  return CORNERS;
}

/* ---------------------------------------------------------- integrands ---- */
typedef double (*ifn)(const double*, int, const double*);

static double ipow(double base, int e) { /* integrands.cpp:14-22 */
  double r = 1.0;
  while (e > 0) {
    if (e & 1) r *= base;
    base *= base;
    e >>= 1;
  }
  return r;
}
static double f1(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += (i + 1) * x[i];
  return cos(s);
}
static double f2(const double* x, int n, const double* p) {
  (void)p;
  double r = 1.0;
  for (int i = 0; i < n; ++i) {
    const double t = x[i] - 0.5;
    r *= 1.0 / (1.0 / 2500.0 + t * t);
  }
  return r;
}
static double f3(const double* x, int n, const double* p) {
  (void)p;
  double s = 1.0;
  for (int i = 0; i < n; ++i) s += (i + 1) * x[i];
  return 1.0 / ipow(s, n + 1);
}
static double f4(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double t = x[i] - 0.5;
    s += t * t;
  }
  return exp(-625.0 * s);
}
static double f5(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += fabs(x[i] - 0.5);
  return exp(-10.0 * s);
}
static double f6(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 1; i <= n; ++i) {
    if (x[i - 1] >= (3.0 + i) / 10.0) return 0.0;
    s += (i + 4) * x[i - 1];
  }
  return exp(s);
}
static double f7(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += x[i] * x[i];
  return ipow(s, 11);
}
static double f8(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += x[i] * x[i];
  return ipow(s, 7) * sqrt(s);
}
/* parameterised reference unit-test integrands (see oracle/ref_shim.cpp) */
static double t_const(const double* x, int n, const double* p) {
  (void)x, (void)n;
  return p[0];
}
static double t_monomial(const double* x, int n, const double* p) {
  double v = 1.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < (int)p[i]; ++k) v *= x[i];
  return v;
}
static double t_rough(const double* x, int n, const double* p) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += cos(p[1] == 2.0 ? p[0] * x[i] * x[i] : p[0] * x[i]);
  return s + p[2] * n;
}
static double t_nanbox(const double* x, int n, const double* p) {
  (void)n;
  return (x[0] > p[0] && (p[1] < 0.0 || x[1] > p[1])) ? NAN : 1.0;
}
static double t_pocket(const double* x, int n, const double* p) {
  (void)n;
  return x[0] > p[0] && x[1] > p[0] && x[2] > p[0] ? 1.0 : 0.0;
}
static double t_cossum(const double* x, int n, const double* p) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += cos(p[1 + i] * 3.0 * x[i]);
  return p[0] * s;
}
static double t_expsq(const double* x, int n, const double* p) {
  (void)p;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += exp(x[i] / 3.0) + x[i] * x[i];
  return s;
}

static ifn lookup(int fid) {
  switch (fid) {
    case 1: return f1;
    case 2: return f2;
    case 3: return f3;
    case 4: return f4;
    case 5: return f5;
    case 6: return f6;
    case 7: return f7;
    case 8: return f8;
    case 100: return t_const;
    case 101: return t_monomial;
    case 102: return t_rough;
    case 103: return t_nanbox;
    case 104: return t_pocket;
    case 105: return t_cossum;
    case 106: return t_expsq;
    default: return NULL;
  }
}

typedef struct {
  ifn f;
  double p[32];
  int mapped;
  double lo[MAXDIM], len[MAXDIM];
} Fn;

static double call(const Fn* F, const double* u, int n) {
  if (!F->mapped) return F->f(u, n, F->p);
  double x[MAXDIM];
  for (int a = 0; a < n; ++a) x[a] = F->lo[a] + u[a] * F->len[a]; /* driver.cpp:68-73 */
  return F->f(x, n, F->p);
}

/* ------------------------------------------------------------- batch ---- */
typedef struct {
  int n;
  int64_t m;
  double *lows, *lens, *est, *err, *pest, *perr;
  int* axis;
} Batch;

static void batch_alloc(Batch* b, int n, int64_t m) {
  b->n = n;
  b->m = m;
  const size_t mm = m > 0 ? (size_t)m : 1;
  b->lows = calloc(mm * n, 8);
  b->lens = calloc(mm * n, 8);
  b->est = calloc(mm, 8);
  b->err = calloc(mm, 8);
  b->pest = calloc(mm, 8);
  b->perr = calloc(mm, 8);
  b->axis = calloc(mm, sizeof(int));
}
static void batch_free(Batch* b) {
  free(b->lows), free(b->lens), free(b->est), free(b->err), free(b->pest), free(b->perr),
      free(b->axis);
}

/* rule.cpp:351-430 */
static void evaluate(const Fn* F, const Batch* B, const Rule* R, double* est, double* raw,
                     int* axes) {
  const int n = B->n;
  const int nprobe = 4 * n;
  double* gen = malloc((size_t)R->N * n * 8);
  int* orb = malloc((size_t)R->N * sizeof(int));
  for (int64_t p = 0; p < R->N; ++p) orb[p] = rule_point(R, p, gen + p * n);
  for (int64_t j = 0; j < B->m; ++j) {
    const double* low = B->lows + j * n;
    const double* len = B->lens + j * n;
    double c[MAXDIM], h[MAXDIM], x[MAXDIM], vals[1 + 4 * MAXDIM];
    double vol = 1.0;
    for (int a = 0; a < n; ++a) {
      h[a] = 0.5 * len[a];
      c[a] = low[a] + h[a];
      vol *= len[a];
    }
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    int finite = 1;
    for (int64_t p = 0; p < R->N; ++p) {
      const double* g = gen + p * n;
      for (int a = 0; a < n; ++a) x[a] = c[a] + g[a] * h[a];
      const double fx = call(F, x, n);
      finite = finite && isfinite(fx);
      if (p <= nprobe) vals[p] = fx;
      const int o = orb[p];
      s0 += R->w[0][o] * fx;
      s1 += R->w[1][o] * fx;
      s2 += R->w[2][o] * fx;
      s3 += R->w[3][o] * fx;
      s4 += R->w[4][o] * fx;
    }
    const double f0 = vals[0];
    int best_axis = 0;
    double best = -1.0;
    for (int a = 0; a < n; ++a) {
      const double near2 = vals[1 + 2 * a] + vals[2 + 2 * a] - 2.0 * f0;
      const double far2 = vals[1 + 2 * n + 2 * a] + vals[2 + 2 * n + 2 * a] - 2.0 * f0;
      const double diff = fabs(near2 - ((9.0 / 70.0) / (9.0 / 10.0)) * far2);
      if (isfinite(diff) && diff > best) {
        best = diff;
        best_axis = a;
      }
    }
    if (best <= 0.0)
      for (int a = 1; a < n; ++a)
        if (len[a] > len[best_axis]) best_axis = a;
    axes[j] = best_axis;
    if (!finite) {
      est[j] = 0.0;
      raw[j] = INFINITY;
      continue;
    }
    const double m12 = fabs(s1) < fabs(s2) ? fabs(s2) : fabs(s1);
    const double m34 = fabs(s3) < fabs(s4) ? fabs(s4) : fabs(s3);
    est[j] = vol * s0;
    raw[j] = vol * (m12 < m34 ? m34 : m12);
  }
  free(gen);
  free(orb);
}

/* errorest.cpp:24-36 */
static void refine(int64_t m, const double* est, const double* raw, const double* pest,
                   double* out) {
  for (int64_t j = 0; j < m; ++j) {
    const int64_t s = j ^ 1;
    const double pair = raw[j] + raw[s];
    if (pair == 0.0 || !isfinite(pair)) {
      out[j] = raw[j];
      continue;
    }
    const double delta = fabs(pest[j] - (est[j] + est[s]));
    double r = delta / pair;
    r = r < 0.125 ? 0.125 : (1.0 < r ? 1.0 : r); /* std::clamp */
    out[j] = raw[j] * r;
  }
}

/* reduce.cpp:10-64 */
static double pairwise(double* p, int64_t m) {
  if (m == 0) return 0.0;
  while (m > 1) {
    const int64_t half = m / 2;
    for (int64_t i = 0; i < half; ++i) p[i] = p[2 * i] + p[2 * i + 1];
    if (m % 2) {
      p[half] = p[m - 1];
      m = half + 1;
    } else {
      m = half;
    }
  }
  return p[0];
}
static double bsum_where(int64_t n, const double* x, const uint8_t* f, int which) {
  if (n == 0) return 0.0;
  const int64_t nb = (n + BLOCK - 1) / BLOCK;
  double* part = malloc((size_t)nb * 8);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = b * BLOCK, hi = lo + BLOCK < n ? lo + BLOCK : n;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i)
      if (!f || f[i] == which) s += x[i];
    part[b] = s;
  }
  const double r = pairwise(part, nb);
  free(part);
  return r;
}
static int64_t count_flags(int64_t n, const uint8_t* f, int which) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c += f[i] == which;
  return c;
}

/* classify.cpp:37-95 */
static void threshold(const uint8_t* active, const double* errors, double v_tot, double e_tot,
                      double e_it, int64_t s, double tau, const orc_config* L, uint8_t* flags_out,
                      orc_threshold_out* r) {
  memset(r, 0, sizeof *r);
  memcpy(flags_out, active, (size_t)s);
  if (s <= 0) return;
  const double e_budget = e_tot - fabs(v_tot) * tau;
  double p_max = L->p_max_start;
  r->budget_limit = p_max * e_budget;
  if (!(e_budget > 0.0)) return;
  double lo = errors[0], hi = lo;
  for (int64_t i = 0; i < s; ++i) {
    if (errors[i] < lo) lo = errors[i];
    if (errors[i] > hi) hi = errors[i];
  }
  double t = e_it / (double)s;
  uint8_t* cand = malloc((size_t)s);
  int last = 0; /* 0 none, 1 toward max, 2 toward min */
  while (r->attempts < L->attempt_limit) {
    ++r->attempts;
    for (int64_t j = 0; j < s; ++j) cand[j] = active[j] & (errors[j] < t ? 0 : 1);
    const int64_t inactive = s - count_flags(s, cand, 1);
    const int memory_ok = 2 * inactive > s;
    const double discarded = bsum_where(s, errors, cand, 0);
    if (memory_ok && discarded <= p_max * e_budget) {
      r->success = 1;
      memcpy(flags_out, cand, (size_t)s);
      r->threshold = t;
      r->discarded_error = discarded;
      r->budget_limit = p_max * e_budget;
      r->finished_count = inactive;
      free(cand);
      return;
    }
    const int dir = memory_ok ? 2 : 1;
    if (last != 0 && dir != last) {
      ++r->direction_changes;
      if (r->direction_changes > L->direction_change_limit) break;
      const double stepped = p_max + L->p_max_step;
      p_max = stepped < L->p_max_cap ? stepped : L->p_max_cap;
    }
    last = dir;
    t = dir == 1 ? (t + hi) * 0.5 : (t + lo) * 0.5;
  }
  r->threshold = t;
  r->budget_limit = p_max * e_budget;
  free(cand);
}

/* classify.cpp:97-129 (finished sums) + geometry.cpp:114-143 (bisect) */
static int64_t filter_bisect(const Batch* B, const uint8_t* flags, double* fin_e, double* fin_r,
                             Batch* out) {
  *fin_e = bsum_where(B->m, B->est, flags, 0);
  *fin_r = bsum_where(B->m, B->err, flags, 0);
  const int64_t kept = count_flags(B->m, flags, 1);
  if (!out) return kept;
  const int n = B->n;
  batch_alloc(out, n, 2 * kept);
  int64_t k = 0;
  for (int64_t j = 0; j < B->m; ++j) {
    if (!flags[j]) continue;
    const int ax = B->axis[j];
    const double* low = B->lows + j * n;
    const double* len = B->lens + j * n;
    const double half = len[ax] * 0.5;
    for (int child = 0; child < 2; ++child) {
      const int64_t c = 2 * k + child;
      for (int a = 0; a < n; ++a) {
        out->lows[c * n + a] = low[a];
        out->lens[c * n + a] = len[a];
      }
      out->lens[c * n + ax] = half;
      if (child == 1) out->lows[c * n + ax] = low[ax] + half;
      out->pest[c] = B->est[j];
      out->perr[c] = B->err[j];
    }
    ++k;
  }
  return kept;
}

static int initial_subdivisions(int n, int64_t target) { /* geometry.cpp:67-81 */
  int d = 1;
  for (;;) {
    int64_t p = 1;
    int over = 0;
    for (int a = 0; a < n; ++a) {
      if (p > target / (d + 1)) {
        over = 1;
        break;
      }
      p *= d + 1;
    }
    if (over || p > target) break;
    ++d;
  }
  return d;
}

static int uniform_split(int n, const double* lo, const double* hi, int d, int64_t maxr,
                         Batch* out) { /* geometry.cpp:83-112 */
  if (d < 1) return fail(-1, "uniform_split: d must be >= 1");
  int64_t m = 1;
  for (int a = 0; a < n; ++a) {
    if (m > maxr / d) return fail(-2, "uniform_split: d^n exceeds max_regions");
    m *= d;
  }
  if (m > maxr) return fail(-2, "uniform_split: d^n exceeds max_regions");
  batch_alloc(out, n, m);
  double step[MAXDIM];
  for (int a = 0; a < n; ++a) step[a] = (hi[a] - lo[a]) / d;
  for (int64_t j = 0; j < m; ++j) {
    int64_t rem = j;
    for (int a = 0; a < n; ++a) {
      const int64_t cell = rem % d;
      rem /= d;
      out->lows[j * n + a] = lo[a] + cell * step[a];
      out->lens[j * n + a] = step[a];
    }
  }
  return 0;
}

static int digits_converged(double a, double b, int digits) { /* driver.cpp:48-58 */
  if (!isfinite(a) || !isfinite(b)) return 0;
  if (a == 0.0 && b == 0.0) return 1;
  if ((a < 0.0) != (b < 0.0)) return 0;
  if (digits < 1) digits = 1;
  if (digits > 17) digits = 17;
  char x[40], y[40];
  snprintf(x, sizeof x, "%.*e", digits - 1, a);
  snprintf(y, sizeof y, "%.*e", digits - 1, b);
  return strcmp(x, y) == 0;
}

static int convergence_digits(double tau) { /* driver.cpp:28-33 */
  const double d = ceil(log10(1.0 / tau));
  if (!(d >= 1.0)) return 1;
  if (d > 17.0) return 17;
  return (int)d;
}

/* ----------------------------------------------------------- integrate ---- */
static int make_fn(int fid, const double* params, int np, Fn* F) {
  memset(F, 0, sizeof *F);
  F->f = lookup(fid);
  if (!F->f) return fail(-1, "unknown integrand id");
  for (int i = 0; i < np && i < 32; ++i) F->p[i] = params[i];
  return 0;
}

/* driver.cpp:83-215 (optionally recording one orc_trace_row per iteration) */
static int run(const Fn* Fin, int n, const double* lower, const double* upper,
               const orc_config* c, orc_result* out, orc_event* events, int max_events,
               orc_trace_row* rows, int max_rows) {
  if (!(c->tau_rel > 0.0)) return fail(-1, "Config: tau_rel must be > 0");
  if (!(c->tau_abs >= 0.0)) return fail(-1, "Config: tau_abs must be >= 0");
  if (c->it_max < 1) return fail(-1, "Config: it_max must be >= 1");
  if (c->init_subdiv == 0 && c->max_regions < 2 * c->init_target)
    return fail(-1, "Config: max_regions must be >= 2 * init_target");
  if (n < 1 || n > MAXDIM) return fail(-1, "Bounds: dimension must be in [1, 16]");
  Fn F = *Fin;
  int mapped = 0;
  double jac = 1.0;
  for (int a = 0; a < n; ++a) {
    if (!(lower[a] < upper[a])) return fail(-1, "Bounds: lower must be < upper on every axis");
    if (!isfinite(lower[a]) || !isfinite(upper[a])) return fail(-1, "Bounds: entries must be finite");
    if (lower[a] != 0.0 || upper[a] != 1.0) mapped = 1;
    jac *= upper[a] - lower[a];
    F.lo[a] = lower[a];
    F.len[a] = upper[a] - lower[a];
  }
  F.mapped = mapped;
  const double tau_abs = mapped ? c->tau_abs / jac : c->tau_abs;
  Rule R;
  int rc = build_rule(n, &R);
  if (rc) return rc;
  const int d = c->init_subdiv > 0 ? c->init_subdiv : initial_subdivisions(n, c->init_target);
  double zero[MAXDIM], one[MAXDIM];
  for (int a = 0; a < n; ++a) zero[a] = 0.0, one[a] = 1.0;
  Batch B;
  rc = uniform_split(n, zero, one, d, c->max_regions, &B);
  if (rc) return rc;
  memset(out, 0, sizeof *out);
  out->regions_generated = B.m;
  double v = 0, e = 0, vf = 0, ef = 0, prev_total = NAN;
  const int digits = convergence_digits(c->tau_rel);
  int nrows = 0, status = 1, iters = c->it_max;
  for (int it = 1; it <= c->it_max; ++it) {
    double* raw = malloc((size_t)(B.m ? B.m : 1) * 8);
    evaluate(&F, &B, &R, B.est, raw, B.axis);
    out->eval_count += B.m * R.N;
    if (it == 1 || c->refiner == 1)
      memcpy(B.err, raw, (size_t)B.m * 8);
    else
      refine(B.m, B.est, raw, B.pest, B.err);
    free(raw);
    uint8_t* flags = malloc((size_t)(B.m ? B.m : 1));
    for (int64_t j = 0; j < B.m; ++j) {
      const int fin = B.est[j] == 0.0 ? B.err[j] == 0.0 : B.err[j] <= fabs(B.est[j]) * c->tau_rel;
      flags[j] = c->rel_filtering_enabled ? (fin ? 0 : 1) : 1;
    }
    v = bsum_where(B.m, B.est, NULL, 0);
    e = bsum_where(B.m, B.err, NULL, 0);
    orc_trace_row row;
    memset(&row, 0, sizeof row);
    row.it = it;
    row.m = B.m;
    row.active_rel = count_flags(B.m, flags, 1);
    const double err_tot = e + ef;
    if (err_tot <= fabs(v + vf) * c->tau_rel || err_tot <= tau_abs) {
      row.v = v, row.e = e, row.v_f = vf, row.e_f = ef, row.active_final = row.active_rel;
      if (rows && nrows < max_rows) rows[nrows] = row;
      ++nrows;
      status = 0, iters = it;
      free(flags);
      break;
    }
    if (it == c->it_max) {
      row.v = v, row.e = e, row.v_f = vf, row.e_f = ef, row.active_final = row.active_rel;
      if (rows && nrows < max_rows) rows[nrows] = row;
      ++nrows;
      free(flags);
      break;
    }
    const int trig_memory = 2 * row.active_rel > c->max_regions;
    const int trig_digits = digits_converged(prev_total, v + vf, digits);
    row.trig_digits = trig_digits;
    row.trig_memory = trig_memory;
    if (trig_digits || trig_memory) {
      uint8_t* tf = malloc((size_t)B.m);
      orc_threshold_out tr;
      threshold(flags, B.err, v + vf, e + ef, e, B.m, c->tau_rel, c, tf, &tr);
      if (events && out->n_events < max_events)
        events[out->n_events] = (orc_event){it, tr.success, B.m, tr.finished_count,
                                            tr.discarded_error, tr.budget_limit};
      out->n_events++;
      const int affordable = ef + tr.discarded_error <= 0.25 * c->tau_rel * fabs(v + vf);
      row.thr_invoked = 1;
      row.thr_success = tr.success;
      row.thr_attempts = tr.attempts;
      row.thr_dir_changes = tr.direction_changes;
      row.thr_threshold = tr.threshold;
      row.thr_discarded = tr.discarded_error;
      row.thr_budget = tr.budget_limit;
      row.thr_finished = tr.finished_count;
      if (tr.success && (trig_memory || affordable)) {
        memcpy(flags, tf, (size_t)B.m);
        row.thr_accepted = 1;
      }
      free(tf);
    }
    row.v = v, row.e = e, row.v_f = vf, row.e_f = ef;
    double fin_v, fin_e;
    const int64_t kept = filter_bisect(&B, flags, &fin_v, &fin_e, NULL);
    row.active_final = kept;
    row.fin_v = fin_v, row.fin_e = fin_e, row.kept = kept;
    if (rows && nrows < max_rows) rows[nrows] = row;
    ++nrows;
    vf += fin_v;
    ef += fin_e;
    v -= fin_v;
    e -= fin_e;
    prev_total = v + vf;
    if (kept == 0) {
      status = 1, iters = it;
      free(flags);
      break;
    }
    if (2 * kept > c->max_regions) {
      status = 2, iters = it;
      free(flags);
      break;
    }
    Batch nb;
    filter_bisect(&B, flags, &fin_v, &fin_e, &nb);
    free(flags);
    batch_free(&B);
    B = nb;
    out->regions_generated += B.m;
  }
  batch_free(&B);
  out->status = status;
  out->iterations = iters;
  out->estimate = (v + vf) * jac;
  out->errorest = (e + ef) * jac;
  return nrows;
}

/* ------------------------------------------------------------ orc_* API ---- */
int orc_integrate(int fid, const double* params, int np, int n, const double* lo,
                  const double* hi, const orc_config* c, orc_result* out, orc_event* ev,
                  int max_ev) {
  Fn F;
  int rc = make_fn(fid, params, np, &F);
  if (rc) return rc;
  rc = run(&F, n, lo, hi, c, out, ev, max_ev, NULL, 0);
  return rc < 0 ? rc : 0;
}

int orc_trace(int fid, const double* params, int np, int n, const orc_config* c,
              orc_result* out, orc_trace_row* rows, int max_rows) {
  Fn F;
  int rc = make_fn(fid, params, np, &F);
  if (rc) return rc;
  double lo[MAXDIM], hi[MAXDIM];
  for (int a = 0; a < n && a < MAXDIM; ++a) lo[a] = 0.0, hi[a] = 1.0;
  return run(&F, n, lo, hi, c, out, NULL, 0, rows, max_rows);
}

int64_t orc_rule_point_count(int n) {
  return ((int64_t)1 << n) + (int64_t)2 * n * (n - 1) + 4 * n + 1;
}

int orc_build_rule(int n, double* points, double* weight_sets, int* probes) {
  Rule R;
  const int rc = build_rule(n, &R);
  if (rc) return rc;
  for (int64_t p = 0; p < R.N; ++p) {
    double g[MAXDIM];
    const int o = rule_point(&R, p, g);
    if (points) memcpy(points + p * n, g, (size_t)n * 8);
    if (weight_sets)
      for (int k = 0; k < 5; ++k) weight_sets[k * R.N + p] = R.w[k][o];
  }
  if (probes)
    for (int a = 0; a < n; ++a) {
      probes[4 * a + 0] = 1 + 2 * a;
      probes[4 * a + 1] = 2 + 2 * a;
      probes[4 * a + 2] = 1 + 2 * n + 2 * a;
      probes[4 * a + 3] = 2 + 2 * n + 2 * a;
    }
  return 0;
}

int orc_evaluate_batch(int fid, const double* params, int np, int n, int64_t m,
                       const double* lows, const double* lengths, double* est, double* raw,
                       int* axes, int64_t* eval_count) {
  Fn F;
  int rc = make_fn(fid, params, np, &F);
  if (rc) return rc;
  Rule R;
  rc = build_rule(n, &R);
  if (rc) return rc;
  Batch B;
  B.n = n;
  B.m = m;
  B.lows = (double*)lows;
  B.lens = (double*)lengths;
  evaluate(&F, &B, &R, est, raw, axes);
  if (eval_count) *eval_count = m * R.N;
  return 0;
}

int orc_two_level_refine(int64_t m, const double* est, const double* raw, const double* pest,
                         const double* perr, double* out) {
  (void)perr;
  if (m % 2) return fail(-1, "two_level_refine: batch must pair siblings");
  refine(m, est, raw, pest, out);
  return 0;
}

int orc_rel_err_classify(int64_t m, const double* est, const double* err, double tau,
                         int enabled, uint8_t* flags) {
  for (int64_t j = 0; j < m; ++j) {
    const int fin = est[j] == 0.0 ? err[j] == 0.0 : err[j] <= fabs(est[j]) * tau;
    flags[j] = enabled ? (fin ? 0 : 1) : 1;
  }
  return 0;
}

int orc_threshold_classify(int64_t m, const uint8_t* active, const double* errors, double v_tot,
                           double e_tot, double e_it, int64_t s_it, double tau,
                           const orc_config* lim, uint8_t* flags_out, orc_threshold_out* out) {
  if (s_it != m) return fail(-1, "threshold_classify: array length mismatch");
  orc_config L = {0};
  L.direction_change_limit = 4, L.attempt_limit = 40;
  L.p_max_start = 0.25, L.p_max_step = 0.10, L.p_max_cap = 0.95;
  if (lim) L = *lim;
  threshold(active, errors, v_tot, e_tot, e_it, s_it, tau, &L, flags_out, out);
  return 0;
}

int orc_filter(int n, int64_t m, const double* lows, const double* lengths, const double* est,
               const double* err, const int* axis, const double* pest, const double* perr,
               const uint8_t* flags, double* kl, double* kn, double* ke, double* kr, int* ka,
               double* kp, double* kq, int64_t* kept, double* fin_est, double* fin_err,
               double* fin_vol) {
  *fin_est = bsum_where(m, est, flags, 0);
  *fin_err = bsum_where(m, err, flags, 0);
  int64_t k = 0;
  double fv = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    if (!flags[j]) {
      double v = 1.0;
      for (int a = 0; a < n; ++a) v *= lengths[j * n + a];
      fv += v;
      continue;
    }
    memcpy(kl + k * n, lows + j * n, (size_t)n * 8);
    memcpy(kn + k * n, lengths + j * n, (size_t)n * 8);
    ke[k] = est[j], kr[k] = err[j], ka[k] = axis[j], kp[k] = pest[j], kq[k] = perr[j];
    ++k;
  }
  *kept = k;
  *fin_vol = fv;
  return 0;
}

int orc_bisect(int n, int64_t m, const double* lows, const double* lengths, const double* est,
               const double* err, const int* axis, int64_t max_regions, double* cl, double* cn,
               double* cp, double* cq) {
  if (2 * m > max_regions) return fail(-3, "bisect: doubling would exceed max_regions");
  Batch B = {n, m, (double*)lows, (double*)lengths, (double*)est, (double*)err, NULL, NULL,
             (int*)axis};
  uint8_t* all = malloc((size_t)(m ? m : 1));
  memset(all, 1, (size_t)(m ? m : 1));
  Batch out;
  double a, b;
  filter_bisect(&B, all, &a, &b, &out);
  memcpy(cl, out.lows, (size_t)(2 * m * n) * 8);
  memcpy(cn, out.lens, (size_t)(2 * m * n) * 8);
  memcpy(cp, out.pest, (size_t)(2 * m) * 8);
  memcpy(cq, out.perr, (size_t)(2 * m) * 8);
  batch_free(&out);
  free(all);
  return 0;
}

int orc_uniform_split(int n, const double* lo, const double* hi, int d, int64_t maxr,
                      int64_t* count, double* lows, double* lengths, int64_t cap) {
  Batch B;
  const int rc = uniform_split(n, lo, hi, d, maxr, &B);
  if (rc) return rc;
  *count = B.m;
  if (B.m <= cap) {
    memcpy(lows, B.lows, (size_t)(B.m * n) * 8);
    memcpy(lengths, B.lens, (size_t)(B.m * n) * 8);
  }
  batch_free(&B);
  return 0;
}

int orc_initial_subdivisions(int n, int64_t target) { return initial_subdivisions(n, target); }
double orc_block_sum(int64_t m, const double* x) { return bsum_where(m, x, NULL, 0); }
double orc_block_sum_where(int64_t m, const double* x, const uint8_t* f, int which) {
  return bsum_where(m, x, f, which);
}
int orc_digits_converged(double a, double b, int digits) { return digits_converged(a, b, digits); }
int orc_convergence_digits(double tau) { return convergence_digits(tau); }
double orc_reference_value(const char* id, int dim) {
  (void)id, (void)dim;
  return NAN; /* support data, not part of the hot path */
}
double orc_call_integrand(int fid, const double* params, int np, const double* x, int n) {
  Fn F;
  if (make_fn(fid, params, np, &F)) return NAN;
  return call(&F, x, n);
}
