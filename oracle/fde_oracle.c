/* Plain-C CPU restatement of the reference CN-WSGD hot path.
 * TEST INFRASTRUCTURE ONLY -- see fde_oracle.h for the rules and the pinning.
 * Citations are file:line relative to /root/reference/proj unless noted. */
#define _GNU_SOURCE
#include "fde_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[256];
static int fail(const char* m) {
  snprintf(g_err, sizeof g_err, "%s", m);
  return 1;
}
const char* orc_last_error(void) { return g_err; }

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  return p;
}
#define NEWD(n) ((double*)xcalloc((size_t)(n), sizeof(double)))

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* ---------------- synthetic inputs ---------------- */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t src_key(uint64_t seed, uint64_t m, uint64_t j, uint64_t i) {
  return seed ^ (m << 42) ^ (j << 21) ^ i;
}
static double u01(uint64_t key) { return (double)(mix64(key) >> 11) * 0x1.0p-53; }
static double gauss01(uint64_t key) {
  const double a = u01(key), b = u01(key ^ (1ull << 63));
  return sqrt(-2.0 * log(1.0 - a)) * cos(2.0 * M_PI * b);
}

/* ---------------- weights: weights.cpp:21-51 (+ (1,-1), unpinned) -------- */
static int check_gamma(double g) { return (g > 1.0 && g <= 2.0) ? 0 : 1; }

/* g_0 = 1, g_k = g_{k-1} (1 - (gamma+1)/k)          weights.cpp:21-28 */
static void binom(double gamma, int K, double* g) {
  g[0] = 1.0;
  for (int k = 1; k <= K; ++k) g[k] = g[k - 1] * (1.0 - (gamma + 1.0) / (double)k);
}

/* (1,0): w_0 = gamma/2, w_k = (gamma/2) g_k + ((2-gamma)/2) g_{k-1}  weights.cpp:42-47.
 * (1,-1): WSGD l1 = (gamma+2)/4, l2 = (2-gamma)/4, w_k = l1 g_k + l2 g_{k-2}
 * (not in the reference; SURVEY.md 8(a')). */
static void wsgd(double gamma, int K, int pq, double* w) {
  double* g = NEWD(K + 1);
  binom(gamma, K, g);
  if (pq == 0) {
    const double cg = 0.5 * gamma, cg1 = 0.5 * (2.0 - gamma);
    w[0] = cg;
    for (int k = 1; k <= K; ++k) w[k] = cg * g[k] + cg1 * g[k - 1];
  } else {
    const double l1 = (gamma + 2.0) / 4.0, l2 = (2.0 - gamma) / 4.0;
    for (int k = 0; k <= K; ++k) w[k] = l1 * g[k] + (k >= 2 ? l2 * g[k - 2] : 0.0);
  }
  free(g);
}

int orc_wsgd_weights(double gamma, int K, int pq, double* g, double* w) {
  if (check_gamma(gamma)) return fail("weights: gamma must lie in (1, 2]");
  if (K < 2) return fail("weights: K must be >= 2");
  binom(gamma, K, g);
  wsgd(gamma, K, pq, w);
  return 0;
}

/* ---------------- FFT: fft.cpp:11-64 (radix-2 DIT, bit reversal) --------- */
typedef struct { double re, im; } cplx;
static cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}
static void fft_run(int n, cplx* a, int inverse) {
  if (n <= 1) return;
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  for (int i = 0; i < n; ++i) { /* bit-reverse swap, fft.cpp:44-47 */
    int r = 0;
    for (int b = 0; b < lg; ++b) r |= ((i >> b) & 1) << (lg - 1 - b);
    if (i < r) { cplx t = a[i]; a[i] = a[r]; a[r] = t; }
  }
  for (int s = 0; s < lg; ++s) { /* stages with half-block h = 2^s, fft.cpp:48-53 */
    const int h = 1 << s, m = h << 1;
    for (int j = 0; j < h; ++j) {
      const double ang = -M_PI * (double)j / (double)h;
      cplx w = {cos(ang), inverse ? -sin(ang) : sin(ang)};
      for (int b = 0; b < n; b += m) {
        cplx t = cmul(w, a[b + h + j]);
        cplx lo = a[b + j];
        a[b + h + j].re = lo.re - t.re; a[b + h + j].im = lo.im - t.im;
        a[b + j].re = lo.re + t.re; a[b + j].im = lo.im + t.im;
      }
    }
  }
  if (inverse) /* fft.cpp:60-64 */
    for (int i = 0; i < n; ++i) { a[i].re /= (double)n; a[i].im /= (double)n; }
}
int orc_fft(int n, double* a, int inverse) {
  if (n > 0 && (n & (n - 1))) return fail("fft: size not a power of two");
  fft_run(n, (cplx*)a, inverse);
  return 0;
}
int orc_naive_dft(int n, const double* in, double* out, int inverse) { /* fft.cpp:66-80 */
  const cplx* a = (const cplx*)in;
  cplx* o = (cplx*)out;
  const double sgn = inverse ? 1.0 : -1.0;
  for (int k = 0; k < n; ++k) {
    double sr = 0, si = 0;
    for (int j = 0; j < n; ++j) {
      const double ang = sgn * 2.0 * M_PI * (double)k * (double)j / (double)n;
      const double c = cos(ang), s = sin(ang);
      sr += a[j].re * c - a[j].im * s;
      si += a[j].re * s + a[j].im * c;
    }
    o[k].re = inverse ? sr / n : sr;
    o[k].im = inverse ? si / n : si;
  }
  return 0;
}

/* ---------------- Toeplitz block: structured.cpp:21-89 -------------------- */
typedef struct {
  int n, L;
  double *col, *row;
  cplx *spec, *spec_t;
} tblock;

static cplx* symbol(int n, int L, const double* col, const double* row) { /* structured.cpp:21-30 */
  cplx* c = (cplx*)xcalloc((size_t)L, sizeof(cplx));
  for (int i = 0; i < n; ++i) c[i].re = col[i];
  for (int j = 1; j < n; ++j) c[L - j].re = row[j];
  fft_run(L, c, 0);
  return c;
}
static int tb_init(tblock* t, int n, const double* col, const double* row) { /* :34-45 */
  if (n <= 0) return fail("toeplitz column and row sizes must match");
  if (col[0] != row[0]) return fail("toeplitz corner entry mismatch");
  t->n = n;
  t->L = next_pow2(2 * n - 1);
  t->col = NEWD(n);
  t->row = NEWD(n);
  memcpy(t->col, col, sizeof(double) * n);
  memcpy(t->row, row, sizeof(double) * n);
  t->spec = symbol(n, t->L, t->col, t->row);
  t->spec_t = symbol(n, t->L, t->row, t->col);
  return 0;
}
/* ToeplitzBlock::fractional, structured.cpp:47-55 (pq selects the weight table) */
static int tb_fractional(tblock* t, double gamma, int n, int pq) {
  if (n <= 0) return fail("empty toeplitz block");
  if (check_gamma(gamma)) return fail("weights: gamma must lie in (1, 2]");
  const int K = n < 2 ? 2 : n;
  double* w = NEWD(K + 1);
  wsgd(gamma, K, pq, w);
  double *col = NEWD(n), *row = NEWD(n);
  for (int i = 0; i < n; ++i) col[i] = -w[i + 1];
  row[0] = -w[1];
  if (n > 1) row[1] = -w[0];
  const int rc = tb_init(t, n, col, row);
  free(w); free(col); free(row);
  return rc;
}
static void tb_free(tblock* t) {
  free(t->col); free(t->row); free(t->spec); free(t->spec_t);
}
/* apply_both: one forward FFT, two spectral products, two inverse FFTs
 * (structured.cpp:74-89).  scratch: 3L complex. */
static void tb_apply_both(const tblock* t, const double* x, double* y, double* yt,
                          cplx* scratch) {
  const int L = t->L, n = t->n;
  cplx *in = scratch, *a = scratch + L, *b = scratch + 2 * L;
  for (int i = 0; i < L; ++i) { in[i].re = i < n ? x[i] : 0.0; in[i].im = 0.0; }
  fft_run(L, in, 0);
  for (int i = 0; i < L; ++i) { a[i] = cmul(in[i], t->spec[i]); b[i] = cmul(in[i], t->spec_t[i]); }
  fft_run(L, a, 1);
  fft_run(L, b, 1);
  for (int i = 0; i < n; ++i) { y[i] = a[i].re; yt[i] = b[i].re; }
}
int orc_toeplitz_apply_colrow(int n, const double* col, const double* row, const double* x,
                              double* y, double* yt) {
  tblock t;
  if (tb_init(&t, n, col, row)) return 1;
  cplx* s = (cplx*)xcalloc(3 * (size_t)t.L, sizeof(cplx));
  tb_apply_both(&t, x, y, yt, s);
  free(s);
  tb_free(&t);
  return 0;
}
int orc_toeplitz_apply_both(double gamma, int n, int pq, const double* x, double* y,
                            double* yt) {
  tblock t;
  if (tb_fractional(&t, gamma, n, pq)) return 1;
  cplx* s = (cplx*)xcalloc(3 * (size_t)t.L, sizeof(cplx));
  tb_apply_both(&t, x, y, yt, s);
  free(s);
  tb_free(&t);
  return 0;
}

/* ---------------- structured operator: structured.cpp:99-166 -------------- */
typedef struct {
  int n1, n2;
  double inv_r, s_over_r;
  tblock ax, ay;
  double *dp, *dm, *ep, *em, *diag;
} sop;

/* ctor validation + diagonal, structured.cpp:99-123 (takes ownership of arrays) */
static int sop_init(sop* o, int n1, int n2, double inv_r, double s_over_r, tblock ax,
                    tblock ay, double* dp, double* dm, double* ep, double* em) {
  const size_t n = (size_t)n1 * (size_t)n2;
  o->n1 = n1; o->n2 = n2; o->inv_r = inv_r; o->s_over_r = s_over_r;
  o->ax = ax; o->ay = ay; o->dp = dp; o->dm = dm; o->ep = ep; o->em = em;
  o->diag = NULL;
  if (n == 0) return fail("empty operator");
  if (ax.n != n1 || ay.n != n2) return fail("toeplitz block size mismatch");
  if (!(inv_r > 0.0)) return fail("1/r must be positive");
  if (!(s_over_r > 0.0)) return fail("s/r must be positive");
  for (size_t p = 0; p < n; ++p)
    if (dp[p] < 0.0 || dm[p] < 0.0 || ep[p] < 0.0 || em[p] < 0.0)
      return fail("negative diffusion coefficient sample");
  const double ax0 = ax.col[0], ay0 = ay.col[0];
  o->diag = NEWD(n);
  for (size_t p = 0; p < n; ++p)
    o->diag[p] = inv_r + (dp[p] + dm[p]) * ax0 + s_over_r * (ep[p] + em[p]) * ay0;
  return 0;
}
static void sop_free(sop* o) {
  tb_free(&o->ax); tb_free(&o->ay);
  free(o->dp); free(o->dm); free(o->ep); free(o->em); free(o->diag);
}
static size_t sop_size(const sop* o) { return (size_t)o->n1 * (size_t)o->n2; }

/* apply_impl, structured.cpp:125-148 */
static void sop_apply_impl(const sop* o, const double* x, double* y, double sign) {
  const int n1 = o->n1, n2 = o->n2;
  const size_t n = sop_size(o);
  for (size_t p = 0; p < n; ++p) y[p] = o->inv_r * x[p];
  const int Lm = o->ax.L > o->ay.L ? o->ax.L : o->ay.L;
  cplx* s = (cplx*)xcalloc(3 * (size_t)Lm, sizeof(cplx));
  double *t = NEWD(n1), *tt = NEWD(n1);
  for (int j = 0; j < n2; ++j) { /* x-lines, contiguous */
    const size_t off = (size_t)j * n1;
    tb_apply_both(&o->ax, x + off, t, tt, s);
    for (int i = 0; i < n1; ++i) y[off + i] += sign * o->dp[off + i] * t[i];
    for (int i = 0; i < n1; ++i) y[off + i] += sign * o->dm[off + i] * tt[i];
  }
  double *xc = NEWD(n2), *tc = NEWD(n2), *ttc = NEWD(n2);
  const double c = sign * o->s_over_r;
  for (int i = 0; i < n1; ++i) { /* y-lines, gathered with stride n1 */
    for (int j = 0; j < n2; ++j) xc[j] = x[i + (size_t)j * n1];
    tb_apply_both(&o->ay, xc, tc, ttc, s);
    for (int j = 0; j < n2; ++j) {
      const size_t p = i + (size_t)j * n1;
      y[p] += c * (o->ep[p] * tc[j] + o->em[p] * ttc[j]);
    }
  }
  free(s); free(t); free(tt); free(xc); free(tc); free(ttc);
}
static void sop_apply(const sop* o, const double* x, double* y) { sop_apply_impl(o, x, y, 1.0); }

/* scale, structured.cpp:154-162 */
static void sop_scale(sop* o, double s) {
  const size_t n = sop_size(o);
  o->inv_r *= s;
  o->s_over_r *= s;
  for (size_t p = 0; p < n; ++p) { o->dp[p] *= s; o->dm[p] *= s; o->diag[p] *= s; }
}

/* ---------------- problem / grid: problem.cpp:27-89 + SURVEY App. A ------- */
typedef struct {
  int cfg, n1, n2, steps, pq, skind;
  double alpha, beta, tau, t_final;
  double hx, hy, dt, inv_r, s_over_r;
  uint64_t seed;
} prob;

static int setup(const orc_spec* s, prob* p) {
  int n = 63, steps = 64, pq = 0, skind = 0;
  double al = 1.8, be = 1.6, tau = 1.0 / 64;
  switch (s->cfg) {
    case 0: case 1: break;
    case 2: n = 255; al = 1.5; be = 1.7; tau = 1.0 / 256; steps = 32; break;
    case 3: n = 1023; al = 1.1; be = 1.9; tau = 1.0 / 128; steps = 16; pq = 1; skind = 1; break;
    case 4: n = 2047; al = 1.6; be = 1.4; tau = 1.0 / 64; steps = 8; break;
    case 5: n = 2047; al = 1.7; be = 1.3; tau = 1.0 / 64; steps = 1; break;
    default: return fail("unknown config id");
  }
  p->cfg = s->cfg;
  p->n1 = s->n1 > 0 ? s->n1 : n;
  p->n2 = s->n2 > 0 ? s->n2 : n;
  p->steps = s->steps > 0 ? s->steps : steps;
  p->tau = s->tau > 0 ? s->tau : tau;
  p->alpha = s->alpha > 0 ? s->alpha : al;
  p->beta = s->beta > 0 ? s->beta : be;
  p->pq = s->pq >= 0 ? s->pq : pq;
  p->skind = s->source_kind >= 0 ? s->source_kind : skind;
  p->seed = s->seed;
  p->t_final = p->tau * (double)p->steps;
  /* Grid ctor, problem.cpp:27-48 on [0,1]^2 */
  p->hx = 1.0 / (double)(p->n1 + 1);
  p->hy = 1.0 / (double)(p->n2 + 1);
  p->dt = p->t_final / (double)p->steps;
  const double r = p->dt / (2.0 * pow(p->hx, p->alpha));
  const double sy = p->dt / (2.0 * pow(p->hy, p->beta));
  p->inv_r = 1.0 / r;
  p->s_over_r = sy / r;
  return 0;
}
/* level grid with the same time step (multigrid.cpp:421-423) */
static prob level_prob(const prob* f, int d1, int d2) {
  prob p = *f;
  p.n1 = d1; p.n2 = d2;
  p.hx = 1.0 / (double)(d1 + 1);
  p.hy = 1.0 / (double)(d2 + 1);
  p.dt = p.t_final / (double)p.steps;
  const double r = p.dt / (2.0 * pow(p.hx, p.alpha));
  const double sy = p.dt / (2.0 * pow(p.hy, p.beta));
  p.inv_r = 1.0 / r;
  p.s_over_r = sy / r;
  return p;
}

/* Coefficient fields of the BASELINE configs.  cfg5 uses the
 * reference coefficient preset 1, problem.cpp:196-209, on [0,1]^2. */
static void coeffs_at(const prob* p, double x, double y, double* dp, double* dm, double* ep,
                      double* em) {
  switch (p->cfg) {
    case 2: case 4:
      *dp = 1.0 + x + y; *dm = 2.0 - x + y; *ep = 1.0 + x * y; *em = 1.0 + (1.0 - x) * (1.0 - y);
      return;
    case 3: {
      const double s = sin(M_PI * x), c = cos(M_PI * y);
      *dp = 1.0 + s * s; *dm = 1.0 + c * c; *ep = 2.0 + x - y; *em = 2.0 - x + y;
      return;
    }
    case 5: {
      const double ax = 0.0, bx = 1.0, ay = 0.0, by = 1.0;
      const double ga = tgamma(3.0 - p->alpha), gb = tgamma(3.0 - p->beta);
      *dp = ga * pow(1.0 + x - ax, p->alpha) * (1.0 + y - ay) * (1.0 + y - ay);
      *dm = ga * pow(1.0 + bx - x, p->alpha) * (1.0 + by - y) * (1.0 + by - y);
      *ep = gb * (1.0 + x - ax) * (1.0 + x - ax) * pow(1.0 + y - ay, p->beta);
      *em = gb * (1.0 + bx - x) * (1.0 + bx - x) * pow(1.0 + by - y, p->beta);
      return;
    }
    default: *dp = *dm = *ep = *em = 1.0; return;
  }
}
static double gx(const prob* p, int i) { return 0.0 + p->hx * (double)(i + 1); } /* problem.hpp:46 */
static double gy(const prob* p, int j) { return 0.0 + p->hy * (double)(j + 1); }

/* assemble_step_operator, problem.cpp:50-71 */
static int assemble(const prob* p, sop* o) {
  const size_t n = (size_t)p->n1 * p->n2;
  double *dp = NEWD(n), *dm = NEWD(n), *ep = NEWD(n), *em = NEWD(n);
  for (int j = 0; j < p->n2; ++j)
    for (int i = 0; i < p->n1; ++i) {
      const size_t q = i + (size_t)j * p->n1;
      coeffs_at(p, gx(p, i), gy(p, j), dp + q, dm + q, ep + q, em + q);
    }
  tblock ax, ay;
  if (tb_fractional(&ax, p->alpha, p->n1, p->pq)) return 1;
  if (tb_fractional(&ay, p->beta, p->n2, p->pq)) return 1;
  return sop_init(o, p->n1, p->n2, p->inv_r, p->s_over_r, ax, ay, dp, dm, ep, em);
}

static double source_at(const prob* p, int m, int j, int i) {
  if (p->skind == 2) return 0.0;
  const uint64_t key = src_key(p->seed, (uint64_t)m, (uint64_t)j, (uint64_t)i);
  return p->skind == 1 ? 1e-2 * gauss01(key) : u01(key);
}

/* ---------------- multigrid planning: multigrid.cpp:114-158 ---------------- */
static int coarse_size(int n) { return (n - n % 2) / 2; }

/* eval_q_gamma(gamma, pi), symbols.cpp:14-33 */
static double q_gamma_pi(double gamma) {
  const double xi = M_PI;
  const double s = sin(0.5 * xi), c = cos(0.5 * xi);
  const double complex z = 2.0 * s * s + I * (-2.0 * s * c);
  const double complex factor = -(1.0 - 0.5 * gamma * conj(z));
  return 2.0 * creal(factor * cpow(z, gamma));
}
static double aniso(const sop* o, double alpha, double beta) { /* multigrid.cpp:116-128 */
  const size_t n = sop_size(o);
  double sx = 0.0, sy = 0.0;
  for (size_t i = 0; i < n; ++i) sx += o->dp[i] + o->dm[i];
  for (size_t i = 0; i < n; ++i) sy += o->ep[i] + o->em[i];
  const double cx = sx / (double)n * q_gamma_pi(alpha);
  const double cy = o->s_over_r * (sy / (double)n) * q_gamma_pi(beta);
  return cy / cx;
}
static int plan(int n1, int n2, double ratio0, double alpha, double beta, int* dims, int maxl) {
  int nl = 1;
  dims[0] = n1; dims[1] = n2;
  while (dims[2 * (nl - 1)] > 8 || dims[2 * (nl - 1) + 1] > 8) {
    const int d1 = dims[2 * (nl - 1)], d2 = dims[2 * (nl - 1) + 1];
    const double ratio = ratio0 * pow((double)(n1 + 1) / (double)(d1 + 1), alpha) /
                         pow((double)(n2 + 1) / (double)(d2 + 1), beta);
    int cx = 1, cy = 1;
    if (ratio > 5.0) cx = 0;
    else if (ratio < 1.0 / 5.0) cy = 0;
    if (!cx && d2 <= 8) cx = 1;
    if (!cy && d1 <= 8) cy = 1;
    const int k1 = cx ? coarse_size(d1) : d1, k2 = cy ? coarse_size(d2) : d2;
    if ((cx && k1 == 0) || (cy && k2 == 0)) break;
    if (nl >= maxl) return -1;
    dims[2 * nl] = k1; dims[2 * nl + 1] = k2;
    ++nl;
  }
  return nl;
}
int orc_plan_raw(int n1, int n2, double ratio0, double alpha, double beta, int* dims,
                 int max_levels) {
  return plan(n1, n2, ratio0, alpha, beta, dims, max_levels);
}

/* ---------------- grid transfer: multigrid.cpp:17-71,160-201 -------------- */
typedef struct { int n1, n2, k1, k2, par1, par2, cx, cy; } xfer;
static int xfer_init(xfer* t, int n1, int n2, int cx, int cy) {
  t->n1 = n1; t->n2 = n2;
  t->k1 = cx ? coarse_size(n1) : n1;
  t->k2 = cy ? coarse_size(n2) : n2;
  t->par1 = (n1 + 1) % 2; t->par2 = (n2 + 1) % 2;
  t->cx = cx; t->cy = cy;
  if (t->k1 == 0 || t->k2 == 0 || (!cx && !cy)) return fail("grid too small to coarsen");
  return 0;
}
static void prolong_rows(int k, int n, int par, int nrows, const double* c, double* f) {
  memset(f, 0, sizeof(double) * (size_t)n * nrows);
  for (int r = 0; r < nrows; ++r) {
    const double* cr = c + (size_t)r * k;
    double* fr = f + (size_t)r * n;
    for (int j = 0; j < k; ++j) {
      const int fc = 2 * j + 1 - par;
      fr[fc] += cr[j];
      if (fc > 0) fr[fc - 1] += 0.5 * cr[j];
      if (fc + 1 < n) fr[fc + 1] += 0.5 * cr[j];
    }
  }
}
static void prolong_cols(int k, int n, int par, int width, const double* c, double* f) {
  memset(f, 0, sizeof(double) * (size_t)n * width);
  for (int j = 0; j < k; ++j) {
    const int fc = 2 * j + 1 - par;
    const double* cr = c + (size_t)j * width;
    for (int i = 0; i < width; ++i) f[(size_t)fc * width + i] += 1.0 * cr[i];
    if (fc > 0) for (int i = 0; i < width; ++i) f[(size_t)(fc - 1) * width + i] += 0.5 * cr[i];
    if (fc + 1 < n) for (int i = 0; i < width; ++i) f[(size_t)(fc + 1) * width + i] += 0.5 * cr[i];
  }
}
static void restrict_rows(int n, int k, int par, int nrows, double sc, const double* f,
                          double* c) {
  for (int r = 0; r < nrows; ++r) {
    const double* fr = f + (size_t)r * n;
    double* cr = c + (size_t)r * k;
    for (int j = 0; j < k; ++j) {
      const int fc = 2 * j + 1 - par;
      double v = fr[fc];
      if (fc > 0) v += 0.5 * fr[fc - 1];
      if (fc + 1 < n) v += 0.5 * fr[fc + 1];
      cr[j] = sc * v;
    }
  }
}
static void restrict_cols(int n, int k, int par, int width, double sc, const double* f,
                          double* c) {
  for (int j = 0; j < k; ++j) {
    const int fc = 2 * j + 1 - par;
    double* cr = c + (size_t)j * width;
    for (int i = 0; i < width; ++i) cr[i] = f[(size_t)fc * width + i];
    if (fc > 0) for (int i = 0; i < width; ++i) cr[i] += 0.5 * f[(size_t)(fc - 1) * width + i];
    if (fc + 1 < n) for (int i = 0; i < width; ++i) cr[i] += 0.5 * f[(size_t)(fc + 1) * width + i];
    for (int i = 0; i < width; ++i) cr[i] *= sc;
  }
}
static void xfer_prolong(const xfer* t, const double* c, double* f) {
  if (!t->cx) { prolong_cols(t->k2, t->n2, t->par2, t->n1, c, f); return; }
  if (!t->cy) { prolong_rows(t->k1, t->n1, t->par1, t->k2, c, f); return; }
  double* tmp = NEWD((size_t)t->n1 * t->k2);
  prolong_rows(t->k1, t->n1, t->par1, t->k2, c, tmp);
  prolong_cols(t->k2, t->n2, t->par2, t->n1, tmp, f);
  free(tmp);
}
static void xfer_restrict(const xfer* t, const double* f, double* c, double sc) {
  if (!t->cx) { restrict_cols(t->n2, t->k2, t->par2, t->k1, sc, f, c); return; }
  if (!t->cy) { restrict_rows(t->n1, t->k1, t->par1, t->n2, sc, f, c); return; }
  double* tmp = NEWD((size_t)t->k1 * t->n2);
  restrict_rows(t->n1, t->k1, t->par1, t->n2, sc, f, tmp);
  restrict_cols(t->n2, t->k2, t->par2, t->k1, sc, tmp, c);
  free(tmp);
}
int orc_transfer(int n1, int n2, int cx, int cy, int op, const double* in, double* out) {
  xfer t;
  if (xfer_init(&t, n1, n2, cx, cy)) return 1;
  if (op == 0) xfer_prolong(&t, in, out);
  else xfer_restrict(&t, in, out, op == 1 ? 0.5 : 1.0);
  return 0;
}

/* ---------------- CSR (P2 Galerkin path): sparse.cpp:8-140 --------------- */
typedef struct { int rows, cols; int *ptr, *idx; double* val; } csr;
typedef struct { int r, c; double v; } trip;
static int trip_cmp(const void* a, const void* b) {
  const trip *x = (const trip*)a, *y = (const trip*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  return x->c < y->c ? -1 : (x->c > y->c);
}
/* from_triplets: sorted columns, duplicates summed (sparse.cpp:8-38) */
static csr csr_from(int rows, int cols, trip* t, size_t nt) {
  qsort(t, nt, sizeof(trip), trip_cmp);
  csr a = {rows, cols, (int*)xcalloc((size_t)rows + 1, sizeof(int)),
           (int*)xcalloc(nt, sizeof(int)), NEWD(nt)};
  size_t nz = 0;
  for (size_t k = 0; k < nt; ++k) {
    if (nz > 0 && k > 0 && t[k].r == t[k - 1].r && t[k].c == t[k - 1].c) {
      a.val[nz - 1] += t[k].v;
    } else {
      a.idx[nz] = t[k].c;
      a.val[nz] = t[k].v;
      ++nz;
      a.ptr[t[k].r + 1]++;
    }
  }
  for (int r = 0; r < rows; ++r) a.ptr[r + 1] += a.ptr[r];
  return a;
}
static void csr_free(csr* a) { free(a->ptr); free(a->idx); free(a->val); }
static void csr_apply(const csr* a, const double* x, double* y) { /* sparse.cpp:42-49 */
  for (int r = 0; r < a->rows; ++r) {
    double s = 0.0;
    for (int k = a->ptr[r]; k < a->ptr[r + 1]; ++k) s += a->val[k] * x[a->idx[k]];
    y[r] = s;
  }
}
static csr csr_transpose(const csr* a) {
  size_t nz = (size_t)a->ptr[a->rows];
  trip* t = (trip*)xcalloc(nz, sizeof(trip));
  size_t q = 0;
  for (int r = 0; r < a->rows; ++r)
    for (int k = a->ptr[r]; k < a->ptr[r + 1]; ++k) { t[q].r = a->idx[k]; t[q].c = r; t[q].v = a->val[k]; ++q; }
  csr o = csr_from(a->cols, a->rows, t, nz);
  free(t);
  return o;
}
/* Gustavson product (sparse.cpp:71-103): accumulate in row order of the left factor. */
static csr csr_mul(const csr* a, const csr* b) {
  double* acc = NEWD(b->cols);
  int* mark = (int*)xcalloc((size_t)b->cols, sizeof(int));
  int* live = (int*)xcalloc((size_t)b->cols, sizeof(int));
  for (int c = 0; c < b->cols; ++c) mark[c] = -1;
  size_t cap = 16, nt = 0;
  trip* t = (trip*)xcalloc(cap, sizeof(trip));
  for (int r = 0; r < a->rows; ++r) {
    int nl = 0;
    for (int k = a->ptr[r]; k < a->ptr[r + 1]; ++k) {
      const int mid = a->idx[k];
      const double va = a->val[k];
      for (int l = b->ptr[mid]; l < b->ptr[mid + 1]; ++l) {
        const int c = b->idx[l];
        if (mark[c] != r) { mark[c] = r; acc[c] = va * b->val[l]; live[nl++] = c; }
        else acc[c] += va * b->val[l];
      }
    }
    for (int q = 0; q < nl; ++q) {
      if (nt == cap) { cap *= 2; t = (trip*)realloc(t, cap * sizeof(trip)); }
      t[nt].r = r; t[nt].c = live[q]; t[nt].v = acc[live[q]]; ++nt;
    }
  }
  csr o = csr_from(a->rows, b->cols, t, nt);
  free(t); free(acc); free(mark); free(live);
  return o;
}
/* build_p2 (precond.cpp:50-73): 5-point order-2 companion of the step operator */
static csr build_p2(const sop* o) {
  const int n1 = o->n1, n2 = o->n2;
  const size_t n = sop_size(o);
  trip* t = (trip*)xcalloc(5 * n, sizeof(trip));
  size_t q = 0;
  for (int j = 0; j < n2; ++j)
    for (int i = 0; i < n1; ++i) {
      const int p = i + j * n1;
      const double cx = o->dp[p] + o->dm[p];
      const double cy = o->s_over_r * (o->ep[p] + o->em[p]);
      t[q++] = (trip){p, p, o->inv_r + 2.0 * cx + 2.0 * cy};
      if (i > 0) t[q++] = (trip){p, p - 1, -cx};
      if (i + 1 < n1) t[q++] = (trip){p, p + 1, -cx};
      if (j > 0) t[q++] = (trip){p, p - n1, -cy};
      if (j + 1 < n2) t[q++] = (trip){p, p + n1, -cy};
    }
  csr a = csr_from((int)n, (int)n, t, q);
  free(t);
  return a;
}
/* GridTransfer::prolong_matrix, multigrid.cpp:229-253 */
static csr prolong_matrix(const xfer* x) {
  const double wt[3] = {0.5, 1.0, 0.5};
  const int ri = x->cx ? 1 : 0, rj = x->cy ? 1 : 0;
  trip* t = (trip*)xcalloc(9 * (size_t)x->k1 * x->k2, sizeof(trip));
  size_t q = 0;
  for (int b = 0; b < x->k2; ++b) {
    const int fb = x->cy ? 2 * b + 1 - x->par2 : b;
    for (int a = 0; a < x->k1; ++a) {
      const int fa = x->cx ? 2 * a + 1 - x->par1 : a;
      const int col = a + b * x->k1;
      for (int dj = -rj; dj <= rj; ++dj) {
        const int j = fb + dj;
        if (j < 0 || j >= x->n2) continue;
        for (int di = -ri; di <= ri; ++di) {
          const int i = fa + di;
          if (i < 0 || i >= x->n1) continue;
          t[q++] = (trip){i + j * x->n1, col, wt[di + 1] * wt[dj + 1]};
        }
      }
    }
  }
  csr p = csr_from(x->n1 * x->n2, x->k1 * x->k2, t, q);
  free(t);
  return p;
}

/* ---------------- V-cycle hierarchy: multigrid.cpp:284-441 ---------------- */
enum { COARSE_LU = 0, COARSE_SWEEPS = 1, COARSE_NONE = 2 };
typedef struct {
  int nlev, galerkin, coarse, coarse_sweeps;
  double omega;
  sop* ops;    /* geometric levels */
  csr* mats;   /* galerkin levels */
  double** dinv;
  xfer* tr;
  size_t* size;
  double *lu, *wr, *wt, *wbc, *wxc; /* dense LU of the coarsest level; workspaces */
  int* perm;
  double** r;
  double** t;
  double** bc;
  double** xc;
} hier;

static void lev_apply(const hier* h, int l, const double* x, double* y) {
  if (h->galerkin) csr_apply(&h->mats[l], x, y);
  else sop_apply(&h->ops[l], x, y);
}

/* dense assembly of a level through unit vectors (multigrid.cpp:73-86) and a
 * row-pivoted LU (the coarsest CoarseSolve::lu solve, multigrid.cpp:314-328). */
static int coarse_lu(hier* h) {
  const int l = h->nlev - 1;
  const size_t n = h->size[l];
  if (n > 4096) return fail("operator too large to densify");
  double* a = NEWD(n * n); /* column-major */
  double *e = NEWD(n), *col = NEWD(n);
  for (size_t j = 0; j < n; ++j) {
    e[j] = 1.0;
    lev_apply(h, l, e, col);
    e[j] = 0.0;
    memcpy(a + j * n, col, n * sizeof(double));
  }
  free(e); free(col);
  h->perm = (int*)xcalloc(n, sizeof(int));
  for (size_t i = 0; i < n; ++i) h->perm[i] = (int)i;
#define A(i, j) a[(size_t)(i) + (size_t)(j) * n]
  for (size_t k = 0; k < n; ++k) {
    size_t p = k;
    double best = fabs(A(k, k));
    for (size_t i = k + 1; i < n; ++i)
      if (fabs(A(i, k)) > best) { best = fabs(A(i, k)); p = i; }
    if (p != k) {
      for (size_t j = 0; j < n; ++j) { double t = A(k, j); A(k, j) = A(p, j); A(p, j) = t; }
      int t = h->perm[k]; h->perm[k] = h->perm[p]; h->perm[p] = t;
    }
    const double piv = A(k, k);
    if (piv == 0.0) continue;
    for (size_t i = k + 1; i < n; ++i) {
      const double lv = A(i, k) / piv;
      A(i, k) = lv;
      if (lv == 0.0) continue;
      for (size_t j = k + 1; j < n; ++j) A(i, j) -= lv * A(k, j);
    }
  }
#undef A
  h->lu = a;
  return 0;
}
static void lu_solve(const hier* h, const double* b, double* x) {
  const size_t n = h->size[h->nlev - 1];
  const double* a = h->lu;
  double* y = NEWD(n);
  for (size_t i = 0; i < n; ++i) {
    double v = b[h->perm[i]];
    for (size_t j = 0; j < i; ++j) v -= a[i + j * n] * y[j];
    y[i] = v;
  }
  for (size_t i = n; i-- > 0;) {
    double v = y[i];
    for (size_t j = i + 1; j < n; ++j) v -= a[i + j * n] * x[j];
    x[i] = v / a[i + i * n];
  }
  free(y);
}

static int hier_finish(hier* h) { /* MgHierarchy ctor, multigrid.cpp:301-316 */
  if (!(h->omega > 0.0)) return fail("omega must be positive");
  if (h->coarse == COARSE_SWEEPS && h->coarse_sweeps == 0)
    return fail("coarse_sweeps must be positive");
  h->dinv = (double**)xcalloc((size_t)h->nlev, sizeof(double*));
  h->r = (double**)xcalloc((size_t)h->nlev, sizeof(double*));
  h->t = (double**)xcalloc((size_t)h->nlev, sizeof(double*));
  h->bc = (double**)xcalloc((size_t)h->nlev, sizeof(double*));
  h->xc = (double**)xcalloc((size_t)h->nlev, sizeof(double*));
  for (int l = 0; l < h->nlev; ++l) {
    const size_t n = h->size[l];
    h->dinv[l] = NEWD(n);
    for (size_t i = 0; i < n; ++i) {
      double d = 0.0;
      if (h->galerkin) { /* Csr::diag, sparse.cpp:105-120 */
        const csr* a = &h->mats[l];
        for (int k = a->ptr[i]; k < a->ptr[i + 1]; ++k)
          if (a->idx[k] == (int)i) { d = a->val[k]; break; }
      } else {
        d = h->ops[l].diag[i];
      }
      if (!(d > 0.0)) return fail("operator diagonal must be strictly positive");
      h->dinv[l][i] = 1.0 / d;
    }
    h->r[l] = NEWD(n); h->t[l] = NEWD(n); h->bc[l] = NEWD(n); h->xc[l] = NEWD(n);
  }
  if (h->coarse == COARSE_LU) return coarse_lu(h);
  return 0;
}

static int hier_geometric(const prob* p, int omega_set, double omega, int coarse, int sweeps,
                          hier* h) {
  (void)omega_set;
  memset(h, 0, sizeof *h);
  sop fine;
  if (assemble(p, &fine)) return 1;
  int dims[128];
  const int nl = plan(p->n1, p->n2, aniso(&fine, p->alpha, p->beta), p->alpha, p->beta, dims, 64);
  if (nl < 1) return fail("level plan overflow");
  h->nlev = nl;
  h->omega = omega; h->coarse = coarse; h->coarse_sweeps = sweeps;
  h->ops = (sop*)xcalloc((size_t)nl, sizeof(sop));
  h->tr = (xfer*)xcalloc((size_t)nl, sizeof(xfer));
  h->size = (size_t*)xcalloc((size_t)nl, sizeof(size_t));
  h->ops[0] = fine;
  for (int l = 1; l < nl; ++l) { /* multigrid.cpp:416-431 */
    const prob lp = level_prob(p, dims[2 * l], dims[2 * l + 1]);
    if (assemble(&lp, &h->ops[l])) return 1;
    sop_scale(&h->ops[l], pow(p->hx / lp.hx, p->alpha));
  }
  for (int l = 0; l < nl; ++l) h->size[l] = (size_t)dims[2 * l] * dims[2 * l + 1];
  for (int l = 0; l + 1 < nl; ++l)
    if (xfer_init(&h->tr[l], dims[2 * l], dims[2 * l + 1], dims[2 * l + 2] < dims[2 * l],
                  dims[2 * l + 3] < dims[2 * l + 1]))
      return 1;
  return hier_finish(h);
}

/* build_galerkin_hierarchy on P2 (precond.cpp:75-83, multigrid.cpp:443-475):
 * default full-coarsening plan level_dims (multigrid.cpp:98-110), coarsest none. */
static int hier_p2(const prob* p, double omega, hier* h) {
  memset(h, 0, sizeof *h);
  sop fine;
  if (assemble(p, &fine)) return 1;
  int dims[128], nl = 1;
  dims[0] = p->n1; dims[1] = p->n2;
  while (dims[2 * (nl - 1)] > 8 || dims[2 * (nl - 1) + 1] > 8) {
    const int k1 = coarse_size(dims[2 * (nl - 1)]), k2 = coarse_size(dims[2 * (nl - 1) + 1]);
    if (k1 == 0 || k2 == 0) break;
    dims[2 * nl] = k1; dims[2 * nl + 1] = k2;
    ++nl;
  }
  h->nlev = nl; h->galerkin = 1; h->omega = omega; h->coarse = COARSE_NONE; h->coarse_sweeps = 3;
  h->mats = (csr*)xcalloc((size_t)nl, sizeof(csr));
  h->tr = (xfer*)xcalloc((size_t)nl, sizeof(xfer));
  h->size = (size_t*)xcalloc((size_t)nl, sizeof(size_t));
  h->mats[0] = build_p2(&fine);
  sop_free(&fine);
  for (int l = 0; l < nl; ++l) h->size[l] = (size_t)dims[2 * l] * dims[2 * l + 1];
  for (int l = 0; l + 1 < nl; ++l)
    if (xfer_init(&h->tr[l], dims[2 * l], dims[2 * l + 1], dims[2 * l + 2] < dims[2 * l],
                  dims[2 * l + 3] < dims[2 * l + 1]))
      return 1;
  for (int l = 1; l < nl; ++l) { /* rap(P, A) = P^T (A P), sparse.cpp:131-136 */
    csr P = prolong_matrix(&h->tr[l - 1]);
    csr ap = csr_mul(&h->mats[l - 1], &P);
    csr pt = csr_transpose(&P);
    h->mats[l] = csr_mul(&pt, &ap);
    csr_free(&P); csr_free(&ap); csr_free(&pt);
  }
  return hier_finish(h);
}

static void hier_free(hier* h) {
  for (int l = 0; l < h->nlev; ++l) {
    if (h->ops) sop_free(&h->ops[l]);
    if (h->mats) csr_free(&h->mats[l]);
    if (h->dinv) free(h->dinv[l]);
    if (h->r) { free(h->r[l]); free(h->t[l]); free(h->bc[l]); free(h->xc[l]); }
  }
  free(h->ops); free(h->mats); free(h->dinv); free(h->tr); free(h->size); free(h->lu);
  free(h->perm); free(h->r); free(h->t); free(h->bc); free(h->xc);
}

/* MgHierarchy::cycle, multigrid.cpp:318-383 */
static void cycle(const hier* h, int l, const double* b, double* x, int zero) {
  const size_t n = h->size[l];
  const double w = h->omega;
  const double* dinv = h->dinv[l];
  double *r = h->r[l], *t = h->t[l];
  if (l + 1 == h->nlev) {
    if (h->coarse == COARSE_LU) {
      lu_solve(h, b, x);
    } else if (h->coarse == COARSE_SWEEPS) {
      if (zero) {
        for (size_t i = 0; i < n; ++i) x[i] = w * dinv[i] * b[i];
      } else {
        lev_apply(h, l, x, t);
        for (size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
        for (size_t i = 0; i < n; ++i) x[i] += w * dinv[i] * r[i];
      }
      for (int k = 1; k < h->coarse_sweeps; ++k) {
        lev_apply(h, l, x, t);
        for (size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
        for (size_t i = 0; i < n; ++i) x[i] += w * dinv[i] * r[i];
      }
    }
    return;
  }
  if (zero) {
    for (size_t i = 0; i < n; ++i) x[i] = w * dinv[i] * b[i];
  } else {
    lev_apply(h, l, x, t);
    for (size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
    for (size_t i = 0; i < n; ++i) x[i] += w * dinv[i] * r[i];
  }
  lev_apply(h, l, x, t);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
  const size_t nc = h->size[l + 1];
  double *bc = h->bc[l + 1], *xc = h->xc[l + 1];
  xfer_restrict(&h->tr[l], r, bc, h->galerkin ? 1.0 : 0.5);
  memset(xc, 0, nc * sizeof(double));
  cycle(h, l + 1, bc, xc, 1);
  xfer_prolong(&h->tr[l], xc, t);
  for (size_t i = 0; i < n; ++i) x[i] += 1.0 * t[i];
  lev_apply(h, l, x, t);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
  for (size_t i = 0; i < n; ++i) x[i] += w * dinv[i] * r[i];
}
static void vcycle(const hier* h, const double* b, double* x) { /* multigrid.cpp:385-394 */
  int zero = 1;
  for (size_t i = 0; i < h->size[0]; ++i)
    if (x[i] != 0.0) { zero = 0; break; }
  cycle(h, 0, b, x, zero);
}

/* ---------------- preconditioner (precond.cpp:22-26,103-114) -------------- */
typedef struct {
  int kind; /* 0 none, 1 p2, 2 mgm */
  int cycles;
  size_t n;
  hier h;
} pcond;
static int pc_make(const orc_spec* s, const prob* p, pcond* pc) {
  memset(pc, 0, sizeof *pc);
  pc->kind = s->precond;
  pc->cycles = s->cycles > 0 ? s->cycles : 1;
  pc->n = (size_t)p->n1 * p->n2;
  if (s->precond == 2) return hier_geometric(p, 1, s->omega, s->coarse, s->coarse_sweeps, &pc->h);
  if (s->precond == 1) return hier_p2(p, s->omega, &pc->h);
  return 0;
}
static void pc_apply(const pcond* pc, const double* r, double* z) {
  if (pc->kind == 0) { memcpy(z, r, pc->n * sizeof(double)); return; }
  memset(z, 0, pc->n * sizeof(double));
  for (int c = 0; c < pc->cycles; ++c) vcycle(&pc->h, r, z);
}
static void pc_free(pcond* pc) {
  if (pc->kind) hier_free(&pc->h);
}

/* ---------------- Krylov: krylov.cpp:12-166 ------------------------------- */
static double dot(size_t n, const double* x, const double* y) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
static double nrm2(size_t n, const double* x) { return sqrt(dot(n, x, x)); }

typedef struct {
  double* x;
  int iterations, converged, nh, caph;
  double* hist;
} kres;
static void hist_push(kres* r, double v) {
  if (r->nh == r->caph) { r->caph = r->caph ? 2 * r->caph : 64; r->hist = (double*)realloc(r->hist, sizeof(double) * r->caph); }
  r->hist[r->nh++] = v;
}

static void back_sub(const double* h, int ld, const double* g, int k, double* y) {
  for (int i = k; i-- > 0;) {
    double v = g[i];
    for (int j = i + 1; j < k; ++j) v -= h[j * ld + i] * y[j];
    y[i] = h[i * ld + i] != 0.0 ? v / h[i * ld + i] : 0.0;
  }
}

/* ||M^-1 (b - A x)|| / norm_b, the true_rel lambda of krylov.cpp:59-64 */
static double true_rel(const sop* a, const pcond* m, const double* b, const double* x,
                       double* t, double* r, double* z, double norm_b) {
  const size_t n = sop_size(a);
  sop_apply(a, x, t);
  for (size_t q = 0; q < n; ++q) r[q] = b[q] - t[q];
  pc_apply(m, r, z);
  return nrm2(n, z) / norm_b;
}

static int gmres(const sop* a, const pcond* m, double tol, int rst, int max_outer,
                 const double* b, kres* res) {
  const size_t n = sop_size(a);
  if (rst <= 0 || !(tol > 0.0)) return fail("invalid solver configuration");
  memset(res, 0, sizeof *res);
  res->x = NEWD(n);
  double* x = res->x;
  double *t = NEWD(n), *r = NEWD(n), *z = NEWD(n), *w = NEWD(n), *trial = NEWD(n);
  pc_apply(m, b, z);
  const double norm_b = nrm2(n, z);
  if (norm_b == 0.0) {
    res->converged = 1;
    hist_push(res, 0.0);
    free(t); free(r); free(z); free(w); free(trial);
    return 0;
  }
  const int ld = rst + 1;
  double** v = (double**)xcalloc((size_t)rst + 1, sizeof(double*));
  for (int k = 0; k <= rst; ++k) v[k] = NEWD(n);
  double *h = NEWD((size_t)ld * rst), *g = NEWD(ld), *cs = NEWD(rst), *sn = NEWD(rst),
         *y = NEWD(rst);
  for (int outer = 0; outer < max_outer && !res->converged; ++outer) {
    sop_apply(a, x, t);
    for (size_t q = 0; q < n; ++q) r[q] = b[q] - t[q];
    pc_apply(m, r, z);
    const double beta = nrm2(n, z);
    const double rel0 = beta / norm_b;
    if (outer == 0) hist_push(res, rel0);
    if (rel0 <= tol) { res->converged = 1; break; }
    memset(g, 0, sizeof(double) * ld);
    g[0] = beta;
    for (size_t q = 0; q < n; ++q) z[q] *= 1.0 / beta;
    memcpy(v[0], z, n * sizeof(double));
    int spanned = 0, done = 0;
    for (int i = 0; i < rst && !done; ++i) {
      sop_apply(a, v[i], t);
      pc_apply(m, t, w);
      const double norm0 = nrm2(n, w);
      for (int k = 0; k <= i; ++k) {
        const double hk = dot(n, v[k], w);
        for (size_t q = 0; q < n; ++q) w[q] += -hk * v[k][q];
        h[i * ld + k] = hk;
      }
      if (nrm2(n, w) < 1e-8 * norm0) {
        for (int k = 0; k <= i; ++k) {
          const double c = dot(n, v[k], w);
          for (size_t q = 0; q < n; ++q) w[q] += -c * v[k][q];
          h[i * ld + k] += c;
        }
      }
      const double hip = nrm2(n, w);
      const int happy = hip <= 1e-14 * (norm0 > 0.0 ? norm0 : 1.0);
      for (int k = 0; k + 1 <= i; ++k) {
        const double tmp = cs[k] * h[i * ld + k] + sn[k] * h[i * ld + k + 1];
        h[i * ld + k + 1] = -sn[k] * h[i * ld + k] + cs[k] * h[i * ld + k + 1];
        h[i * ld + k] = tmp;
      }
      const double denom = hypot(h[i * ld + i], hip);
      cs[i] = denom > 0.0 ? h[i * ld + i] / denom : 1.0;
      sn[i] = denom > 0.0 ? hip / denom : 0.0;
      h[i * ld + i] = denom;
      g[i + 1] = -sn[i] * g[i];
      g[i] = cs[i] * g[i];
      ++res->iterations;
      spanned = i + 1;
      const double est = fabs(g[i + 1]) / norm_b;
      hist_push(res, est);
      if (!happy) {
        memcpy(v[i + 1], w, n * sizeof(double));
        for (size_t q = 0; q < n; ++q) v[i + 1][q] *= 1.0 / hip;
      }
      if (est <= tol || happy) { /* verify the estimate, krylov.cpp:132-149 */
        back_sub(h, ld, g, spanned, y);
        memcpy(trial, x, n * sizeof(double));
        for (int k = 0; k < spanned; ++k)
          for (size_t q = 0; q < n; ++q) trial[q] += y[k] * v[k][q];
        double* sw = res->x; res->x = trial; trial = sw; x = res->x;
        if (true_rel(a, m, b, x, t, r, z, norm_b) <= tol) { res->converged = 1; done = 1; }
        else if (happy) { done = 1; }
        else { sw = res->x; res->x = trial; trial = sw; x = res->x; }
      }
    }
    if (!res->converged && !done) {
      back_sub(h, ld, g, spanned, y);
      for (int k = 0; k < spanned; ++k)
        for (size_t q = 0; q < n; ++q) x[q] += y[k] * v[k][q];
    }
  }
  const double final_rel = true_rel(a, m, b, x, t, r, z, norm_b);
  if (final_rel <= tol) res->converged = 1;
  if (res->nh == 0) hist_push(res, final_rel);
  else res->hist[res->nh - 1] = final_rel;
  for (int k = 0; k <= rst; ++k) free(v[k]);
  free(v); free(h); free(g); free(cs); free(sn); free(y);
  free(t); free(r); free(z); free(w); free(trial);
  return 0;
}

/* Left-preconditioned BiCGSTAB (van der Vorst 1992) on M^-1 A x = M^-1 b.
 * NOT IN THE REFERENCE (SURVEY.md 8(a')): same zero initial guess, the same
 * stopping quantity ||M^-1 (b - A x)|| / ||M^-1 b|| <= tol as gmres, and the
 * same "verify the recurrence with the true preconditioned residual" rule.
 * One iteration = two operator applies + two preconditioner applies.
 * History: entry 0 = initial residual, one entry per iteration, last entry
 * recomputed from the returned solution (krylov.hpp:25-28 convention). */
static int bicgstab(const sop* a, const pcond* m, double tol, int max_it, const double* b,
                    kres* res) {
  const size_t n = sop_size(a);
  if (max_it <= 0 || !(tol > 0.0)) return fail("invalid solver configuration");
  memset(res, 0, sizeof *res);
  res->x = NEWD(n);
  double* x = res->x;
  double *r = NEWD(n), *rh = NEWD(n), *p = NEWD(n), *v = NEWD(n), *s = NEWD(n), *t = NEWD(n),
         *tmp = NEWD(n), *tmp2 = NEWD(n);
  pc_apply(m, b, r); /* r = M^-1 (b - A 0) */
  const double norm_b = nrm2(n, r);
  if (norm_b == 0.0) {
    res->converged = 1;
    hist_push(res, 0.0);
    goto out;
  }
  memcpy(rh, r, n * sizeof(double));
  hist_push(res, 1.0);
  double rho = 1.0, alpha = 1.0, omg = 1.0;
  for (int it = 0; it < max_it; ++it) {
    const double rho_new = dot(n, rh, r);
    if (rho_new == 0.0) break; /* breakdown: stop, final check below */
    if (it == 0) {
      memcpy(p, r, n * sizeof(double));
    } else {
      const double beta = (rho_new / rho) * (alpha / omg);
      for (size_t q = 0; q < n; ++q) p[q] = r[q] + beta * (p[q] - omg * v[q]);
    }
    sop_apply(a, p, tmp);
    pc_apply(m, tmp, v);
    const double rv = dot(n, rh, v);
    if (rv == 0.0) break;
    alpha = rho_new / rv;
    for (size_t q = 0; q < n; ++q) s[q] = r[q] - alpha * v[q];
    ++res->iterations;
    const double srel = nrm2(n, s) / norm_b;
    if (srel <= tol) { /* half-step estimate: verify x + alpha p before accepting */
      double* trial = NEWD(n);
      for (size_t q = 0; q < n; ++q) trial[q] = x[q] + alpha * p[q];
      sop_apply(a, trial, tmp);
      for (size_t q = 0; q < n; ++q) tmp2[q] = b[q] - tmp[q];
      pc_apply(m, tmp2, t);
      const double trel = nrm2(n, t) / norm_b;
      if (trel <= tol) {
        memcpy(x, trial, n * sizeof(double));
        free(trial);
        hist_push(res, trel);
        res->converged = 1;
        break;
      }
      free(trial); /* estimate lied: finish the full step */
    }
    sop_apply(a, s, tmp);
    pc_apply(m, tmp, t);
    const double tt = dot(n, t, t);
    omg = tt > 0.0 ? dot(n, t, s) / tt : 0.0;
    for (size_t q = 0; q < n; ++q) x[q] += alpha * p[q] + omg * s[q];
    for (size_t q = 0; q < n; ++q) r[q] = s[q] - omg * t[q];
    rho = rho_new;
    const double rel = nrm2(n, r) / norm_b;
    hist_push(res, rel);
    if (rel <= tol) { /* verify; the recurrence residual r is kept either way */
      sop_apply(a, x, tmp);
      for (size_t q = 0; q < n; ++q) tmp2[q] = b[q] - tmp[q];
      pc_apply(m, tmp2, t);
      if (nrm2(n, t) / norm_b <= tol) { res->converged = 1; break; }
    }
    if (omg == 0.0) break;
  }
  {
    sop_apply(a, x, tmp);
    for (size_t q = 0; q < n; ++q) tmp2[q] = b[q] - tmp[q];
    pc_apply(m, tmp2, r);
    const double final_rel = nrm2(n, r) / norm_b;
    if (final_rel <= tol) res->converged = 1;
    res->hist[res->nh - 1] = final_rel;
  }
out:
  free(r); free(rh); free(p); free(v); free(s); free(t); free(tmp); free(tmp2);
  return 0;
}

/* ---------------- extern "C" entry points (mirror oracle/ref_harness.cpp) - */
#define SETUP(s, p) prob p; if (setup(s, &p)) return 1

int orc_grid(const orc_spec* s, double* out) {
  SETUP(s, p);
  out[0] = p.hx; out[1] = p.hy; out[2] = p.dt; out[3] = p.inv_r; out[4] = p.s_over_r;
  return 0;
}
int orc_coefficients(const orc_spec* s, double* dp, double* dm, double* ep, double* em) {
  SETUP(s, p);
  for (int j = 0; j < p.n2; ++j)
    for (int i = 0; i < p.n1; ++i) {
      const size_t q = i + (size_t)j * p.n1;
      coeffs_at(&p, gx(&p, i), gy(&p, j), dp + q, dm + q, ep + q, em + q);
    }
  return 0;
}
int orc_op_apply(const orc_spec* s, int sign, const double* x, double* y) {
  SETUP(s, p);
  sop o;
  if (assemble(&p, &o)) return 1;
  sop_apply_impl(&o, x, y, sign >= 0 ? 1.0 : -1.0);
  sop_free(&o);
  return 0;
}
int orc_op_diagonal(const orc_spec* s, double* d) {
  SETUP(s, p);
  sop o;
  if (assemble(&p, &o)) return 1;
  memcpy(d, o.diag, sop_size(&o) * sizeof(double));
  sop_free(&o);
  return 0;
}
int orc_plan(const orc_spec* s, int* dims, int max_levels, double* ratio0) {
  SETUP(s, p);
  sop o;
  if (assemble(&p, &o)) return -1;
  const double r = aniso(&o, p.alpha, p.beta);
  sop_free(&o);
  if (ratio0) *ratio0 = r;
  return plan(p.n1, p.n2, r, p.alpha, p.beta, dims, max_levels);
}
int orc_vcycle(const orc_spec* s, const double* b, double* x) {
  SETUP(s, p);
  hier h;
  int rc = s->precond == 1 ? hier_p2(&p, s->omega, &h)
                           : hier_geometric(&p, 1, s->omega, s->coarse, s->coarse_sweeps, &h);
  if (rc) return 1;
  vcycle(&h, b, x);
  hier_free(&h);
  return 0;
}
int orc_precond_apply(const orc_spec* s, const double* r, double* z) {
  SETUP(s, p);
  pcond pc;
  if (pc_make(s, &p, &pc)) return 1;
  pc_apply(&pc, r, z);
  pc_free(&pc);
  return 0;
}
int orc_initial(const orc_spec* s, double* u) { /* sample_initial, problem.cpp:98-104 */
  SETUP(s, p);
  for (int j = 0; j < p.n2; ++j)
    for (int i = 0; i < p.n1; ++i) {
      const double x = gx(&p, i), y = gy(&p, j);
      u[i + (size_t)j * p.n1] = x * x * (1.0 - x) * (1.0 - x) * y * y * (1.0 - y) * (1.0 - y);
    }
  return 0;
}
int orc_source(const orc_spec* s, int m, double* v) {
  SETUP(s, p);
  for (int j = 0; j < p.n2; ++j)
    for (int i = 0; i < p.n1; ++i) v[i + (size_t)j * p.n1] = source_at(&p, m, j, i);
  return 0;
}
/* assemble_rhs, problem.cpp:73-89 */
static void rhs(const prob* p, const sop* o, int m, const double* u, double* b) {
  sop_apply_impl(o, u, b, -1.0);
  const double sc = 2.0 * pow(p->hx, p->alpha);
  for (int j = 0; j < p->n2; ++j)
    for (int i = 0; i < p->n1; ++i) b[i + (size_t)j * p->n1] += sc * source_at(p, m, j, i);
}
int orc_rhs(const orc_spec* s, int m, const double* u_prev, double* b) {
  SETUP(s, p);
  if (m <= 0) return fail("step index starts at 1");
  sop o;
  if (assemble(&p, &o)) return 1;
  rhs(&p, &o, m, u_prev, b);
  sop_free(&o);
  return 0;
}
static int solve_once(const orc_spec* s, int solver, const double* b, double* x, int* iterations,
                      int* converged, double* history, int max_history, int* n_history) {
  SETUP(s, p);
  sop o;
  if (assemble(&p, &o)) return 1;
  pcond pc;
  if (pc_make(s, &p, &pc)) return 1;
  kres r;
  const int rc = solver == 0 ? gmres(&o, &pc, s->tol, s->restart, s->max_outer, b, &r)
                             : bicgstab(&o, &pc, s->tol, s->max_outer * s->restart, b, &r);
  if (!rc) {
    memcpy(x, r.x, sop_size(&o) * sizeof(double));
    *iterations = r.iterations;
    *converged = r.converged;
    *n_history = r.nh;
    for (int k = 0; k < r.nh && k < max_history; ++k) history[k] = r.hist[k];
    free(r.x); free(r.hist);
  }
  pc_free(&pc);
  sop_free(&o);
  return rc;
}
int orc_gmres(const orc_spec* s, const double* b, double* x, int* iterations, int* converged,
              double* history, int max_history, int* n_history) {
  return solve_once(s, 0, b, x, iterations, converged, history, max_history, n_history);
}
int orc_bicgstab(const orc_spec* s, const double* b, double* x, int* iterations, int* converged,
                 double* history, int max_history, int* n_history) {
  return solve_once(s, 1, b, x, iterations, converged, history, max_history, n_history);
}
/* time_march step loop (driver.cpp:20-52), recording every u^m */
int orc_march(const orc_spec* s, int solver, double* u_out, int* its, double* res,
              double* u_steps, double* wall) {
  SETUP(s, p);
  const double t0 = now_s();
  const size_t n = (size_t)p.n1 * p.n2;
  double *u = NEWD(n), *b = NEWD(n);
  orc_initial(s, u);
  sop o;
  if (assemble(&p, &o)) return 1;
  pcond pc;
  if (pc_make(s, &p, &pc)) return 1;
  for (int m = 1; m <= p.steps; ++m) {
    rhs(&p, &o, m, u, b);
    kres r;
    const int rc = solver == 0 ? gmres(&o, &pc, s->tol, s->restart, s->max_outer, b, &r)
                               : bicgstab(&o, &pc, s->tol, s->max_outer * s->restart, b, &r);
    if (rc) return 1;
    its[m - 1] = r.iterations;
    res[m - 1] = r.hist[r.nh - 1];
    memcpy(u, r.x, n * sizeof(double));
    free(r.x); free(r.hist);
    if (u_steps) memcpy(u_steps + (size_t)(m - 1) * n, u, n * sizeof(double));
  }
  memcpy(u_out, u, n * sizeof(double));
  if (wall) *wall = now_s() - t0;
  pc_free(&pc);
  sop_free(&o);
  free(u); free(b);
  return 0;
}
int orc_time_apply(const orc_spec* s, int reps, double* sec) {
  SETUP(s, p);
  sop o;
  if (assemble(&p, &o)) return 1;
  const size_t n = sop_size(&o);
  double *x = NEWD(n), *y = NEWD(n);
  for (size_t k = 0; k < n; ++k) x[k] = 2.0 * u01(k) - 1.0;
  for (int r = 0; r < reps; ++r) {
    const double t0 = now_s();
    sop_apply(&o, x, y);
    sec[r] = now_s() - t0;
  }
  free(x); free(y);
  sop_free(&o);
  return 0;
}
int orc_time_vcycle(const orc_spec* s, int reps, double* sec) {
  SETUP(s, p);
  hier h;
  if (hier_geometric(&p, 1, s->omega, s->coarse, s->coarse_sweeps, &h)) return 1;
  const size_t n = h.size[0];
  double *b = NEWD(n), *x = NEWD(n);
  for (size_t k = 0; k < n; ++k) b[k] = 2.0 * u01(k) - 1.0;
  for (int r = 0; r < reps; ++r) {
    memset(x, 0, n * sizeof(double));
    const double t0 = now_s();
    vcycle(&h, b, x);
    sec[r] = now_s() - t0;
  }
  free(b); free(x);
  hier_free(&h);
  return 0;
}
