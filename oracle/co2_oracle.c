/*
 * co2_oracle.c -- CPU restatement of the reference CO2 outer-step path.
 * TEST INFRASTRUCTURE ONLY (see co2_oracle.h).  Compiled with
 * -ffp-contract=off and without -ffast-math, matching the reference's build
 * (proj/CMakeLists.txt:12-13), so every op below is exactly one IEEE op.
 */
#include "co2_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG */
/* RngStream (proj/include/co2sim/rng.hpp:12-54).  The reference keeps a
 * counter that is pre-incremented before each draw, so draw j (0-based)
 * uses counter j+1. */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;

uint64_t orc_mix(uint64_t z) { /* rng.hpp:45-49 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_rng_key(uint64_t seed, uint64_t stream) { /* rng.hpp:14-15 */
  return orc_mix(orc_mix(seed + kGolden) ^ stream);
}

uint64_t orc_rng_u64_at(uint64_t key, uint64_t j) { /* rng.hpp:17-20 */
  return orc_mix(key + (j + 1) * kGolden);
}

double orc_rng_double_at(uint64_t key, uint64_t j) { /* rng.hpp:22-25 */
  return (double)(orc_rng_u64_at(key, j) >> 11) * 0x1.0p-53;
}

uint64_t orc_rng_below_at(uint64_t key, uint64_t j, uint64_t n) { /* rng.hpp:30-33 */
  return (uint64_t)(((unsigned __int128)orc_rng_u64_at(key, j) * n) >> 64);
}

void orc_rng_fill_u64(uint64_t seed, uint64_t stream, int64_t count, uint64_t* out) {
  uint64_t key = orc_rng_key(seed, stream);
  for (int64_t j = 0; j < count; ++j) out[j] = orc_rng_u64_at(key, (uint64_t)j);
}

/* ----------------------------------------------------------------- bf16 */
uint16_t orc_f32_to_bf16(float f) { /* round to nearest even; NaN -> 0x7fff */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* ------------------------------------------------------------ param_ops */
int orc_ensure_finite_f64(int64_t n, const double* v, const char* context) {
  /* param_ops.cpp:10-14 (Eigen allFinite) */
  for (int64_t j = 0; j < n; ++j) {
    if (!isfinite(v[j])) {
      char buf[200];
      snprintf(buf, sizeof buf, "non-finite value in %s", context);
      return fail(ORC_NUMERIC, buf);
    }
  }
  return ORC_OK;
}

int orc_average_f64(int g, const double* const* c, int64_t n, double* out) {
  /* param_ops.cpp:16-33: sum = c0; sum += c_i ascending; result = sum / G */
  if (g <= 0) return fail(ORC_VALIDATION, "average: empty contribution list");
  for (int64_t j = 0; j < n; ++j) out[j] = c[0][j];
  for (int i = 1; i < g; ++i)
    for (int64_t j = 0; j < n; ++j) out[j] += c[i][j];
  double gd = (double)g;
  for (int64_t j = 0; j < n; ++j) out[j] = out[j] / gd;
  return orc_ensure_finite_f64(n, out, "average");
}

static inline double max_std(double a, double b) { return (a < b) ? b : a; } /* std::max */
static inline double min_std(double a, double b) { return (b < a) ? b : a; } /* std::min */
static inline float max_stdf(float a, float b) { return (a < b) ? b : a; }
static inline float min_stdf(float a, float b) { return (b < a) ? b : a; }

int orc_clip_f64(int64_t n, const double* v, double phi, double* out) {
  /* param_ops.cpp:35-43 */
  if (!(phi > 0.0)) return fail(ORC_VALIDATION, "clip_elementwise: phi must be positive");
  int s = orc_ensure_finite_f64(n, v, "clip_elementwise input");
  if (s) return s;
  for (int64_t j = 0; j < n; ++j) out[j] = min_std(max_std(v[j], -phi), phi);
  return ORC_OK;
}

/* ------------------------------------------------------------ outer ops */
int orc_hyper_validate(const orc_hyper* h) { /* outer_algorithms.cpp:37-46 */
  if (!(h->alpha > 0.0)) return fail(ORC_VALIDATION, "hyper: alpha must be positive");
  if (h->beta < 0.0 || h->beta >= 1.0)
    return fail(ORC_VALIDATION, "hyper: beta must lie in [0, 1)");
  if (!(h->phi > 0.0)) return fail(ORC_VALIDATION, "hyper: phi must be positive");
  if (!(h->epsilon > 0.0)) return fail(ORC_VALIDATION, "hyper: epsilon must be positive");
  return ORC_OK;
}

/* outer_algorithms.cpp:48-64.  One pass per Eigen expression, each into a
 * fresh temporary, as the reference evaluates them. */
static int gap_f64_range(int64_t n, const double* x_t0, const double* p0, const double* p1,
                         int tau, double eps, double* gap) {
  double* numer = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double* denom = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double td = (double)tau;
  for (int64_t j = 0; j < n; ++j) numer[j] = fabs(x_t0[j] - p0[j]);
  for (int64_t j = 0; j < n; ++j) denom[j] = max_std(fabs(td * (p1[j] - p0[j])), eps);
  for (int64_t j = 0; j < n; ++j) gap[j] = numer[j] / denom[j] + 1.0;
  free(numer);
  free(denom);
  return orc_ensure_finite_f64(n, gap, "staleness_gap");
}

/* staleness_gap, proj/src/outer_algorithms.cpp:48-64 */
int orc_staleness_gap_f64(int64_t n, const double* x_t0, const double* p0,
                          const double* p1, int tau, double epsilon, double* gap) {
  if (tau < 1) return fail(ORC_VALIDATION, "staleness_gap: tau must be >= 1");
  if (!(epsilon > 0.0)) return fail(ORC_VALIDATION, "staleness_gap: epsilon must be positive");
  return gap_f64_range(n, x_t0, p0, p1, tau, epsilon, gap);
}

static int momentum_f64_range(int64_t n, const double* m_prev, double beta, const double* gap,
                              const double* delta, int penalty, double* m) {
  if (penalty) { /* outer_algorithms.cpp:78-84 */
    for (int64_t j = 0; j < n; ++j)
      if (gap[j] < 1.0) return fail(ORC_VALIDATION, "momentum update: gap coordinate below 1");
    for (int64_t j = 0; j < n; ++j) m[j] = beta * m_prev[j] + delta[j] / gap[j];
  } else {
    for (int64_t j = 0; j < n; ++j) m[j] = beta * m_prev[j] + delta[j];
  }
  return orc_ensure_finite_f64(n, m, "momentum update");
}

/* penalized_momentum_update, proj/src/outer_algorithms.cpp:66-90 */
int orc_penalized_momentum_f64(int64_t n, const double* m_prev, double beta,
                               const double* gap, const double* delta, int penalty,
                               double* m) {
  if (beta < 0.0 || beta >= 1.0)
    return fail(ORC_VALIDATION, "momentum update: beta must lie in [0, 1)");
  return momentum_f64_range(n, m_prev, beta, gap, delta, penalty, m);
}

static int iterate_f64_range(int64_t n, const double* x_t0, double alpha, const double* m,
                             double phi, int clip, double* x) {
  if (clip) { /* outer_algorithms.cpp:101-102 */
    double* c = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    int s = orc_clip_f64(n, m, phi, c);
    if (s) {
      free(c);
      return s;
    }
    for (int64_t j = 0; j < n; ++j) x[j] = x_t0[j] - alpha * c[j];
    free(c);
  } else {
    for (int64_t j = 0; j < n; ++j) x[j] = x_t0[j] - alpha * m[j];
  }
  return orc_ensure_finite_f64(n, x, "outer_iterate");
}

/* outer_iterate, proj/src/outer_algorithms.cpp:92-108 (clip through
 * clip_elementwise, proj/src/param_ops.cpp:35-43) */
int orc_outer_iterate_f64(int64_t n, const double* x_t0, double alpha, const double* m,
                          double phi, int clip, double* x) {
  if (!(alpha > 0.0)) return fail(ORC_VALIDATION, "outer_iterate: alpha must be positive");
  return iterate_f64_range(n, x_t0, alpha, m, phi, clip, x);
}

/* ------------------------------------------- co2_round per-worker body */
typedef struct {
  int64_t n;
  const double *x_t0, *p0, *p1, *avg;
  const double* m_prev;
  const orc_hyper* h;
  double *m_out, *next, *gap_out;
  double min_gap, max_step;
  int status;
  int stage; /* 0 ok, 1 gap, 2 momentum, 3 iterate */
  char err[256];
} step_job;

static void* step_range(void* arg) {
  /* outer_algorithms.cpp:186-196 for one contiguous coordinate range */
  step_job* jb = (step_job*)arg;
  int64_t n = jb->n;
  const orc_hyper* h = jb->h;
  double* gap = jb->gap_out;
  int s = gap_f64_range(n, jb->x_t0, jb->p0, jb->p1, h->tau, h->epsilon, gap);
  if (s) {
    jb->status = s;
    jb->stage = 1;
    snprintf(jb->err, sizeof jb->err, "%s", g_err);
    return NULL;
  }
  double* delta = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1)); /* cpp:189 */
  for (int64_t j = 0; j < n; ++j) delta[j] = jb->p0[j] - jb->avg[j];
  s = momentum_f64_range(n, jb->m_prev, h->beta, gap, delta, h->penalty, jb->m_out);
  free(delta);
  if (s) {
    jb->status = s;
    jb->stage = 2;
    snprintf(jb->err, sizeof jb->err, "%s", g_err);
    return NULL;
  }
  s = iterate_f64_range(n, jb->x_t0, h->alpha, jb->m_out, h->phi, h->clip, jb->next);
  if (s) {
    jb->status = s;
    jb->stage = 3;
    snprintf(jb->err, sizeof jb->err, "%s", g_err);
    return NULL;
  }
  double mg = INFINITY, ms = 0.0; /* cpp:194-196 */
  for (int64_t j = 0; j < n; ++j) mg = gap[j] < mg ? gap[j] : mg;
  for (int64_t j = 0; j < n; ++j) {
    double d = fabs(jb->next[j] - jb->x_t0[j]);
    ms = d > ms ? d : ms;
  }
  jb->min_gap = mg;
  jb->max_step = ms;
  jb->status = ORC_OK;
  jb->stage = 0;
  return NULL;
}

/* co2_round's per-worker body, proj/src/outer_algorithms.cpp:186-202, with
 * the reference's unfused passes and temporaries */
int orc_worker_step_f64(int64_t n, const double* x_t0, const double* p0, const double* p1,
                        const double* avg, double* m_inout, const orc_hyper* h, double* next,
                        double* gap_out, double* min_gap, double* max_step, int threads) {
  int s = orc_hyper_validate(h);
  if (s) return s;
  if (h->tau < 1) return fail(ORC_VALIDATION, "staleness_gap: tau must be >= 1");
  if (threads < 1) threads = 1;
  if ((int64_t)threads > n) threads = n > 0 ? (int)n : 1;
  /* The reference allocates fresh gap and m vectors and moves them into the
   * worker's outer state (cpp:197-198); mirror that with fresh buffers. */
  double* gap = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double* m_new = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  step_job* jobs = (step_job*)calloc((size_t)threads, sizeof(step_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    int64_t a = (int64_t)t * chunk, b = a + chunk;
    if (a > n) a = n;
    if (b > n) b = n;
    step_job* jb = &jobs[t];
    jb->n = b - a;
    jb->x_t0 = x_t0 + a;
    jb->p0 = p0 + a;
    jb->p1 = p1 + a;
    jb->avg = avg + a;
    jb->m_prev = m_inout + a;
    jb->h = h;
    jb->m_out = m_new + a;
    jb->next = next + a;
    jb->gap_out = gap + a;
    if (threads > 1)
      pthread_create(&tids[t], NULL, step_range, jb);
    else
      step_range(jb);
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  /* Error precedence = the earliest failing stage over all coordinates,
   * which is what the reference's whole-vector passes report. */
  int best = 0, stage = 99;
  double mg = INFINITY, ms = 0.0;
  for (int t = 0; t < threads; ++t) {
    if (jobs[t].status && jobs[t].stage < stage) {
      stage = jobs[t].stage;
      best = t;
    }
    if (jobs[t].min_gap < mg) mg = jobs[t].min_gap;
    if (jobs[t].max_step > ms) ms = jobs[t].max_step;
  }
  int status = ORC_OK;
  if (stage != 99) {
    status = jobs[best].status;
    snprintf(g_err, sizeof g_err, "%s", jobs[best].err);
  } else {
    memcpy(m_inout, m_new, sizeof(double) * (size_t)n);
    if (gap_out) memcpy(gap_out, gap, sizeof(double) * (size_t)n);
    if (min_gap) *min_gap = n ? mg : INFINITY;
    if (max_step) *max_step = ms;
  }
  free(jobs);
  free(tids);
  free(gap);
  free(m_new);
  return status;
}

/* ----------------------------------------------- fused same-order step */
/* SURVEY.md 8(a) "Fused per-element semantics": the composition of the
 * reference's element-wise passes for one coordinate, no FMA:
 *   n0 = |x_t0 - p0|; d = max(|tau*(p1 - p0)|, eps); L = n0/d + 1
 *   D = p0 - xbar; m' = beta*m + D/L  (or beta*m + D)
 *   c = min(max(m', -phi), phi)       (or m');  x' = x_t0 - alpha*c
 * q0s is the point the inner loop started from: q0 itself in fp64 / fp32, and
 * bf16(q0) in bf16-mixed, where the inner loop runs on the bf16 rounding of
 * the fp32 anchor (the GPU's start_of_inner, csrc/outer_step.cu). */
#define FUSED_BODY(T, ABS, ISFIN, MAXF, MINF)                                      \
  T n0 = ABS(x - q0);                                                              \
  T a = ABS(tf * (q1 - q0s));                                                      \
  int floored = a < epsf;                                                          \
  T d = MAXF(a, epsf);                                                             \
  T lam = n0 / d + (T)1;                                                           \
  T dl = q0 - xb;                                                                  \
  T mn = h->penalty ? (betaf * mo + dl / lam) : (betaf * mo + dl);                 \
  T c = mn;                                                                        \
  int clipped = 0;                                                                 \
  if (h->clip) {                                                                   \
    clipped = (mn < -phif) || (phif < mn);                                         \
    c = MINF(MAXF(mn, -phif), phif);                                               \
  }                                                                                \
  T xn = x - alphaf * c;                                                           \
  if (!ISFIN(lam)) flags |= ORC_FLAG_GAP_NONFINITE;                                \
  if (h->penalty && lam < (T)1) flags |= ORC_FLAG_GAP_BELOW_ONE;                   \
  if (!ISFIN(mn)) flags |= ORC_FLAG_M_NONFINITE;                                   \
  if (!ISFIN(xn)) flags |= ORC_FLAG_X_NONFINITE;                                   \
  n_floored += floored;                                                            \
  n_clipped += clipped;                                                            \
  if (lam < min_gap) min_gap = (double)lam;                                        \
  {                                                                                \
    T st = ABS(xn - x);                                                            \
    if (st > max_step) max_step = (double)st;                                      \
  }

/* The fused same-op-order restatement of proj/src/outer_algorithms.cpp:
 * 186-196 (SURVEY.md 8a "Fused per-element semantics") in the GPU's storage
 * and compute types */
int orc_outer_step(int mode, int64_t n, const void* x_t0v, const void* p0v, const void* p1v,
                   const void* xbarv, int divisor, void* mv, void* anchorv, void* paramsv,
                   void* gapv, const orc_hyper* h, orc_diag* diag) {
  int s = orc_hyper_validate(h);
  if (s) return s;
  if (h->tau < 1) return fail(ORC_VALIDATION, "staleness_gap: tau must be >= 1");
  if (divisor < 1) return fail(ORC_VALIDATION, "outer step: divisor must be >= 1");
  uint32_t flags = 0;
  int64_t n_floored = 0, n_clipped = 0;
  double min_gap = INFINITY, max_step = 0.0;
  if (mode == ORC_MODE_F64) {
    const double *X = x_t0v, *P0 = p0v, *P1 = p1v, *XB = xbarv;
    double *M = mv, *A = anchorv, *PR = paramsv, *G = gapv;
    double tf = (double)h->tau, epsf = h->epsilon, betaf = h->beta, phif = h->phi,
           alphaf = h->alpha, gd = (double)divisor;
    for (int64_t j = 0; j < n; ++j) {
      double x = X[j], q0 = P0[j], q1 = P1[j], mo = M[j];
      double q0s = q0;
      double xb = divisor > 1 ? XB[j] / gd : XB[j];
      FUSED_BODY(double, fabs, isfinite, max_std, min_std)
      M[j] = mn;
      if (A) A[j] = xn;
      if (PR) PR[j] = xn;
      if (G) G[j] = lam;
    }
  } else if (mode == ORC_MODE_F32 || mode == ORC_MODE_BF16_MIXED) {
    int bf = mode == ORC_MODE_BF16_MIXED;
    const float *X = x_t0v, *P0 = p0v;
    float *M = mv, *A = anchorv, *G = gapv;
    float tf = (float)h->tau, epsf = (float)h->epsilon, betaf = (float)h->beta,
          phif = (float)h->phi, alphaf = (float)h->alpha, gd = (float)divisor;
    for (int64_t j = 0; j < n; ++j) {
      float x = X[j], q0 = P0[j], mo = M[j];
      float q1 = bf ? orc_bf16_to_f32(((const uint16_t*)p1v)[j]) : ((const float*)p1v)[j];
      float xb = bf ? orc_bf16_to_f32(((const uint16_t*)xbarv)[j]) : ((const float*)xbarv)[j];
      if (divisor > 1) xb = xb / gd;
      float q0s = bf ? orc_bf16_to_f32(orc_f32_to_bf16(q0)) : q0;
      FUSED_BODY(float, fabsf, isfinite, max_stdf, min_stdf)
      M[j] = mn;
      if (A) A[j] = xn;
      if (paramsv) {
        if (bf)
          ((uint16_t*)paramsv)[j] = orc_f32_to_bf16(xn);
        else
          ((float*)paramsv)[j] = xn;
      }
      if (G) G[j] = lam;
    }
  } else {
    return fail(ORC_VALIDATION, "outer step: unknown mode");
  }
  diag->min_gap = min_gap;
  diag->max_outer_step = max_step;
  diag->n_clipped = n_clipped;
  diag->n_floored = n_floored;
  diag->flags = flags;
  diag->pad = 0;
  return orc_diag_status(diag);
}

/* Ghost-consistent / sharded step (outer_algorithms.cpp:161-184) in the
 * same op order as the GPU: x_t0 = average of `ghost` identical anchors (or
 * xbar itself when ghost == 0), prev_x1 = p1sum / p1_div, xbar = xsum / xdiv;
 * bar0_out receives the x_t0 used.  Storage as orc_outer_step. */
int orc_outer_step_ghost(int mode, int64_t n, const void* anchorv, const void* p0v,
                         const void* p1v, int p1_div, const void* xsumv, int xdiv, int ghost,
                         void* mv, void* anchor_out, void* bar0_out, void* paramsv, void* gapv,
                         const orc_hyper* h, orc_diag* diag) {
  int s = orc_hyper_validate(h);
  if (s) return s;
  uint32_t flags = 0;
  int64_t n_floored = 0, n_clipped = 0;
  double min_gap = INFINITY, max_step = 0.0;
  if (mode == ORC_MODE_F64) {
    const double *AN = anchorv, *P0 = p0v, *P1 = p1v, *XS = xsumv;
    double *M = mv, *A = anchor_out, *B0 = bar0_out, *PR = paramsv, *G = gapv;
    double tf = (double)h->tau, epsf = h->epsilon, betaf = h->beta, phif = h->phi,
           alphaf = h->alpha;
    for (int64_t j = 0; j < n; ++j) {
      double xb = XS[j];
      if (xdiv > 1) xb = xb / (double)xdiv;
      double x;
      if (ghost == 0) {
        x = xb;
      } else {
        double sum = AN[j];
        for (int i = 1; i < ghost; ++i) sum = sum + AN[j];
        x = sum / (double)ghost;
      }
      double q0 = P0[j], q1 = P1[j], mo = M[j];
      double q0s = q0;
      if (p1_div > 1) q1 = q1 / (double)p1_div;
      FUSED_BODY(double, fabs, isfinite, max_std, min_std)
      M[j] = mn;
      if (B0) B0[j] = x;
      if (A) A[j] = xn;
      if (PR) PR[j] = xn;
      if (G) G[j] = lam;
    }
  } else {
    int bf = mode == ORC_MODE_BF16_MIXED;
    const float *AN = anchorv, *P0 = p0v;
    float *M = mv, *A = anchor_out, *B0 = bar0_out, *G = gapv;
    float tf = (float)h->tau, epsf = (float)h->epsilon, betaf = (float)h->beta,
          phif = (float)h->phi, alphaf = (float)h->alpha;
    for (int64_t j = 0; j < n; ++j) {
      float xb = bf ? orc_bf16_to_f32(((const uint16_t*)xsumv)[j]) : ((const float*)xsumv)[j];
      if (xdiv > 1) xb = xb / (float)xdiv;
      float x;
      if (ghost == 0) {
        x = xb;
      } else {
        float sum = AN[j];
        for (int i = 1; i < ghost; ++i) sum = sum + AN[j];
        x = sum / (float)ghost;
      }
      float q0 = P0[j], mo = M[j];
      float q1 = bf ? orc_bf16_to_f32(((const uint16_t*)p1v)[j]) : ((const float*)p1v)[j];
      if (p1_div > 1) q1 = q1 / (float)p1_div;
      float q0s = bf ? orc_bf16_to_f32(orc_f32_to_bf16(q0)) : q0;
      FUSED_BODY(float, fabsf, isfinite, max_stdf, min_stdf)
      M[j] = mn;
      if (B0) B0[j] = x;
      if (A) A[j] = xn;
      if (paramsv) {
        if (bf)
          ((uint16_t*)paramsv)[j] = orc_f32_to_bf16(xn);
        else
          ((float*)paramsv)[j] = xn;
      }
      if (G) G[j] = lam;
    }
  }
  diag->min_gap = min_gap;
  diag->max_outer_step = max_step;
  diag->n_clipped = n_clipped;
  diag->n_floored = n_floored;
  diag->flags = flags;
  diag->pad = 0;
  return orc_diag_status(diag);
}

int orc_diag_status(const orc_diag* d) {
  /* Reference precedence: staleness_gap numeric (cpp:62) -> gap<1
   * validation (cpp:81-83) -> momentum numeric (cpp:88) -> clip input
   * numeric (param_ops.cpp:41) -> outer_iterate numeric (cpp:106). */
  uint32_t f = d->flags;
  if (f & ORC_FLAG_GAP_NONFINITE) return fail(ORC_NUMERIC, "non-finite value in staleness_gap");
  if (f & ORC_FLAG_GAP_BELOW_ONE)
    return fail(ORC_VALIDATION, "momentum update: gap coordinate below 1");
  if (f & ORC_FLAG_M_NONFINITE) return fail(ORC_NUMERIC, "non-finite value in momentum update");
  if (f & ORC_FLAG_NORM_NONFINITE) return fail(ORC_NUMERIC, "non-finite value in global clip norm");
  if (f & ORC_FLAG_CLIP_NONFINITE)
    return fail(ORC_NUMERIC, "non-finite value in clip_elementwise input");
  if (f & ORC_FLAG_X_NONFINITE) return fail(ORC_NUMERIC, "non-finite value in outer_iterate");
  if (f & ORC_FLAG_SLOWMO_M) return fail(ORC_NUMERIC, "non-finite value in slowmo momentum");
  if (f & ORC_FLAG_SLOWMO_X) return fail(ORC_NUMERIC, "non-finite value in slowmo outer iterate");
  if (f & ORC_FLAG_OVERLAP) return fail(ORC_NUMERIC, "non-finite value in overlap correction");
  return ORC_OK;
}

/* ------------------------------------- global-norm clip (extension) */
#define GC_THREADS 256
#define GC_MAX_CHUNKS 32768

int64_t orc_gc_chunk(int64_t n, int V) {
  const int64_t unit = (int64_t)V * GC_THREADS;
  int64_t c = (n + GC_MAX_CHUNKS - 1) / GC_MAX_CHUNKS;
  c = (c + unit - 1) / unit * unit;
  return c < unit * 16 ? unit * 16 : c;
}

/* 256 per-thread partials -> xor butterfly per warp -> warps in order. */
static double gc_block_sum(double* t) {
  double w[GC_THREADS / 32];
  for (int k = 0; k < GC_THREADS / 32; ++k) {
    double* v = t + 32 * k;
    for (int o = 16; o > 0; o >>= 1) {
      double nv[32];
      for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
      memcpy(v, nv, sizeof nv);
    }
    w[k] = v[0];
  }
  double r = w[0];
  for (int k = 1; k < GC_THREADS / 32; ++k) r = r + w[k];
  return r;
}

int orc_outer_step_global_clip(int mode, int64_t n, const void* x_t0v, const void* p0v,
                               const void* p1v, const void* xbarv, int divisor, void* mv,
                               void* anchorv, void* paramsv, void* gapv, const orc_hyper* h,
                               orc_diag* diag, double* norm_out) {
  int s = orc_hyper_validate(h);
  if (s) return s;
  if (h->tau < 1) return fail(ORC_VALIDATION, "staleness_gap: tau must be >= 1");
  if (divisor < 1) return fail(ORC_VALIDATION, "outer step: divisor must be >= 1");
  if (mode != ORC_MODE_F64 && mode != ORC_MODE_F32 && mode != ORC_MODE_BF16_MIXED)
    return fail(ORC_VALIDATION, "outer step: unknown mode");
  const int V = mode == ORC_MODE_F64 ? 2 : (mode == ORC_MODE_F32 ? 4 : 8);
  const int bf = mode == ORC_MODE_BF16_MIXED;
  uint32_t flags = 0;
  int64_t n_floored = 0, n_clipped = 0;
  double min_gap = INFINITY, max_step = 0.0;
  /* pass 1: m' (in place), gap, and the per-coordinate squares */
  for (int64_t j = 0; j < n; ++j) {
    if (mode == ORC_MODE_F64) {
      const double x = ((const double*)x_t0v)[j], q0 = ((const double*)p0v)[j],
                   q1 = ((const double*)p1v)[j], mo = ((double*)mv)[j];
      double xb = ((const double*)xbarv)[j];
      if (divisor > 1) xb = xb / (double)divisor;
      const double tf = (double)h->tau, epsf = h->epsilon, betaf = h->beta;
      double n0 = fabs(x - q0), a = fabs(tf * (q1 - q0));
      int floored = a < epsf;
      double lam = n0 / max_std(a, epsf) + 1.0;
      double dl = q0 - xb;
      double mn = h->penalty ? (betaf * mo + dl / lam) : (betaf * mo + dl);
      if (!isfinite(lam)) flags |= ORC_FLAG_GAP_NONFINITE;
      if (h->penalty && lam < 1.0) flags |= ORC_FLAG_GAP_BELOW_ONE;
      if (!isfinite(mn)) flags |= ORC_FLAG_M_NONFINITE;
      n_floored += floored;
      if (lam < min_gap) min_gap = lam;
      ((double*)mv)[j] = mn;
      if (gapv) ((double*)gapv)[j] = lam;
    } else {
      const float x = ((const float*)x_t0v)[j], q0 = ((const float*)p0v)[j],
                  mo = ((float*)mv)[j];
      const float q1 = bf ? orc_bf16_to_f32(((const uint16_t*)p1v)[j]) : ((const float*)p1v)[j];
      float xb = bf ? orc_bf16_to_f32(((const uint16_t*)xbarv)[j]) : ((const float*)xbarv)[j];
      if (divisor > 1) xb = xb / (float)divisor;
      const float tf = (float)h->tau, epsf = (float)h->epsilon, betaf = (float)h->beta;
      const float q0s = bf ? orc_bf16_to_f32(orc_f32_to_bf16(q0)) : q0;
      float n0 = fabsf(x - q0), a = fabsf(tf * (q1 - q0s));
      int floored = a < epsf;
      float lam = n0 / max_stdf(a, epsf) + 1.0f;
      float dl = q0 - xb;
      float mn = h->penalty ? (betaf * mo + dl / lam) : (betaf * mo + dl);
      if (!isfinite(lam)) flags |= ORC_FLAG_GAP_NONFINITE;
      if (h->penalty && lam < 1.0f) flags |= ORC_FLAG_GAP_BELOW_ONE;
      if (!isfinite(mn)) flags |= ORC_FLAG_M_NONFINITE;
      n_floored += floored;
      if (lam < min_gap) min_gap = (double)lam;
      ((float*)mv)[j] = mn;
      if (gapv) ((float*)gapv)[j] = lam;
    }
  }
  /* the norm in the GPU's fixed order */
  const int64_t chunk = orc_gc_chunk(n, V);
  const int64_t K = n == 0 ? 0 : (n + chunk - 1) / chunk;
  const int64_t nvE = n / V * V;
  double* cs = K ? malloc(sizeof(double) * (size_t)K) : NULL;
  if (K && !cs) return fail(ORC_VALIDATION, "global clip: out of memory");
  double t[GC_THREADS];
  for (int64_t c = 0; c < K; ++c) {
    const int64_t e0 = c * chunk, e1 = e0 + chunk < nvE ? e0 + chunk : nvE;
    for (int th = 0; th < GC_THREADS; ++th) {
      double acc = 0.0;
      for (int64_t e = e0 + (int64_t)th * V; e < e1; e += (int64_t)GC_THREADS * V)
        for (int v = 0; v < V; ++v) {
          double md = mode == ORC_MODE_F64 ? ((double*)mv)[e + v] : (double)((float*)mv)[e + v];
          acc = acc + md * md;
        }
      if (th == 0 && c == K - 1)
        for (int64_t e = nvE; e < n; ++e) {
          double md = mode == ORC_MODE_F64 ? ((double*)mv)[e] : (double)((float*)mv)[e];
          acc = acc + md * md;
        }
      t[th] = acc;
    }
    cs[c] = gc_block_sum(t);
  }
  for (int th = 0; th < GC_THREADS; ++th) {
    double acc = 0.0;
    for (int64_t i = th; i < K; i += GC_THREADS) acc = acc + cs[i];
    t[th] = acc;
  }
  const double norm = sqrt(gc_block_sum(t));
  free(cs);
  if (!isfinite(norm)) flags |= ORC_FLAG_NORM_NONFINITE;
  const double sc = (h->clip && norm > h->phi) ? h->phi / norm : 1.0;
  /* pass 2: x' = x_t0 - alpha * (m' * scale) */
  for (int64_t j = 0; j < n; ++j) {
    if (mode == ORC_MODE_F64) {
      const double x = ((const double*)x_t0v)[j], m = ((double*)mv)[j];
      const double c = m * sc;
      const double xn = x - h->alpha * c;
      if (!isfinite(xn)) flags |= ORC_FLAG_X_NONFINITE;
      double st = fabs(xn - x);
      if (st > max_step) max_step = st;
      if (anchorv) ((double*)anchorv)[j] = xn;
      if (paramsv) ((double*)paramsv)[j] = xn;
    } else {
      const float x = ((const float*)x_t0v)[j], m = ((float*)mv)[j];
      const float c = (float)((double)m * sc);
      const float xn = x - (float)h->alpha * c;
      if (!isfinite(xn)) flags |= ORC_FLAG_X_NONFINITE;
      float st = fabsf(xn - x);
      if (st > max_step) max_step = (double)st;
      if (anchorv) ((float*)anchorv)[j] = xn;
      if (paramsv) {
        if (bf)
          ((uint16_t*)paramsv)[j] = orc_f32_to_bf16(xn);
        else
          ((float*)paramsv)[j] = xn;
      }
    }
    n_clipped += sc < 1.0;
  }
  diag->min_gap = min_gap;
  diag->max_outer_step = max_step;
  diag->n_clipped = n_clipped;
  diag->n_floored = n_floored;
  diag->flags = flags;
  diag->pad = 0;
  if (norm_out) *norm_out = norm;
  return orc_diag_status(diag);
}

static double ld_any(int dtype, const void* v, int64_t j) {
  if (dtype == 0) return ((const double*)v)[j];
  if (dtype == 1) return (double)((const float*)v)[j];
  return (double)orc_bf16_to_f32(((const uint16_t*)v)[j]);
}

double orc_l2_norm(int dtype, int64_t n, const void* v) {
  const int V = dtype == 0 ? 2 : (dtype == 1 ? 4 : 8);
  const int64_t chunk = orc_gc_chunk(n, V);
  const int64_t K = n == 0 ? 0 : (n + chunk - 1) / chunk;
  const int64_t nvE = n / V * V;
  double* cs = K ? malloc(sizeof(double) * (size_t)K) : NULL;
  if (K && !cs) return NAN;
  double t[GC_THREADS];
  for (int64_t c = 0; c < K; ++c) {
    const int64_t e0 = c * chunk, e1 = e0 + chunk < nvE ? e0 + chunk : nvE;
    for (int th = 0; th < GC_THREADS; ++th) {
      double acc = 0.0;
      for (int64_t e = e0 + (int64_t)th * V; e < e1; e += (int64_t)GC_THREADS * V)
        for (int k = 0; k < V; ++k) {
          const double d = ld_any(dtype, v, e + k);
          acc = acc + d * d;
        }
      if (th == 0 && c == K - 1)
        for (int64_t e = nvE; e < n; ++e) {
          const double d = ld_any(dtype, v, e);
          acc = acc + d * d;
        }
      t[th] = acc;
    }
    cs[c] = gc_block_sum(t);
  }
  for (int th = 0; th < GC_THREADS; ++th) {
    double acc = 0.0;
    for (int64_t i = th; i < K; i += GC_THREADS) acc = acc + cs[i];
    t[th] = acc;
  }
  free(cs);
  return sqrt(gc_block_sum(t));
}

/* ------------------------------------------------ baseline outer steps */
/* Element access in the mode's storage types (see orc_outer_step). */
static double ld_state(int mode, const void* p, int64_t j) {
  return mode == ORC_MODE_F64 ? ((const double*)p)[j] : (double)((const float*)p)[j];
}
static double ld_low(int mode, const void* p, int64_t j) {
  if (mode == ORC_MODE_F64) return ((const double*)p)[j];
  if (mode == ORC_MODE_F32) return ((const float*)p)[j];
  return orc_bf16_to_f32(((const uint16_t*)p)[j]);
}
static void st_state(int mode, void* p, int64_t j, double v) {
  if (mode == ORC_MODE_F64)
    ((double*)p)[j] = v;
  else
    ((float*)p)[j] = (float)v;
}
static void st_low(int mode, void* p, int64_t j, double v) {
  if (mode == ORC_MODE_F64)
    ((double*)p)[j] = v;
  else if (mode == ORC_MODE_F32)
    ((float*)p)[j] = (float)v;
  else
    ((uint16_t*)p)[j] = orc_f32_to_bf16((float)v);
}

static void diag_init(orc_diag* d) {
  d->min_gap = INFINITY;
  d->max_outer_step = 0.0;
  d->n_clipped = d->n_floored = 0;
  d->flags = 0;
  d->pad = 0;
}

/* Arithmetic in the mode's compute type: fp64 for F64, fp32 otherwise (every
 * fp32 op below rounds exactly as the GPU's). */

int orc_slowmo_step(int mode, int64_t n, const void* x_start, const void* xbar, int divisor,
                    void* m, void* params_out, double alpha, double beta, orc_diag* diag) {
  /* slowmo_round, outer_algorithms.cpp:219-236 */
  if (!(alpha > 0.0)) return fail(ORC_VALIDATION, "slowmo: alpha must be positive");
  if (beta < 0.0 || beta >= 1.0) return fail(ORC_VALIDATION, "slowmo: beta must lie in [0, 1)");
  diag_init(diag);
  if (mode == ORC_MODE_F64) {
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double x = ld_state(mode, x_start, j), xb = ld_low(mode, xbar, j);
      if (divisor > 1) xb = xb / (double)divisor;
      double delta = x - xb;
      double mn = beta * ld_state(mode, m, j) + delta;
      double xn = x - alpha * mn;
      if (!isfinite(mn)) diag->flags |= ORC_FLAG_SLOWMO_M;
      if (!isfinite(xn)) diag->flags |= ORC_FLAG_SLOWMO_X;
      st_state(mode, m, j, mn);
      st_low(mode, params_out, j, xn);
      double s = fabs(xn - x);
      if (s > mx) mx = s;
    }
    diag->max_outer_step = mx;
  } else {
    float mx = 0.0f, af = (float)alpha, bf = (float)beta, gd = (float)divisor;
    for (int64_t j = 0; j < n; ++j) {
      float x = (float)ld_state(mode, x_start, j), xb = (float)ld_low(mode, xbar, j);
      if (divisor > 1) xb = xb / gd;
      float delta = x - xb;
      float bm = bf * (float)ld_state(mode, m, j);
      float mn = bm + delta;
      float am = af * mn;
      float xn = x - am;
      if (!isfinite(mn)) diag->flags |= ORC_FLAG_SLOWMO_M;
      if (!isfinite(xn)) diag->flags |= ORC_FLAG_SLOWMO_X;
      st_state(mode, m, j, mn);
      st_low(mode, params_out, j, xn);
      float s = fabsf(xn - x);
      if (s > mx) mx = s;
    }
    diag->max_outer_step = mx;
  }
  return orc_diag_status(diag);
}

int orc_local_sgd_step(int mode, int64_t n, const void* x_start, const void* xbar, int divisor,
                       void* params_out, orc_diag* diag) {
  /* local_sgd_round, outer_algorithms.cpp:251-256 */
  diag_init(diag);
  if (mode == ORC_MODE_F64) {
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double xb = ld_low(mode, xbar, j);
      if (divisor > 1) xb = xb / (double)divisor;
      double s = fabs(xb - ld_state(mode, x_start, j));
      if (s > mx) mx = s;
      st_low(mode, params_out, j, xb);
    }
    diag->max_outer_step = mx;
  } else {
    float mx = 0.0f, gd = (float)divisor;
    for (int64_t j = 0; j < n; ++j) {
      float xb = (float)ld_low(mode, xbar, j);
      if (divisor > 1) xb = xb / gd;
      float s = fabsf(xb - (float)ld_state(mode, x_start, j));
      if (s > mx) mx = s;
      st_low(mode, params_out, j, xb);
    }
    diag->max_outer_step = mx;
  }
  return orc_diag_status(diag);
}

int orc_overlap_correction(int mode, int64_t n, void* params, const void* anchor,
                           const void* xbar, int divisor, orc_diag* diag) {
  /* overlap_local_sgd_round, outer_algorithms.cpp:277-280 / :293-296 */
  diag_init(diag);
  if (mode == ORC_MODE_F64) {
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double xb = ld_low(mode, xbar, j);
      if (divisor > 1) xb = xb / (double)divisor;
      double p = ld_low(mode, params, j);
      double pn = p - (ld_state(mode, anchor, j) - xb);
      if (!isfinite(pn)) diag->flags |= ORC_FLAG_OVERLAP;
      st_low(mode, params, j, pn);
      double s = fabs(pn - p);
      if (s > mx) mx = s;
    }
    diag->max_outer_step = mx;
  } else {
    float mx = 0.0f, gd = (float)divisor;
    for (int64_t j = 0; j < n; ++j) {
      float xb = (float)ld_low(mode, xbar, j);
      if (divisor > 1) xb = xb / gd;
      float p = (float)ld_low(mode, params, j);
      float d = (float)ld_state(mode, anchor, j) - xb;
      float pn = p - d;
      if (!isfinite(pn)) diag->flags |= ORC_FLAG_OVERLAP;
      st_low(mode, params, j, pn);
      /* the step actually stored (bf16 params round pn) */
      float stored = (float)ld_low(mode, params, j);
      float s = fabsf(stored - p);
      if (s > mx) mx = s;
    }
    diag->max_outer_step = mx;
  }
  return orc_diag_status(diag);
}

int orc_average_lp(int bf, int g, const void* const* c, int64_t n, void* out) {
  /* average() (param_ops.cpp:16-33) in fp32 arithmetic: ascending-worker
   * fp32 sum, one fp32 division by G, stored in the params dtype. */
  if (g <= 0) return fail(ORC_VALIDATION, "average: empty contribution list");
  float gf = (float)g;
  int nonfinite = 0;
  for (int64_t j = 0; j < n; ++j) {
    float s = bf ? orc_bf16_to_f32(((const uint16_t*)c[0])[j]) : ((const float*)c[0])[j];
    for (int i = 1; i < g; ++i)
      s += bf ? orc_bf16_to_f32(((const uint16_t*)c[i])[j]) : ((const float*)c[i])[j];
    float r = s / gf;
    if (!isfinite(r)) nonfinite = 1;
    if (bf)
      ((uint16_t*)out)[j] = orc_f32_to_bf16(r);
    else
      ((float*)out)[j] = r;
  }
  if (nonfinite) return fail(ORC_NUMERIC, "non-finite value in average");
  return ORC_OK;
}

/* ----------------------------------------------------- synthetic inputs */
/* counter SplitMix64 uniforms, seed/stream keyed per buffer
 * and worker, mapped to s*(2U-1) in double and rounded once to storage. */
static double sym(uint64_t seed, uint64_t buf, int worker, int64_t j) {
  uint64_t key = orc_rng_key(seed, (buf << 32) | (uint64_t)(uint32_t)worker);
  return 2.0 * orc_rng_double_at(key, (uint64_t)j) - 1.0;
}

static void store_state(int mode, void* p, int64_t i, double v) {
  if (mode == ORC_MODE_F64)
    ((double*)p)[i] = v;
  else
    ((float*)p)[i] = (float)v;
}

static double store_low(int mode, void* p, int64_t i, double v) {
  /* returns the stored value, widened */
  if (mode == ORC_MODE_F64) {
    if (p) ((double*)p)[i] = v;
    return v;
  }
  if (mode == ORC_MODE_F32) {
    float f = (float)v;
    if (p) ((float*)p)[i] = f;
    return f;
  }
  uint16_t b = orc_f32_to_bf16((float)v);
  if (p) ((uint16_t*)p)[i] = b;
  return orc_bf16_to_f32(b);
}

static double round_state(int mode, double v) { return mode == ORC_MODE_F64 ? v : (double)(float)v; }

/* SURVEY.md 8d synthetic inputs on the RngStream generator
 * (proj/include/co2sim/rng.hpp:14-25), random-access form */
void orc_synth(int mode, uint64_t seed, int worker, int64_t j0, int64_t count, void* x_t0,
               void* p0, void* p1, void* x_end, void* m) {
  for (int64_t i = 0; i < count; ++i) {
    int64_t j = j0 + i;
    /* p0 = x_{t-1,0} is drawn from a worker-independent stream; everything
     * else is per worker. */
    double p0v = round_state(mode, 0.02 * sym(seed, ORC_BUF_P0, 0, j));
    int stalled = (j % 61) == 0;
    if (stalled) p0v = store_low(mode, NULL, 0, p0v); /* representable in both dtypes */
    if (p0) store_state(mode, p0, i, p0v);
    if (p1) {
      if (stalled)
        store_low(mode, p1, i, p0v);
      else
        store_low(mode, p1, i, p0v - 1e-3 * sym(seed, ORC_BUF_P1, worker, j));
    }
    if (x_t0) store_state(mode, x_t0, i, p0v + 4e-3 * sym(seed, ORC_BUF_XT0, worker, j));
    if (x_end) store_low(mode, x_end, i, p0v - 4e-3 * sym(seed, ORC_BUF_XEND, worker, j));
    if (m) store_state(mode, m, i, 1e-2 * sym(seed, ORC_BUF_M, worker, j));
  }
}
