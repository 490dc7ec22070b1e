/*
 * halp_oracle.c -- CPU restatement of the reference HALP hot path.
 * TEST INFRASTRUCTURE ONLY (see halp_oracle.h for the contract and the
 * reference file:line map).  Compiled with -ffp-contract=off so that no
 * a*b+c is fused unless written as fma() (MIRROR mode only).
 */
#define _GNU_SOURCE
#include "halp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* oq_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG */
/* rng.hpp:12-18 split_mix */
static uint64_t split_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
/* rng.hpp:29-32 */
void oq_rng_init(oq_rng* r, uint64_t seed, uint64_t stream) {
  r->state = split_mix(seed ^ split_mix(stream ^ 0xA5A5A5A5A5A5A5A5ULL));
  if (r->state == 0) r->state = 0x9E3779B97F4A7C15ULL;
}
/* rng.hpp:34-39 */
uint64_t oq_next_u64(oq_rng* r) {
  uint64_t s = r->state;
  s ^= s >> 12;
  s ^= s << 25;
  s ^= s >> 27;
  r->state = s;
  return s * 0x2545F4914F6CDD1DULL;
}
/* rng.hpp:42-44 */
double oq_next_uniform(oq_rng* r) { return (double)(oq_next_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:48-51 */
uint64_t oq_next_index(oq_rng* r, uint64_t n) {
  unsigned __int128 p = (unsigned __int128)oq_next_u64(r) * (unsigned __int128)n;
  return (uint64_t)(p >> 64);
}
/* rng.hpp:55-60 (std::numbers::pi == M_PI; 2.0 * pi * u2 evaluates left to right) */
double oq_next_normal(oq_rng* r) {
  const double u1 = oq_next_uniform(r);
  const double u2 = oq_next_uniform(r);
  const double rr = sqrt(-2.0 * log1p(-u1));
  return rr * cos(2.0 * M_PI * u2);
}
void oq_fill_u64(uint64_t seed, uint64_t stream, uint64_t skip, uint64_t* out, int64_t count) {
  oq_rng r;
  oq_rng_init(&r, seed, stream);
  for (uint64_t i = 0; i < skip; ++i) (void)oq_next_u64(&r);
  for (int64_t i = 0; i < count; ++i) out[i] = oq_next_u64(&r);
}

/* ------------------------------------------------------------ quantizer */
/* fixed_point.cpp:14-22 */
static int64_t min_code_for(int bits) { return bits == 64 ? INT64_MIN : -((int64_t)1 << (bits - 1)); }
static int64_t max_code_for(int bits) { return bits == 64 ? INT64_MAX : ((int64_t)1 << (bits - 1)) - 1; }

/* fixed_point.cpp:30-50 quantize_code */
int64_t oq_quantize_code(double x, double delta, int bits, double u, int* err) {
  if (!isfinite(x)) { if (err) *err = 1; return 0; }
  const double t = x / delta;
  const double hi = (double)max_code_for(bits);
  const double lo = (double)min_code_for(bits);
  if (t >= hi) return max_code_for(bits);
  if (t <= lo) return min_code_for(bits);
  const double snapped = nearbyint(t);
  if (snapped * delta == x) return (int64_t)snapped;
  const double fl = floor(t);
  const double frac = t - fl;
  int64_t code = (int64_t)fl;
  if (frac > 0.0 && u < frac) ++code;
  return code;
}

/* theory.cpp:33-35 code_span, :93-102 halp_scale */
double oq_halp_scale(double grad_norm, double mu, int bits) {
  if (!(isfinite(grad_norm) && grad_norm >= 0.0)) return -1.0;
  if (!(isfinite(mu) && mu > 0.0)) return -1.0;
  if (bits < 2 || bits > 64) return -1.0;
  const double span = ldexp(1.0, bits - 1) - 1.0;
  return grad_norm / (mu * span);
}

/* ----------------------------------------------------------------- data */
/* objectives.cpp:27-45 make_regression (fill_gaussian_rowwise :17-23) */
int oq_make_regression(int64_t n, int d, double noise_sd, uint64_t seed, double* X, double* y) {
  if (n < 1 || d < 1) { set_err("make_regression: n and d must be positive"); return OQ_INVALID_INPUT; }
  if (!(isfinite(noise_sd) && noise_sd >= 0.0)) {
    set_err("make_regression: noise_sd must be finite and >= 0");
    return OQ_INVALID_INPUT;
  }
  oq_rng rng;
  oq_rng_init(&rng, seed, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) X[i * d + j] = oq_next_normal(&rng);
  double* wt = (double*)malloc(sizeof(double) * (size_t)d);
  for (int j = 0; j < d; ++j) wt[j] = oq_next_normal(&rng);
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc += X[i * d + j] * wt[j];
    y[i] = acc;
  }
  if (noise_sd > 0.0)
    for (int64_t i = 0; i < n; ++i) y[i] += noise_sd * oq_next_normal(&rng);
  free(wt);
  return OQ_OK;
}

static inline double bf16_to_double(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}
/* load row i of X into out[0..d) as doubles (exact upcast) */
static void load_row(const oq_objective* o, int64_t i, double* out) {
  const int d = o->d;
  if (o->dtype == OQ_F64) {
    memcpy(out, (const double*)o->X + i * d, sizeof(double) * (size_t)d);
  } else if (o->dtype == OQ_F32) {
    const float* p = (const float*)o->X + i * d;
    for (int j = 0; j < d; ++j) out[j] = (double)p[j];
  } else {
    const uint16_t* p = (const uint16_t*)o->X + i * d;
    for (int j = 0; j < d; ++j) out[j] = bf16_to_double(p[j]);
  }
}

static int check_objective(const oq_objective* o) {
  if (!(isfinite(o->l2) && o->l2 >= 0.0)) { set_err("Objective: l2 must be finite and >= 0"); return OQ_INVALID_INPUT; }
  if (o->n < 1) { set_err("Objective: dataset is empty"); return OQ_INVALID_INPUT; }
  if (o->loss == OQ_SQUARED) {
    if (!o->y || o->C != 1) { set_err("Objective: squared loss needs one target per row"); return OQ_INVALID_INPUT; }
  } else {
    if (o->C < 2 || !o->labels) { set_err("Objective: softmax loss needs labels and classes"); return OQ_INVALID_INPUT; }
    for (int64_t i = 0; i < o->n; ++i)
      if (o->labels[i] < 0 || o->labels[i] >= o->C) {
        set_err("Objective: label outside [0, num_classes)");
        return OQ_INVALID_INPUT;
      }
  }
  return OQ_OK;
}

/* ======================================================================
 * MIRROR-mode arithmetic helpers (the B200 kernels' operation order).
 * ====================================================================== */

/* Deterministic exp/log built only from IEEE +,-,*,/,fma, rint and
 * exponent manipulation; the device code (csrc/halp_device.cuh hexp/hlog) performs the
 * identical sequence, so results agree bit for bit. */
double oq_mexp(double x) {
  if (!(x == x)) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.1332191019412) return 0.0;
  const double kf = rint(x * 1.4426950408889634);
  const double r1 = fma(-kf, 6.93147180369123816490e-01, x);
  const double r = fma(-kf, 1.90821492927058770002e-10, r1);
  /* Taylor polynomial of degree 13 evaluated by Estrin's scheme (depth 5
   * instead of 13 dependent fma; k_inner.cu/k_fullgrad.cu use the same) */
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double q0 = fma(1.0, r, 1.0);
  const double q1 = fma(1.66666666666666666667e-01, r, 0.5);
  const double q2 = fma(8.33333333333333333333e-03, r, 4.16666666666666666667e-02);
  const double q3 = fma(1.98412698412698412698e-04, r, 1.38888888888888888889e-03);
  const double q4 = fma(2.75573192239858906526e-06, r, 2.48015873015873015873e-05);
  const double q5 = fma(2.50521083854417187751e-08, r, 2.75573192239858906526e-07);
  const double q6 = fma(1.60590438368216145994e-10, r, 2.08767569878680989792e-09);
  const double e0 = fma(q1, r2, q0), e1 = fma(q3, r2, q2), e2 = fma(q5, r2, q4);
  const double u0 = fma(e1, r4, e0), u1 = fma(q6, r4, e2);
  const double p = fma(u1, r8, u0);
  const int k = (int)kf;
  /* scale by 2^k in two steps so subnormal results round once */
  if (k > -1000) {
    const int k1 = k / 2, k2 = k - k1;
    double s1, s2;
    uint64_t b1 = (uint64_t)(k1 + 1023) << 52, b2 = (uint64_t)(k2 + 1023) << 52;
    memcpy(&s1, &b1, 8);
    memcpy(&s2, &b2, 8);
    return (p * s1) * s2;
  }
  {
    double s1, s2;
    uint64_t b1 = (uint64_t)(k + 600 + 1023) << 52, b2 = (uint64_t)(-600 + 1023) << 52;
    memcpy(&s1, &b1, 8);
    memcpy(&s2, &b2, 8);
    return (p * s1) * s2;
  }
}

/* log for x > 0 finite: x = m * 2^e with m in [sqrt(1/2), sqrt(2)),
 * log(m) = 2 atanh(f), f = (m-1)/(m+1), odd polynomial in f. */
double oq_mlog(double x) {
  if (!(x == x) || x < 0.0) return NAN;
  if (x == 0.0) return -INFINITY;
  if (isinf(x)) return x;
  uint64_t b;
  memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7FF);
  if (e == 0) { /* subnormal: normalise */
    x = x * 0x1.0p54;
    memcpy(&b, &x, 8);
    e = (int)((b >> 52) & 0x7FF) - 54;
  }
  e -= 1023;
  uint64_t mb = (b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL;
  double m;
  memcpy(&m, &mb, 8);
  if (m > 1.4142135623730951) { m = m * 0.5; e += 1; }
  const double f = (m - 1.0) / (m + 1.0);
  const double f2 = f * f;
  double p = 1.0 / 23.0;
  p = fma(p, f2, 1.0 / 21.0);
  p = fma(p, f2, 1.0 / 19.0);
  p = fma(p, f2, 1.0 / 17.0);
  p = fma(p, f2, 1.0 / 15.0);
  p = fma(p, f2, 1.0 / 13.0);
  p = fma(p, f2, 1.0 / 11.0);
  p = fma(p, f2, 1.0 / 9.0);
  p = fma(p, f2, 1.0 / 7.0);
  p = fma(p, f2, 1.0 / 5.0);
  p = fma(p, f2, 1.0 / 3.0);
  const double s = (2.0 * f) * (f2 * p);           /* 2 f^3 P(f^2) */
  const double ef = (double)e;
  const double hi = fma(ef, 6.93147180369123816490e-01, 2.0 * f);
  return hi + fma(ef, 1.90821492927058770002e-10, s);
}

/* ======================================================================
 * REF mode: the reference's structure with sequential inner reductions.
 * ====================================================================== */
#define REF_BLOCK 1024 /* objectives.cpp:13 kBlock */

/* packet width of the reference build's Eigen kernels: 1 = scalar,
 * 2 = SSE2 (Packet2d), 4 = AVX (Packet4d).  Selected by pinning against the
 * golden traces (tests/test_oracle_golden.py). */
static int g_ref_lanes = 2;
void oq_set_ref_lanes(int lanes) { g_ref_lanes = lanes; }

/* logits for one row, REF order: sequential over features, which is what
 * Eigen's column-major GEMV kernel does per output row when d < 128
 * (GeneralMatrixVector.h block_cols == cols).  W is d x C column-major
 * (objectives.hpp:56-58). */
static void ref_row_logits(const double* x, const double* w, int d, int C, double* logits) {
  for (int c = 0; c < C; ++c) {
    double acc = 0.0;
    const double* wc = w + (size_t)c * d;
    for (int j = 0; j < d; ++j) acc += x[j] * wc[j];
    logits[c] = acc;
  }
}

/* softmax derivative in place (objectives.cpp:277-283 / :241-245) */
static void ref_softmax_dl(double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) { l[c] = exp(l[c] - mx); }
  for (int c = 0; c < C; ++c) s += l[c];
  for (int c = 0; c < C; ++c) l[c] = l[c] / s;
  l[label] -= 1.0;
}

static double ref_softmax_loss(const double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) s += exp(l[c] - mx);
  const double lse = mx + log(s);
  return lse - l[label];
}

/* Eigen's LinearVectorizedTraversal redux of squaredNorm() on an aligned
 * VectorXd (Eigen/src/Core/Redux.h) with P-double packets: two packet
 * accumulators over blocks of 2P, combined lane-wise, a trailing packet,
 * the horizontal add (predux), then the scalar tail. */
static double predux(const double* p, int P) {
  if (P == 1) return p[0];
  if (P == 2) return p[0] + p[1];
  return (p[0] + p[2]) + (p[1] + p[3]);
}
static double ref_sqnorm(const double* v, int64_t len) {
  const int P = g_ref_lanes;
  if (P == 1 || len < P) {
    double s = len ? v[0] * v[0] : 0.0;
    for (int64_t i = 1; i < len; ++i) s = s + v[i] * v[i];
    return s;
  }
  const int64_t a1 = (len / P) * P, a2 = (len / (2 * P)) * (2 * P);
  double p0[4], p1[4];
  for (int l = 0; l < P; ++l) p0[l] = v[l] * v[l];
  if (a1 > P) {
    for (int l = 0; l < P; ++l) p1[l] = v[P + l] * v[P + l];
    for (int64_t i = 2 * P; i < a2; i += 2 * P)
      for (int l = 0; l < P; ++l) {
        p0[l] = p0[l] + v[i + l] * v[i + l];
        p1[l] = p1[l] + v[i + P + l] * v[i + P + l];
      }
    for (int l = 0; l < P; ++l) p0[l] = p0[l] + p1[l];
    if (a1 > a2)
      for (int l = 0; l < P; ++l) p0[l] = p0[l] + v[a2 + l] * v[a2 + l];
  }
  double res = predux(p0, P);
  for (int64_t i = a1; i < len; ++i) res = res + v[i] * v[i];
  return res;
}

/* objectives.cpp:193-223 Objective::loss */
static double ref_loss(const oq_objective* o, const double* w) {
  const int d = o->d, C = o->C;
  const int64_t n = o->n;
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  double lg[64];
  double acc = 0.0;
  for (int64_t r0 = 0; r0 < n; r0 += REF_BLOCK) {
    const int64_t m = (n - r0) < REF_BLOCK ? (n - r0) : REF_BLOCK;
    double blk = 0.0;
    for (int64_t r = 0; r < m; ++r) {
      load_row(o, r0 + r, x);
      ref_row_logits(x, w, d, C, lg);
      if (o->loss == OQ_SQUARED) {
        const double e = lg[0] - o->y[r0 + r];
        blk += 0.5 * e * e;
      } else {
        blk += ref_softmax_loss(lg, C, o->labels[r0 + r]);
      }
    }
    acc += blk;
  }
  free(x);
  return acc / (double)n + 0.5 * o->l2 * ref_sqnorm(w, (int64_t)d * C);
}

/* one block of objectives.cpp:271-287: partial = X_blk^T dl */
static void ref_block_partial(const oq_objective* o, const double* w, int64_t b, double* partial,
                              double* x, double* dl) {
  const int d = o->d, C = o->C;
  const int64_t r0 = b * REF_BLOCK;
  const int64_t m = (o->n - r0) < REF_BLOCK ? (o->n - r0) : REF_BLOCK;
  for (int64_t r = 0; r < m; ++r) {
    load_row(o, r0 + r, x);
    ref_row_logits(x, w, d, C, dl + r * C);
    if (o->loss == OQ_SQUARED) dl[r] -= o->y[r0 + r];
    else ref_softmax_dl(dl + r * C, C, o->labels[r0 + r]);
  }
  /* partial(j,c) = X_blk(:,j) . dl(:,c).  Eigen evaluates X_blk^T * dl with
   * the row-major GEMV kernel (GeneralMatrixVector.h): one P-lane packet
   * accumulator per output (lane l sums rows r = l mod P), a horizontal add
   * (predux), then the scalar tail over the last m mod P rows. */
  const int P = g_ref_lanes;
  const size_t DC = (size_t)d * C;
  double* acc = (double*)calloc(DC * (size_t)P, sizeof(double));
  const int64_t mp = (m / P) * P;
  for (int64_t r = 0; r < mp; ++r) {
    load_row(o, r0 + r, x);
    double* a = acc + (size_t)(r % P) * DC;
    for (int c = 0; c < C; ++c) {
      const double dv = dl[r * C + c];
      double* pc = a + (size_t)c * d;
      for (int j = 0; j < d; ++j) pc[j] = pc[j] + x[j] * dv;
    }
  }
  for (size_t k = 0; k < DC; ++k) {
    double lanes[4];
    for (int l = 0; l < P; ++l) lanes[l] = acc[(size_t)l * DC + k];
    partial[k] = predux(lanes, P);
  }
  for (int64_t r = mp; r < m; ++r) {
    load_row(o, r0 + r, x);
    for (int c = 0; c < C; ++c) {
      const double dv = dl[r * C + c];
      double* pc = partial + (size_t)c * d;
      for (int j = 0; j < d; ++j) pc[j] = pc[j] + x[j] * dv;
    }
  }
  free(acc);
}

typedef struct {
  const oq_objective* o;
  const double* w;
  double* partials;
  int64_t nblk;
  int tid, nth;
} fg_job;

static void* fg_worker(void* arg) {
  fg_job* j = (fg_job*)arg;
  const int d = j->o->d, C = j->o->C;
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  double* dl = (double*)malloc(sizeof(double) * REF_BLOCK * (size_t)C);
  for (int64_t b = j->tid; b < j->nblk; b += j->nth)
    ref_block_partial(j->o, j->w, b, j->partials + (size_t)b * d * C, x, dl);
  free(x);
  free(dl);
  return NULL;
}

/* objectives.cpp:258-311 Objective::full_gradient (threads over blocks,
 * partials combined in block order => independent of num_threads) */
static void ref_full_gradient(const oq_objective* o, const double* w, int num_threads, double* g) {
  const int D = o->d * o->C;
  const int64_t nblk = (o->n + REF_BLOCK - 1) / REF_BLOCK;
  double* partials = (double*)malloc(sizeof(double) * (size_t)D * (size_t)nblk);
  int nth = num_threads < 1 ? 1 : num_threads;
  if (nth > nblk) nth = (int)nblk;
  fg_job* jobs = (fg_job*)calloc((size_t)nth, sizeof(fg_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nth, sizeof(pthread_t));
  for (int t = 0; t < nth; ++t) {
    jobs[t] = (fg_job){o, w, partials, nblk, t, nth};
    if (nth > 1) pthread_create(&th[t], NULL, fg_worker, &jobs[t]);
  }
  if (nth == 1) fg_worker(&jobs[0]);
  else for (int t = 0; t < nth; ++t) pthread_join(th[t], NULL);
  for (int k = 0; k < D; ++k) g[k] = 0.0;
  for (int64_t b = 0; b < nblk; ++b)
    for (int k = 0; k < D; ++k) g[k] += partials[(size_t)b * D + k];
  for (int k = 0; k < D; ++k) g[k] = g[k] / (double)o->n;
  for (int k = 0; k < D; ++k) g[k] += o->l2 * w[k];
  free(partials);
  free(jobs);
  free(th);
}

/* objectives.cpp:225-250 component_gradient_into, REF order */
static void ref_component_gradient(const oq_objective* o, const double* x, int64_t i, const double* w,
                                   double* out) {
  const int d = o->d, C = o->C;
  if (o->loss == OQ_SQUARED) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc += x[j] * w[j];
    const double e = acc - o->y[i];
    for (int j = 0; j < d; ++j) out[j] = e * x[j];
  } else {
    double p[64];
    ref_row_logits(x, w, d, C, p);
    ref_softmax_dl(p, C, o->labels[i]);
    for (int c = 0; c < C; ++c)
      for (int j = 0; j < d; ++j) out[(size_t)c * d + j] = x[j] * p[c];
  }
  for (int k = 0; k < d * C; ++k) out[k] += o->l2 * w[k];
}

/* ======================================================================
 * MIRROR mode: the B200 kernels' order.
 * ====================================================================== */

/* xor-butterfly over 32 lanes, bits 16,8,4,2,1: lane 0's final value */
static double warp_butterfly(double* v /*[32], destroyed*/) {
  for (int b = 16; b >= 1; b >>= 1) {
    double nv[32];
    for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ b];
    memcpy(v, nv, sizeof nv);
  }
  return v[0];
}

/* K1 row dot: thread t owns feature groups t, t+T, ... of width V;
 * sequential fma within a thread, warp butterfly, warps summed in order. */
static double mirror_fg_dot(const double* x, const double* w, int d, int T, int V) {
  double warpsum[64] = {0};
  const int nw = T / 32;
  for (int wi = 0; wi < nw; ++wi) {
    double v[32];
    for (int l = 0; l < 32; ++l) {
      const int t = wi * 32 + l;
      double acc = 0.0;
      for (int g = t; g * V < d; g += T)
        for (int q = 0; q < V && g * V + q < d; ++q) acc = fma(x[g * V + q], w[g * V + q], acc);
      v[l] = acc;
    }
    warpsum[wi] = warp_butterfly(v);
  }
  double s = warpsum[0];
  for (int wi = 1; wi < nw; ++wi) s = s + warpsum[wi];
  return s;
}

static void mirror_softmax_dl(double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) l[c] = oq_mexp(l[c] - mx);
  for (int c = 0; c < C; ++c) s = s + l[c];
  for (int c = 0; c < C; ++c) l[c] = l[c] / s;
  l[label] = l[label] - 1.0;
}

static double mirror_softmax_loss(const double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) s = s + oq_mexp(l[c] - mx);
  return (mx + oq_mlog(s)) - l[label];
}

/* K3's softmax derivative: exact max, deterministic exp, denominator summed
 * by a pairwise tree over 16 class slots padded with zeros (k_inner.cu) */
static void mirror_softmax_dl_k3(double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c) if (l[c] > mx) mx = l[c];
  double e[64];
  int P = 16;
  while (P < C) P *= 2; /* the device supports C <= 15 */
  for (int c = 0; c < P; ++c) e[c] = c < C ? oq_mexp(l[c] - mx) : 0.0;
  for (int h = 1; h < P; h <<= 1)
    for (int c = 0; c < P; c += 2 * h) e[c] = e[c] + e[c + h];
  const double s = e[0];
  for (int c = 0; c < C; ++c) l[c] = oq_mexp(l[c] - mx) / s;
  l[label] = l[label] - 1.0;
}

/* Two-class softmax in K1 (k_fullgrad_stream.cu): the logits enter only
 * through s = x.(w1 - w0), so K1 makes ONE dot per row with v = w1 - w0
 * (IEEE differences) and evaluates
 *   q = exp(-|s|), den = 1 + q, p0 = (s > 0 ? q : 1) / den,
 *   dl0 = p0 - [y == 0], dl1 = -dl0,
 *   loss = max(a, 0) + log(den),  a = s (y == 0) or -s (y == 1),
 * the reference's softmax rows (objectives.cpp:206-217, :277-283) for C = 2
 * up to rounding (tests: MIRROR vs REF within 1e-12).  The class-1 gradient
 * column is the exact negation of class 0's.  Returns the loss term. */
static double mirror_logistic_row(double s, int label, double* dl0) {
  const double q = oq_mexp(-fabs(s));
  const double den = 1.0 + q;
  const double p0 = (s > 0.0 ? q : 1.0) / den;
  *dl0 = label == 0 ? p0 - 1.0 : p0;
  const double a = label == 0 ? s : -s;
  return (a > 0.0 ? a : 0.0) + oq_mlog(den);
}

/* pairwise tree over n items (split at the largest power of two < n) */
static double tree_sum(const double* v, int64_t stride, int64_t n) {
  if (n == 1) return v[0];
  int64_t h = 1;
  while (h * 2 < n) h *= 2;
  return tree_sum(v, stride, h) + tree_sum(v + h * stride, stride, n - h);
}

/* K1 fused pass: per split, gradient columns accumulated by sequential fma
 * over the split's rows, per-row loss summed sequentially; splits combined
 * by a pairwise tree; then g = sum/n + l2*w, loss = tree/n + (0.5*l2)*|w|^2
 * with |w|^2 and |g|^2 computed by the finalize kernel's order. */
static void mirror_fullpass(const oq_objective* o, const double* w, const oq_plan* pl, double* g,
                            double* loss_out) {
  const int d = o->d, C = o->C, D = d * C;
  const int64_t n = o->n;
  const int S = pl->fg_splits;
  double* part = (double*)calloc((size_t)S * D, sizeof(double));
  double* lpart = (double*)calloc((size_t)S, sizeof(double));
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  double* vdiff = (double*)malloc(sizeof(double) * (size_t)d);
  if (C == 2)
    for (int j = 0; j < d; ++j) vdiff[j] = w[d + j] - w[j];
  double lg[64];
  for (int s = 0; s < S; ++s) {
    const int64_t r0 = (int64_t)((__int128)n * s / S), r1 = (int64_t)((__int128)n * (s + 1) / S);
    double* ps = part + (size_t)s * D;
    double la = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      load_row(o, r, x);
      if (C == 2) { /* two classes: the logistic form of K1 */
        const double sd = mirror_fg_dot(x, vdiff, d, pl->fg_threads, pl->fg_vec);
        double dl0;
        la = la + mirror_logistic_row(sd, o->labels[r], &dl0);
        for (int j = 0; j < d; ++j) ps[j] = fma(dl0, x[j], ps[j]);
        continue;
      }
      for (int c = 0; c < C; ++c) lg[c] = mirror_fg_dot(x, w + (size_t)c * d, d, pl->fg_threads, pl->fg_vec);
      if (o->loss == OQ_SQUARED) {
        const double e = lg[0] - o->y[r];
        la = la + (0.5 * e) * e;
        for (int j = 0; j < d; ++j) ps[j] = fma(e, x[j], ps[j]);
      } else {
        const int y = o->labels[r];
        la = la + mirror_softmax_loss(lg, C, y);
        mirror_softmax_dl(lg, C, y);
        for (int c = 0; c < C; ++c)
          for (int j = 0; j < d; ++j) ps[(size_t)c * d + j] = fma(lg[c], x[j], ps[(size_t)c * d + j]);
      }
    }
    if (C == 2)
      for (int j = 0; j < d; ++j) ps[d + j] = -ps[j];
    lpart[s] = la;
  }
  for (int k = 0; k < D; ++k) {
    const double sum = tree_sum(part + k, D, S);
    g[k] = sum / (double)n + o->l2 * w[k];
  }
  if (loss_out) {
    /* finalize kernel: |w|^2 by the 256-thread strided + butterfly order */
    double v[256];
    for (int t = 0; t < 256; ++t) {
      double a = 0.0;
      for (int k = t; k < D; k += 256) a = fma(w[k], w[k], a);
      v[t] = a;
    }
    double ws[8];
    for (int wi = 0; wi < 8; ++wi) ws[wi] = warp_butterfly(v + wi * 32);
    double sq = ws[0];
    for (int wi = 1; wi < 8; ++wi) sq = sq + ws[wi];
    *loss_out = tree_sum(lpart, 1, S) / (double)n + (0.5 * o->l2) * sq;
  }
  free(part);
  free(lpart);
  free(x);
  free(vdiff);
}

/* Root of the pairwise split tree over splits [s0, s1) in MIRROR order:
 * out[0..D) gradient column sums, out[D] the loss sum (what one rank's K1 +
 * k1_tree_pass produce before the NCCL all-gather). */
int oq_split_subtree(const oq_objective* o, const double* w, const oq_plan* pl, int64_t s0, int64_t s1,
                     double* out) {
  const int d = o->d, C = o->C, D = d * C;
  const int64_t n = o->n;
  const int S = pl->fg_splits;
  const int64_t ns = s1 - s0;
  double* part = (double*)calloc((size_t)ns * (D + 1), sizeof(double));
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  double* vdiff = (double*)malloc(sizeof(double) * (size_t)d);
  if (C == 2)
    for (int j = 0; j < d; ++j) vdiff[j] = w[d + j] - w[j];
  double lg[64];
  for (int64_t s = s0; s < s1; ++s) {
    const int64_t r0 = (int64_t)((__int128)n * s / S), r1 = (int64_t)((__int128)n * (s + 1) / S);
    double* ps = part + (size_t)(s - s0) * (D + 1);
    double la = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      load_row(o, r, x);
      if (C == 2) { /* two classes: the logistic form of K1 */
        const double sd = mirror_fg_dot(x, vdiff, d, pl->fg_threads, pl->fg_vec);
        double dl0;
        la = la + mirror_logistic_row(sd, o->labels[r], &dl0);
        for (int j = 0; j < d; ++j) ps[j] = fma(dl0, x[j], ps[j]);
        continue;
      }
      for (int c = 0; c < C; ++c) lg[c] = mirror_fg_dot(x, w + (size_t)c * d, d, pl->fg_threads, pl->fg_vec);
      if (o->loss == OQ_SQUARED) {
        const double e = lg[0] - o->y[r];
        la = la + (0.5 * e) * e;
        for (int j = 0; j < d; ++j) ps[j] = fma(e, x[j], ps[j]);
      } else {
        const int y = o->labels[r];
        la = la + mirror_softmax_loss(lg, C, y);
        mirror_softmax_dl(lg, C, y);
        for (int c = 0; c < C; ++c)
          for (int j = 0; j < d; ++j) ps[(size_t)c * d + j] = fma(lg[c], x[j], ps[(size_t)c * d + j]);
      }
    }
    if (C == 2)
      for (int j = 0; j < d; ++j) ps[d + j] = -ps[j];
    ps[D] = la;
  }
  for (int k = 0; k <= D; ++k) out[k] = tree_sum(part + k, D + 1, ns);
  free(part);
  free(x);
  free(vdiff);
  return OQ_OK;
}

/* K2 finalize over G gathered rank sums (pairwise tree over ranks) */
int oq_finalize(const oq_objective* o, const double* w, const double* rank_sums, int G, double* g, double* loss) {
  const int D = o->d * o->C;
  for (int k = 0; k < D; ++k) g[k] = tree_sum(rank_sums + k, D + 1, G) / (double)o->n + o->l2 * w[k];
  double v[256];
  for (int t = 0; t < 256; ++t) {
    double a = 0.0;
    for (int k = t; k < D; k += 256) a = fma(w[k], w[k], a);
    v[t] = a;
  }
  double ws[8];
  for (int wi = 0; wi < 8; ++wi) ws[wi] = warp_butterfly(v + wi * 32);
  double sq = ws[0];
  for (int wi = 1; wi < 8; ++wi) sq = sq + ws[wi];
  *loss = tree_sum(rank_sums + D, D + 1, G) / (double)o->n + (0.5 * o->l2) * sq;
  return OQ_OK;
}

/* finalize kernel order for |g| */
static double mirror_norm(const double* g, int D) {
  double v[256];
  for (int t = 0; t < 256; ++t) {
    double a = 0.0;
    for (int k = t; k < D; k += 256) a = fma(g[k], g[k], a);
    v[t] = a;
  }
  double ws[8];
  for (int wi = 0; wi < 8; ++wi) ws[wi] = warp_butterfly(v + wi * 32);
  double sq = ws[0];
  for (int wi = 1; wi < 8; ++wi) sq = sq + ws[wi];
  return sqrt(sq);
}

/* K3 dot order for one class c of the flat D = d*C coordinate vector:
 * global thread tau = cta*T + tid owns flat coords [tau*m, (tau+1)*m);
 * its partial for class c is a sequential fma over its coords of that
 * class; lanes are combined by the warp butterfly; the warp sums are then
 * added sequentially in global warp order (cta-major), which is the same as
 * skipping the warps that hold no coordinate of class c (their sum is +0). */
/* K3's fixed-point exchange (plan in_levels 3, squared loss, HALP): every
 * thread partial rounded to an integer at 2^S, the integers summed exactly
 * (the order no longer matters), the sum scaled back once; a non-finite
 * partial makes the dot NaN.  S from oq_fx_exponent. */
static __thread double g_fx_scale = 0.0, g_fx_inv = 0.0; /* 0: not in use (per thread: tests run oracles concurrently) */

int oq_fx_exponent(double xmax, const double* w, int64_t D, double delta, int bits) {
  double l1 = 0.0;
  for (int64_t j = 0; j < D; ++j) l1 += fabs(w[j]);
  const double B = xmax * (l1 + (double)D * delta * ldexp(1.0, bits - 1));
  if (!(B > 0.0) || !isfinite(B)) return 0;
  const int S = 59 - ilogb(B);
  return S < -1000 ? -1000 : S > 1000 ? 1000 : S;
}

static void mirror_inner_dots(const double* x, const double* wa, const double* wb, int d, int C,
                              const oq_plan* pl, double* la, double* lb) {
  if (C == 1 && g_fx_scale != 0.0) {
    const int D = d, T = pl->in_threads, m = pl->in_per, NC = pl->in_ctas;
    const int64_t nthr = (int64_t)NC * T;
    uint64_t sa = 0, sb = 0;
    int nanp = 0;
    for (int64_t tau = 0; tau < nthr; ++tau) {
      double aa = 0.0, ab = 0.0;
      for (int64_t k = tau * m; k < (tau + 1) * m && k < D; ++k) {
        aa = fma(x[k], wa[k], aa);
        ab = fma(x[k], wb[k], ab);
      }
      if (!(isfinite(aa) && isfinite(ab))) { nanp = 1; continue; }
      sa += (uint64_t)llrint(aa * g_fx_scale);
      sb += (uint64_t)llrint(ab * g_fx_scale);
    }
    la[0] = nanp ? NAN : (double)(int64_t)sa * g_fx_inv;
    lb[0] = nanp ? NAN : (double)(int64_t)sb * g_fx_inv;
    return;
  }
  const int D = d * C, T = pl->in_threads, m = pl->in_per, NC = pl->in_ctas;
  const int ngw = NC * (T / 32);
  double wsa[512], wsb[512];
  int first[64];
  for (int c = 0; c < C; ++c) { la[c] = 0.0; lb[c] = 0.0; first[c] = 1; }
  for (int gw = 0; gw < ngw; ++gw) {
    const int64_t k_lo = (int64_t)gw * 32 * m, k_hi0 = k_lo + 32 * (int64_t)m;
    const int64_t k_hi = k_hi0 < D ? k_hi0 : D;
    if (k_lo >= k_hi) {
      /* warps past D hold no coordinate: +0 records (squared loss keeps them) */
      if (C == 1) { wsa[gw] = 0.0; wsb[gw] = 0.0; }
      continue;
    }
    const int c_lo = (int)(k_lo / d), c_hi = (int)((k_hi - 1) / d);
    for (int c = c_lo; c <= c_hi; ++c) {
      double va[32], vb[32];
      for (int l = 0; l < 32; ++l) {
        const int64_t tau = (int64_t)gw * 32 + l;
        double aa = 0.0, ab = 0.0;
        for (int64_t k = tau * m; k < (tau + 1) * m && k < D; ++k) {
          if (k / d != c) continue;
          const int j = (int)(k % d);
          aa = fma(x[j], wa[k], aa);
          ab = fma(x[j], wb[k], ab);
        }
        va[l] = aa;
        vb[l] = ab;
      }
      const double sa = warp_butterfly(va), sb = warp_butterfly(vb);
      if (C == 1) { wsa[gw] = sa; wsb[gw] = sb; continue; }
      if (first[c]) { la[c] = sa; lb[c] = sb; first[c] = 0; }
      else { la[c] = la[c] + sa; lb[c] = lb[c] + sb; }
    }
  }
  if (C == 1) {
    /* in_levels 2: each CTA's warps summed in warp order first (one record
     * per CTA); then lane l sums records l, l+32, ... sequentially from 0.0;
     * lane butterfly */
    int nrec = ngw;
    if (pl->in_levels == 2) {
      const int nw = T / 32;
      for (int c = 0; c < NC; ++c) {
        double sa = wsa[c * nw], sb = wsb[c * nw];
        for (int q = 1; q < nw; ++q) { sa = sa + wsa[c * nw + q]; sb = sb + wsb[c * nw + q]; }
        wsa[c] = sa;
        wsb[c] = sb;
      }
      nrec = NC;
    }
    double va[32], vb[32];
    for (int l = 0; l < 32; ++l) {
      double aa = 0.0, ab = 0.0;
      for (int q = l; q < nrec; q += 32) { aa = aa + wsa[q]; ab = ab + wsb[q]; }
      va[l] = aa;
      vb[l] = ab;
    }
    la[0] = warp_butterfly(va);
    lb[0] = warp_butterfly(vb);
  }
}

/* Markstein division check used by tests/test_division.py: the device
 * quantizer computes u/delta as fma(x - q0*delta, rcp, q0) with
 * q0 = x*rcp, rcp = 1/delta; count mismatches against IEEE division. */
int64_t oq_div_check(int64_t n, uint64_t seed) {
  oq_rng r;
  oq_rng_init(&r, seed, 7);
  int64_t bad = 0;
  for (int64_t it = 0; it < n; ++it) {
    uint64_t mb = oq_next_u64(&r) & 0x000FFFFFFFFFFFFFULL;
    const int mode = (int)(it % 4);
    if (mode == 1) mb = 0x000FFFFFFFFFFFFFULL;
    if (mode == 2) mb &= 0x000FF00000000000ULL;
    const int e = 1023 + (int)(oq_next_u64(&r) % 120) - 60;
    const uint64_t db = mb | ((uint64_t)e << 52);
    double delta;
    memcpy(&delta, &db, 8);
    const double t = ldexp((double)(int64_t)(oq_next_u64(&r) >> 11) * 0x1.0p-53 * 2.0 - 1.0,
                           (int)(oq_next_u64(&r) % 24));
    double x = t * delta;
    if (it % 7 == 0) x = nextafter(x, (oq_next_u64(&r) & 1) ? INFINITY : -INFINITY);
    if (it % 11 == 0) x = (double)((int64_t)(oq_next_u64(&r) % 65536) - 32768) * delta;
    const double rc = 1.0 / delta;
    const double q0 = x * rc;
    const double rem = fma(-q0, delta, x);
    const double q1 = fma(rem, rc, q0);
    const double qt = x / delta;
    if (q1 != qt && !(q1 == 0.0 && qt == 0.0)) ++bad;
  }
  return bad;
}

/* ------------------------------------------------------------ public API */
int oq_loss(const oq_objective* o, const double* w, const oq_plan* plan, double* out) {
  int rc = check_objective(o);
  if (rc) return rc;
  if (!plan) { *out = ref_loss(o, w); return OQ_OK; }
  double* g = (double*)malloc(sizeof(double) * (size_t)o->d * o->C);
  mirror_fullpass(o, w, plan, g, out);
  free(g);
  return OQ_OK;
}

int oq_full_gradient(const oq_objective* o, const double* w, int num_threads, const oq_plan* plan,
                     double* g) {
  int rc = check_objective(o);
  if (rc) return rc;
  if (num_threads < 1) { set_err("full_gradient: num_threads must be >= 1"); return OQ_INVALID_INPUT; }
  if (!plan) ref_full_gradient(o, w, num_threads, g);
  else mirror_fullpass(o, w, plan, g, NULL);
  return OQ_OK;
}

int oq_component_gradient(const oq_objective* o, int64_t i, const double* w, const oq_plan* plan,
                          double* out) {
  int rc = check_objective(o);
  if (rc) return rc;
  if (i < 0 || i >= o->n) { set_err("component_gradient: index out of range"); return OQ_INVALID_INPUT; }
  double* x = (double*)malloc(sizeof(double) * (size_t)o->d);
  load_row(o, i, x);
  (void)plan;
  ref_component_gradient(o, x, i, w, out);
  free(x);
  return OQ_OK;
}

/* optimizers.cpp:209-216 */
int64_t oq_resolve_inner_steps(const oq_config* cfg, int64_t n) {
  const int64_t t = cfg->inner_steps > 0 ? cfg->inner_steps : (int64_t)cfg->full_grad_period * n;
  return t < 1 ? -1 : t;
}

/* optimizers.cpp:218-227 FNV-1a over the iterate's bytes */
uint64_t oq_hash_vector(const double* v, int64_t len) {
  uint64_t h = 1469598103934665603ULL;
  const unsigned char* p = (const unsigned char*)v;
  const size_t nb = sizeof(double) * (size_t)len;
  for (size_t i = 0; i < nb; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

uint64_t oq_code_hash(const int64_t* codes, int64_t len) {
  uint64_t h = 1469598103934665603ULL;
  for (int64_t q = 0; q < len; ++q) {
    uint64_t v = (uint64_t)codes[q];
    for (int b = 0; b < 8; ++b, v >>= 8) {
      h ^= v & 255u;
      h *= 1099511628211ULL;
    }
  }
  return h;
}

/* optimizers.cpp:36-97 (the HALP-relevant checks) */
static int validate_config(const oq_objective* o, const oq_config* c) {
  (void)o;
  if (!(isfinite(c->alpha) && c->alpha >= 0.0)) { set_err("optimizer: alpha must be finite and >= 0"); return OQ_INVALID_INPUT; }
  if (c->epochs < 0) { set_err("optimizer: epochs must be >= 0"); return OQ_INVALID_INPUT; }
  if (c->inner_steps < 0) { set_err("optimizer: inner_steps must be >= 0"); return OQ_INVALID_INPUT; }
  if (c->full_grad_period < 1) { set_err("optimizer: full_grad_period must be >= 1"); return OQ_INVALID_INPUT; }
  if (!(isfinite(c->metric_every_passes) && c->metric_every_passes >= 0.0)) {
    set_err("optimizer: metric_every_passes must be finite and >= 0");
    return OQ_INVALID_INPUT;
  }
  if (!(isfinite(c->divergence_limit) && c->divergence_limit > 0.0)) {
    set_err("optimizer: divergence_limit must be positive");
    return OQ_INVALID_INPUT;
  }
  if (!(isfinite(c->delta_min) && c->delta_min > 0.0)) { set_err("optimizer: delta_min must be positive"); return OQ_INVALID_INPUT; }
  if (c->algorithm == OQ_ALGO_LP_SVRG || c->algorithm == OQ_ALGO_LP_SGD) { /* uses_fixed_scale */
    if (c->bits < 2 || c->bits > 64) { set_err("optimizer: bits must be in [2, 64]"); return OQ_INVALID_INPUT; }
    if (!(isfinite(c->delta) && c->delta > 0.0)) {
      set_err("optimizer: delta must be positive for fixed-scale runs");
      return OQ_INVALID_INPUT;
    }
  }
  if (c->algorithm == OQ_ALGO_HALP) { /* uses_bit_centering */
    if (c->bits < 2 || c->bits > 64) { set_err("optimizer: bits must be in [2, 64]"); return OQ_INVALID_INPUT; }
    if (!(isfinite(c->mu) && c->mu > 0.0)) { set_err("optimizer: mu must be positive for bit-centered runs"); return OQ_INVALID_INPUT; }
  }
  return OQ_OK;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* optimizers.cpp:104-167 Recorder */
typedef struct {
  const oq_config* cfg;
  oq_record* rec;
  double t0, next_pass;
  int D;
  double delta_inner, delta_aux; /* LM-HALP rows only (set before rec_boundary) */
} recorder;

static int rec_due(const recorder* r, double pass, int forced) {
  return forced || r->cfg->metric_every_passes <= 0.0 || pass + 1e-9 >= r->next_pass;
}

/* returns OQ_DIVERGED if the guard fired (record finalised) */
static int rec_boundary(recorder* r, double pass, const double* w, double loss, double gn, double delta,
                        int forced) {
  const int bad = !(isfinite(loss) && isfinite(gn)) || loss > r->cfg->divergence_limit ||
                  gn > r->cfg->divergence_limit;
  if (rec_due(r, pass, forced) || bad) {
    if (r->rec->rows_n >= r->rec->rows_cap) { set_err("oracle: rows capacity exceeded"); return OQ_CAPACITY; }
    oq_row* row = &r->rec->rows[r->rec->rows_n++];
    row->pass = pass;
    row->seconds = now_s() - r->t0;
    row->loss = loss;
    row->grad_norm = gn;
    row->delta = delta;
    row->iterate_hash = oq_hash_vector(w, r->D);
    row->delta_inner = r->delta_inner;
    row->delta_aux = r->delta_aux;
    if (r->cfg->metric_every_passes > 0.0) r->next_pass = pass + r->cfg->metric_every_passes;
  }
  if (bad) {
    r->rec->status = OQ_STATUS_DIVERGED;
    memcpy(r->rec->final_iterate, w, sizeof(double) * (size_t)r->D);
    char m[128];
    snprintf(m, sizeof m, "run diverged near pass %f", pass);
    set_err(m);
    return OQ_DIVERGED;
  }
  return OQ_OK;
}

/* one epoch-boundary measurement: gradient, norm, delta, loss */
static void measure(const oq_objective* o, const double* wt, const oq_config* cfg, const oq_plan* plan,
                    int fg_threads, double* gt, double* gn, double* delta, double* loss, double* tsec) {
  const double t0 = now_s();
  if (!plan) {
    ref_full_gradient(o, wt, fg_threads, gt);
    *gn = sqrt(ref_sqnorm(gt, (int64_t)o->d * o->C));
  } else {
    mirror_fullpass(o, wt, plan, gt, loss);
    *gn = mirror_norm(gt, o->d * o->C);
  }
  *delta = 0.0;
  if (cfg->algorithm == OQ_ALGO_HALP && isfinite(*gn) && *gn > 0.0) {
    double s = oq_halp_scale(*gn, cfg->mu, cfg->bits);
    *delta = s > cfg->delta_min ? s : cfg->delta_min;
  }
  if (!plan) *loss = ref_loss(o, wt);
  *tsec += now_s() - t0;
}

/* optimizers.cpp:387-459 run_halp */
int oq_run_halp(const oq_objective* o, const oq_config* cfg, const oq_plan* plan, oq_record* rec) {
  int rc = check_objective(o);
  if (rc) return rc;
  rc = validate_config(o, cfg);
  if (rc) return rc;
  const int d = o->d, C = o->C, D = d * C;
  const int64_t n = o->n;
  const int64_t T = oq_resolve_inner_steps(cfg, n);
  if (T < 1) { set_err("optimizer: epoch length must be >= 1"); return OQ_INVALID_INPUT; }
  oq_rng sample, rounder;
  oq_rng_init(&sample, cfg->seed, 0);  /* kSampleStream, optimizers.cpp:17 */
  oq_rng_init(&rounder, cfg->seed, 1); /* kRoundStream,  optimizers.cpp:18 */

  double* wt = (double*)calloc((size_t)D, sizeof(double));
  if (cfg->init) memcpy(wt, cfg->init, sizeof(double) * (size_t)D);
  double* z = (double*)calloc((size_t)D, sizeof(double));
  double* wz = (double*)malloc(sizeof(double) * (size_t)D);
  double* u = (double*)malloc(sizeof(double) * (size_t)D);
  double* g1 = (double*)malloc(sizeof(double) * (size_t)D);
  double* g2 = (double*)malloc(sizeof(double) * (size_t)D);
  double* gt = (double*)malloc(sizeof(double) * (size_t)D);
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  int64_t* code = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  int64_t* snap = (int64_t*)calloc((size_t)D, sizeof(int64_t));

  rec->rows_n = 0;
  rec->status = OQ_STATUS_OK;
  rec->steps_taken = 0;
  rec->inner_fp_vector_ops = 0;
  rec->fullgrad_seconds = 0.0;
  rec->inner_seconds = 0.0;
  recorder r = {cfg, rec, now_s(), 0.0, D, 0.0, 0.0};
  int64_t steps = 0, traced = 0, hashed = 0;
  int converged = 0;
  const int fgth = rec->fullgrad_threads > 0 ? rec->fullgrad_threads : 1;
  rc = OQ_OK;

  const int fx = plan && plan->in_levels == 3 && C == 1;
  double xmax = 0.0;
  if (fx) {
    for (int64_t i = 0; i < n; ++i) {
      load_row(o, i, x);
      for (int j = 0; j < d; ++j) {
        const double v = fabs(x[j]);
        if (v > xmax || v != v) xmax = v;
      }
    }
  }
  for (int k = 0; k < cfg->epochs && !converged; ++k) {
    double gn, delta, loss;
    measure(o, wt, cfg, plan, fgth, gt, &gn, &delta, &loss, &rec->fullgrad_seconds);
    rc = rec_boundary(&r, (double)steps / (double)n, wt, loss, gn, delta, k == 0 || gn == 0.0);
    if (rc) goto done;
    if (gn == 0.0) { rec->status = OQ_STATUS_CONVERGED; converged = 1; break; }
    if (fx) {
      const int S = oq_fx_exponent(xmax, wt, D, delta, cfg->bits);
      g_fx_scale = ldexp(1.0, S);
      g_fx_inv = ldexp(1.0, -S);
    }
    /* z = Q(0): D draws, all codes 0 (optimizers.cpp:414-417) */
    for (int q = 0; q < D; ++q) {
      const double uu = oq_next_uniform(&rounder);
      code[q] = oq_quantize_code(0.0, delta, cfg->bits, uu, NULL);
      snap[q] = code[q];
    }
    for (int q = 0; q < D; ++q) z[q] = (double)code[q] * delta;
    int64_t t_pick = -1;
    if (cfg->option == 1) t_pick = (int64_t)oq_next_index(&sample, (uint64_t)T);
    const double ti0 = now_s();
    for (int64_t t = 0; t < T; ++t) {
      if (t == t_pick) memcpy(snap, code, sizeof(int64_t) * (size_t)D);
      const int64_t i = (int64_t)oq_next_index(&sample, (uint64_t)n);
      for (int q = 0; q < D; ++q) wz[q] = wt[q] + z[q];
      load_row(o, i, x);
      if (!plan) {
        ref_component_gradient(o, x, i, wz, g1);
        ref_component_gradient(o, x, i, wt, g2);
      } else {
        double la[64], lb[64];
        mirror_inner_dots(x, wz, wt, d, C, plan, la, lb);
        if (o->loss == OQ_SQUARED) {
          const double e1 = la[0] - o->y[i], e2 = lb[0] - o->y[i];
          for (int j = 0; j < d; ++j) {
            g1[j] = e1 * x[j] + o->l2 * wz[j];
            g2[j] = e2 * x[j] + o->l2 * wt[j];
          }
        } else {
          const int y = o->labels[i];
          mirror_softmax_dl_k3(la, C, y);
          mirror_softmax_dl_k3(lb, C, y);
          for (int c = 0; c < C; ++c)
            for (int j = 0; j < d; ++j) {
              const size_t q = (size_t)c * d + j;
              g1[q] = x[j] * la[c] + o->l2 * wz[q];
              g2[q] = x[j] * lb[c] + o->l2 * wt[q];
            }
        }
      }
      int finite = 1;
      for (int q = 0; q < D; ++q) {
        u[q] = z[q] - cfg->alpha * ((g1[q] - g2[q]) + gt[q]);
        if (!isfinite(u[q])) finite = 0;
      }
      if (!finite) {
        /* Recorder::blowup (optimizers.cpp:156-160, 432-434) */
        rc = rec_boundary(&r, (double)(steps + t + 1) / (double)n, u, INFINITY, INFINITY, delta, 1);
        goto done;
      }
      for (int q = 0; q < D; ++q) {
        const double uu = oq_next_uniform(&rounder);
        code[q] = oq_quantize_code(u[q], delta, cfg->bits, uu, NULL);
      }
      for (int q = 0; q < D; ++q) z[q] = (double)code[q] * delta;
      if (rec->trace_codes && traced + D <= rec->trace_cap) {
        memcpy(rec->trace_codes + traced, code, sizeof(int64_t) * (size_t)D);
        traced += D;
      }
      if (rec->step_hash && hashed < rec->step_hash_cap) rec->step_hash[hashed++] = oq_code_hash(code, D);
    }
    rec->inner_seconds += now_s() - ti0;
    rec->inner_fp_vector_ops += (uint64_t)(8 * T);
    if (cfg->option == 1)
      for (int q = 0; q < D; ++q) z[q] = (double)snap[q] * delta;
    for (int q = 0; q < D; ++q) wt[q] += z[q];
    steps += T;
  }
  if (!converged) {
    double gn, delta, loss;
    measure(o, wt, cfg, plan, fgth, gt, &gn, &delta, &loss, &rec->fullgrad_seconds);
    rc = rec_boundary(&r, (double)steps / (double)n, wt, loss, gn, delta, 1);
    if (rc) goto done;
    if (gn == 0.0) rec->status = OQ_STATUS_CONVERGED;
  }
  memcpy(rec->final_iterate, wt, sizeof(double) * (size_t)D);
  rec->steps_taken = steps;
done:
  g_fx_scale = g_fx_inv = 0.0;
  /* a DivergenceError's partial record keeps steps_taken == 0: the
   * reference only assigns it after the loop (optimizers.cpp:457) */
  if (rc == OQ_DIVERGED) rec->steps_taken = 0;
  free(wt); free(z); free(wz); free(u); free(g1); free(g2); free(gt); free(x); free(code); free(snap);
  return rc;
}

/* Component gradients at w (g1) and wt (g2) of row i, REF or MIRROR order
 * (MIRROR = the inner-loop kernel's dots, k_inner.cu). */
static void component_pair(const oq_objective* o, const oq_plan* plan, const double* x, int64_t i, const double* w,
                           const double* wt, double* g1, double* g2) {
  const int d = o->d, C = o->C;
  if (!plan) {
    ref_component_gradient(o, x, i, w, g1);
    ref_component_gradient(o, x, i, wt, g2);
    return;
  }
  double la[64], lb[64];
  mirror_inner_dots(x, w, wt, d, C, plan, la, lb);
  if (o->loss == OQ_SQUARED) {
    const double e1 = la[0] - o->y[i], e2 = lb[0] - o->y[i];
    for (int j = 0; j < d; ++j) {
      g1[j] = e1 * x[j] + o->l2 * w[j];
      g2[j] = e2 * x[j] + o->l2 * wt[j];
    }
  } else {
    const int y = o->labels[i];
    mirror_softmax_dl_k3(la, C, y);
    mirror_softmax_dl_k3(lb, C, y);
    for (int c = 0; c < C; ++c)
      for (int j = 0; j < d; ++j) {
        const size_t q = (size_t)c * d + j;
        g1[q] = x[j] * la[c] + o->l2 * w[q];
        g2[q] = x[j] * lb[c] + o->l2 * wt[q];
      }
  }
}

/* optimizers.cpp:258-296 run_svrg (lp = 0) and :336-385 run_lp_svrg (lp = 1).
 * SVRG: w -= alpha*((g1 - g2) + gt), no finiteness check inside the epoch;
 * LP-SVRG: the iterate is Q(u) at the fixed scale cfg->delta (one rounding
 * draw per coordinate, the initial iterate quantized once), a non-finite u
 * is a blow-up row.  Rows carry delta = 0 (SVRG) / cfg->delta (LP-SVRG). */
static int run_svrg_family(const oq_objective* o, const oq_config* cfg, const oq_plan* plan, oq_record* rec, int lp) {
  int rc = check_objective(o);
  if (rc) return rc;
  rc = validate_config(o, cfg);
  if (rc) return rc;
  const int d = o->d, C = o->C, D = d * C;
  const int64_t n = o->n;
  const int64_t T = oq_resolve_inner_steps(cfg, n);
  if (T < 1) { set_err("optimizer: epoch length must be >= 1"); return OQ_INVALID_INPUT; }
  const double rdelta = lp ? cfg->delta : 0.0;
  oq_rng sample, rounder;
  oq_rng_init(&sample, cfg->seed, 0);
  oq_rng_init(&rounder, cfg->seed, 1);
  double* wt = (double*)calloc((size_t)D, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (size_t)D);
  double* snapw = (double*)malloc(sizeof(double) * (size_t)D);
  double* u = (double*)malloc(sizeof(double) * (size_t)D);
  double* g1 = (double*)malloc(sizeof(double) * (size_t)D);
  double* g2 = (double*)malloc(sizeof(double) * (size_t)D);
  double* gt = (double*)malloc(sizeof(double) * (size_t)D);
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  int64_t* wt_lp = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  int64_t* w_lp = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  int64_t* snap_lp = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  if (cfg->init) memcpy(wt, cfg->init, sizeof(double) * (size_t)D);
  if (lp) { /* wt_lp = quantize_vector(w0), wt = to_real(wt_lp) */
    for (int q = 0; q < D; ++q) {
      const double uu = oq_next_uniform(&rounder);
      int err = 0;
      wt_lp[q] = oq_quantize_code(wt[q], cfg->delta, cfg->bits, uu, &err);
      if (err) { set_err("quantize: non-finite input"); rc = OQ_INVALID_INPUT; goto done; }
    }
    for (int q = 0; q < D; ++q) wt[q] = (double)wt_lp[q] * cfg->delta;
  }
  rec->rows_n = 0;
  rec->status = OQ_STATUS_OK;
  rec->steps_taken = 0;
  rec->inner_fp_vector_ops = 0;
  rec->fullgrad_seconds = 0.0;
  rec->inner_seconds = 0.0;
  recorder r = {cfg, rec, now_s(), 0.0, D, 0.0, 0.0};
  int64_t steps = 0, traced = 0;
  const int fgth = rec->fullgrad_threads > 0 ? rec->fullgrad_threads : 1;
  for (int k = 0; k < cfg->epochs; ++k) {
    double gn, dl, loss;
    measure(o, wt, cfg, plan, fgth, gt, &gn, &dl, &loss, &rec->fullgrad_seconds);
    rc = rec_boundary(&r, (double)steps / (double)n, wt, loss, gn, rdelta, k == 0);
    if (rc) goto done;
    int64_t t_pick = -1;
    if (cfg->option == 1) t_pick = (int64_t)oq_next_index(&sample, (uint64_t)T);
    memcpy(w, wt, sizeof(double) * (size_t)D);
    memcpy(snapw, wt, sizeof(double) * (size_t)D);
    memcpy(w_lp, wt_lp, sizeof(int64_t) * (size_t)D);
    memcpy(snap_lp, wt_lp, sizeof(int64_t) * (size_t)D);
    const double ti0 = now_s();
    for (int64_t t = 0; t < T; ++t) {
      if (t == t_pick) {
        if (lp) memcpy(snap_lp, w_lp, sizeof(int64_t) * (size_t)D);
        else memcpy(snapw, w, sizeof(double) * (size_t)D);
      }
      const int64_t i = (int64_t)oq_next_index(&sample, (uint64_t)n);
      load_row(o, i, x);
      component_pair(o, plan, x, i, w, wt, g1, g2);
      if (!lp) {
        for (int q = 0; q < D; ++q) w[q] = w[q] - cfg->alpha * ((g1[q] - g2[q]) + gt[q]);
        continue;
      }
      int finite = 1;
      for (int q = 0; q < D; ++q) {
        u[q] = w[q] - cfg->alpha * ((g1[q] - g2[q]) + gt[q]);
        if (!isfinite(u[q])) finite = 0;
      }
      if (!finite) {
        rc = rec_boundary(&r, (double)(steps + t + 1) / (double)n, u, INFINITY, INFINITY, cfg->delta, 1);
        goto done;
      }
      for (int q = 0; q < D; ++q) {
        const double uu = oq_next_uniform(&rounder);
        w_lp[q] = oq_quantize_code(u[q], cfg->delta, cfg->bits, uu, NULL);
      }
      for (int q = 0; q < D; ++q) w[q] = (double)w_lp[q] * cfg->delta;
      if (rec->trace_codes && traced + D <= rec->trace_cap) {
        memcpy(rec->trace_codes + traced, w_lp, sizeof(int64_t) * (size_t)D);
        traced += D;
      }
    }
    rec->inner_seconds += now_s() - ti0;
    rec->inner_fp_vector_ops += (uint64_t)((lp ? 7 : 5) * T); /* 2 component gradients (2 each) + the update (+ quantize, to_real) */
    if (lp) {
      memcpy(wt_lp, cfg->option == 1 ? snap_lp : w_lp, sizeof(int64_t) * (size_t)D);
      for (int q = 0; q < D; ++q) wt[q] = (double)wt_lp[q] * cfg->delta;
    } else {
      memcpy(wt, cfg->option == 1 ? snapw : w, sizeof(double) * (size_t)D);
    }
    steps += T;
  }
  {
    double gn, dl, loss;
    measure(o, wt, cfg, plan, fgth, gt, &gn, &dl, &loss, &rec->fullgrad_seconds);
    rc = rec_boundary(&r, (double)steps / (double)n, wt, loss, gn, rdelta, 1);
    if (rc) goto done;
  }
  memcpy(rec->final_iterate, wt, sizeof(double) * (size_t)D);
  rec->steps_taken = steps;
done:
  if (rc == OQ_DIVERGED) rec->steps_taken = 0;
  free(wt); free(w); free(snapw); free(u); free(g1); free(g2); free(gt); free(x);
  free(wt_lp); free(w_lp); free(snap_lp);
  return rc;
}

/* optimizers.cpp:229-256 run_sgd (lp = 0) and :297-334 run_lp_sgd (lp = 1):
 * w -= alpha*g (SGD, no in-epoch finiteness check) or w = Q(w - alpha*g) at
 * the fixed scale (the initial iterate quantized once; blow-up rows). */
static int run_sgd_family(const oq_objective* o, const oq_config* cfg, const oq_plan* plan, oq_record* rec, int lp) {
  int rc = check_objective(o);
  if (rc) return rc;
  rc = validate_config(o, cfg);
  if (rc) return rc;
  const int d = o->d, C = o->C, D = d * C;
  const int64_t n = o->n;
  const int64_t T = oq_resolve_inner_steps(cfg, n);
  if (T < 1) { set_err("optimizer: epoch length must be >= 1"); return OQ_INVALID_INPUT; }
  const double rdelta = lp ? cfg->delta : 0.0;
  oq_rng sample, rounder;
  oq_rng_init(&sample, cfg->seed, 0);
  oq_rng_init(&rounder, cfg->seed, 1);
  double* w = (double*)calloc((size_t)D, sizeof(double));
  double* u = (double*)malloc(sizeof(double) * (size_t)D);
  double* g = (double*)malloc(sizeof(double) * (size_t)D);
  double* g2 = (double*)malloc(sizeof(double) * (size_t)D);
  double* gt = (double*)malloc(sizeof(double) * (size_t)D);
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  int64_t* w_lp = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  if (cfg->init) memcpy(w, cfg->init, sizeof(double) * (size_t)D);
  if (lp) {
    for (int q = 0; q < D; ++q) {
      const double uu = oq_next_uniform(&rounder);
      int err = 0;
      w_lp[q] = oq_quantize_code(w[q], cfg->delta, cfg->bits, uu, &err);
      if (err) { set_err("quantize: non-finite input"); rc = OQ_INVALID_INPUT; goto done; }
    }
    for (int q = 0; q < D; ++q) w[q] = (double)w_lp[q] * cfg->delta;
  }
  rec->rows_n = 0;
  rec->status = OQ_STATUS_OK;
  rec->steps_taken = 0;
  rec->inner_fp_vector_ops = 0;
  rec->fullgrad_seconds = 0.0;
  rec->inner_seconds = 0.0;
  recorder r = {cfg, rec, now_s(), 0.0, D, 0.0, 0.0};
  int64_t steps = 0, traced = 0;
  const int fgth = rec->fullgrad_threads > 0 ? rec->fullgrad_threads : 1;
  for (int k = 0; k < cfg->epochs; ++k) {
    double gn, dl, loss;
    measure(o, w, cfg, plan, fgth, gt, &gn, &dl, &loss, &rec->fullgrad_seconds);
    rc = rec_boundary(&r, (double)steps / (double)n, w, loss, gn, rdelta, k == 0);
    if (rc) goto done;
    const double ti0 = now_s();
    for (int64_t t = 0; t < T; ++t) {
      const int64_t i = (int64_t)oq_next_index(&sample, (uint64_t)n);
      load_row(o, i, x);
      component_pair(o, plan, x, i, w, w, g, g2);
      if (!lp) {
        for (int q = 0; q < D; ++q) w[q] = w[q] - cfg->alpha * g[q];
        continue;
      }
      int finite = 1;
      for (int q = 0; q < D; ++q) {
        u[q] = w[q] - cfg->alpha * g[q];
        if (!isfinite(u[q])) finite = 0;
      }
      if (!finite) {
        rc = rec_boundary(&r, (double)(steps + t + 1) / (double)n, u, INFINITY, INFINITY, cfg->delta, 1);
        goto done;
      }
      for (int q = 0; q < D; ++q) {
        const double uu = oq_next_uniform(&rounder);
        w_lp[q] = oq_quantize_code(u[q], cfg->delta, cfg->bits, uu, NULL);
      }
      for (int q = 0; q < D; ++q) w[q] = (double)w_lp[q] * cfg->delta;
      if (rec->trace_codes && traced + D <= rec->trace_cap) {
        memcpy(rec->trace_codes + traced, w_lp, sizeof(int64_t) * (size_t)D);
        traced += D;
      }
    }
    rec->inner_seconds += now_s() - ti0;
    rec->inner_fp_vector_ops += (uint64_t)((lp ? 5 : 3) * T); /* component gradient (2) + update (+ quantize, to_real) */
    steps += T;
  }
  {
    double gn, dl, loss;
    measure(o, w, cfg, plan, fgth, gt, &gn, &dl, &loss, &rec->fullgrad_seconds);
    rc = rec_boundary(&r, (double)steps / (double)n, w, loss, gn, rdelta, 1);
    if (rc) goto done;
  }
  memcpy(rec->final_iterate, w, sizeof(double) * (size_t)D);
  rec->steps_taken = steps;
done:
  if (rc == OQ_DIVERGED) rec->steps_taken = 0;
  free(w); free(u); free(g); free(g2); free(gt); free(x); free(w_lp);
  return rc;
}

int oq_run(const oq_objective* o, const oq_config* cfg, const oq_plan* plan, oq_record* rec) {
  switch (cfg->algorithm) {
    case OQ_ALGO_SGD: return run_sgd_family(o, cfg, plan, rec, 0);
    case OQ_ALGO_LP_SGD: return run_sgd_family(o, cfg, plan, rec, 1);
    case OQ_ALGO_HALP: return oq_run_halp(o, cfg, plan, rec);
    case OQ_ALGO_SVRG: return run_svrg_family(o, cfg, plan, rec, 0);
    case OQ_ALGO_LP_SVRG: return run_svrg_family(o, cfg, plan, rec, 1);
    case OQ_ALGO_LM_HALP: set_err("lm_halp: dataset has no quantized examples"); return OQ_INVALID_INPUT;
    default: set_err("oracle: algorithm not restated"); return OQ_INVALID_INPUT;
  }
}

/* ======================================================================
 * LM-HALP (optimizers.cpp:461-627): the integer inner loop of the paper's
 * linear-model form.  REF = the reference's order (sequential epoch sweep,
 * std::exp); MIRROR = the B200 kernels' (k_lm.cu: split tree over the
 * device's splits with 128-thread row dots, deterministic exp).  The inner
 * loop is integer arithmetic (exact in any order) apart from the link
 * derivative.
 * ====================================================================== */

/* fixed_point.cpp data_scale (objectives.cpp:112-122) + quantize_dataset
 * (:124-133): one LPRepr for the whole matrix, stream 2, row-major draws */
int oq_quantize_dataset(const double* X, int64_t n, int d, int bits, uint64_t seed, int64_t* codes, double* delta) {
  if (bits < 2 || bits > 64) { set_err("data_scale: bits must be in [2, 64]"); return OQ_INVALID_INPUT; }
  double max_abs = 0.0;
  for (int64_t k = 0; k < n * (int64_t)d; ++k) {
    const double a = fabs(X[k]);
    if (!(a <= max_abs)) max_abs = a; /* NaN propagates like Eigen's maxCoeff of cwiseAbs */
  }
  if (!isfinite(max_abs)) { set_err("data_scale: matrix has non-finite entries"); return OQ_INVALID_INPUT; }
  const double span = ldexp(1.0, bits - 1) - 1.0;
  const double dl = max_abs == 0.0 ? 1.0 : max_abs / span;
  oq_rng rng;
  oq_rng_init(&rng, seed, 2);
  for (int64_t k = 0; k < n * (int64_t)d; ++k) {
    const double u = oq_next_uniform(&rng);
    codes[k] = oq_quantize_code(X[k], dl, bits, u, NULL);
  }
  *delta = dl;
  return OQ_OK;
}

static int64_t lm_sat(int64_t c, int bits) {
  const int64_t lo = min_code_for(bits), hi = max_code_for(bits);
  return c < lo ? lo : c > hi ? hi : c;
}
/* sub_same_scale (fixed_point.cpp:150-165) */
static int64_t lm_sub(int64_t a, int64_t b, int bits) {
  int64_t s;
  if (__builtin_sub_overflow(a, b, &s)) s = a > b ? INT64_MAX : INT64_MIN;
  return lm_sat(s, bits);
}
/* requantize_shift (fixed_point.cpp:223-243) for one code */
static int64_t lm_requant(int64_t c, int shift, int out_bits, double u) {
  int64_t hi = c >> shift;
  const int64_t low = c - (int64_t)((uint64_t)hi << shift);
  if (low != 0 && u < ldexp((double)low, -shift)) ++hi;
  return lm_sat(hi, out_bits);
}

/* squared: dl = l - y; softmax: the order of the mode (REF std::exp, MIRROR hexp) */
static void lm_link_dl(const oq_objective* o, int64_t i, const double* l, double* dl, int mirror) {
  const int C = o->C;
  for (int c = 0; c < C; ++c) dl[c] = l[c];
  if (o->loss == OQ_SQUARED) { dl[0] = l[0] - o->y[i]; return; }
  if (mirror) mirror_softmax_dl(dl, C, o->labels[i]);
  else ref_softmax_dl(dl, C, o->labels[i]);
}
static double lm_link_loss(const oq_objective* o, int64_t i, const double* l, int mirror) {
  if (o->loss == OQ_SQUARED) {
    const double r = l[0] - o->y[i];
    return 0.5 * r * r;
  }
  return mirror ? mirror_softmax_loss(l, o->C, o->labels[i]) : ref_softmax_loss(l, o->C, o->labels[i]);
}

/* epoch_stats (optimizers.cpp:486-505): phi [n][C], g, loss; returns gn */
static double lm_epoch_stats(const oq_objective* o, const oq_quantized* q, const double* wt, const oq_plan* plan,
                             double* phi, double* g, double* loss_out) {
  const int d = o->d, C = o->C, D = d * C;
  const int64_t n = o->n;
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  double lg[64], dl[64];
  if (!plan) {
    for (int k = 0; k < D; ++k) g[k] = 0.0;
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      for (int j = 0; j < d; ++j) x[j] = (double)q->codes[i * d + j] * q->delta;
      ref_row_logits(x, wt, d, C, lg);
      for (int c = 0; c < C; ++c) phi[i * C + c] = lg[c];
      acc += lm_link_loss(o, i, lg, 0);
      lm_link_dl(o, i, lg, dl, 0);
      for (int c = 0; c < C; ++c)
        for (int j = 0; j < d; ++j) g[(size_t)c * d + j] += x[j] * dl[c];
    }
    for (int k = 0; k < D; ++k) g[k] /= (double)n;
    for (int k = 0; k < D; ++k) g[k] += o->l2 * wt[k];
    *loss_out = acc / (double)n + 0.5 * o->l2 * ref_sqnorm(wt, D);
    free(x);
    return sqrt(ref_sqnorm(g, D));
  }
  /* MIRROR: splits of the device plan, sequential rows inside a split,
   * 128-thread row dots (V = 1), gradient by fma, pairwise split tree */
  const int S = plan->fg_splits;
  double* part = (double*)calloc((size_t)S * D, sizeof(double));
  double* lpart = (double*)calloc((size_t)S, sizeof(double));
  for (int s = 0; s < S; ++s) {
    const int64_t r0 = (int64_t)((__int128)n * s / S), r1 = (int64_t)((__int128)n * (s + 1) / S);
    double* ps = part + (size_t)s * D;
    double la = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      for (int j = 0; j < d; ++j) x[j] = (double)q->codes[r * d + j] * q->delta;
      for (int c = 0; c < C; ++c) lg[c] = mirror_fg_dot(x, wt + (size_t)c * d, d, 128, 1);
      for (int c = 0; c < C; ++c) phi[r * C + c] = lg[c];
      la = la + lm_link_loss(o, r, lg, 1);
      lm_link_dl(o, r, lg, dl, 1);
      for (int c = 0; c < C; ++c)
        for (int j = 0; j < d; ++j) ps[(size_t)c * d + j] = fma(dl[c], x[j], ps[(size_t)c * d + j]);
    }
    lpart[s] = la;
  }
  for (int k = 0; k < D; ++k) g[k] = tree_sum(part + k, D, S) / (double)n + o->l2 * wt[k];
  double v[256];
  for (int t = 0; t < 256; ++t) {
    double a = 0.0;
    for (int k = t; k < D; k += 256) a = fma(wt[k], wt[k], a);
    v[t] = a;
  }
  double ws[8];
  for (int wi = 0; wi < 8; ++wi) ws[wi] = warp_butterfly(v + wi * 32);
  double sq = ws[0];
  for (int wi = 1; wi < 8; ++wi) sq = sq + ws[wi];
  *loss_out = tree_sum(lpart, 1, S) / (double)n + (0.5 * o->l2) * sq;
  free(part);
  free(lpart);
  free(x);
  return mirror_norm(g, D);
}

/* the scale chain of optimizers.cpp:509-521 (and :600-606); 0 = fine, else invalid */
static int lm_scales(double gn, const oq_config* cfg, double delta_d, double* dm, double* di, double* daux, int check) {
  *dm = *di = *daux = 0.0;
  if (isfinite(gn) && gn > 0.0) {
    double s = oq_halp_scale(gn, cfg->mu, cfg->bits);
    if (s < cfg->delta_min) s = cfg->delta_min;
    const double di0 = ldexp(s, -cfg->bits);
    *daux = di0 / delta_d;
    if (check && !(isfinite(*daux) && *daux > 0.0)) {
      set_err("lm_halp: auxiliary scale left the double range");
      return OQ_INVALID_INPUT;
    }
    *di = *daux * delta_d;
    *dm = ldexp(*di, cfg->bits);
  }
  return OQ_OK;
}

int oq_run_lm_halp(const oq_objective* o, const oq_quantized* q, const oq_config* cfg, const oq_plan* plan,
                   oq_record* rec) {
  int rc = check_objective(o);
  if (rc) return rc;
  oq_config c2 = *cfg;
  c2.algorithm = OQ_ALGO_HALP; /* the generic checks of validate_config (bit-centred) */
  rc = validate_config(o, &c2);
  if (rc) return rc;
  if (cfg->bits > 32) { set_err("lm_halp: bits must be <= 32 (inner arithmetic is 2b wide)"); return OQ_INVALID_INPUT; }
  if (cfg->option != 0) { set_err("lm_halp: only the last-iterate epoch update is defined"); return OQ_INVALID_INPUT; }
  if (!q || !q->codes) { set_err("lm_halp: dataset has no quantized examples"); return OQ_INVALID_INPUT; }
  if (q->bits != cfg->bits) { set_err("lm_halp: dataset quantized at a different width"); return OQ_INVALID_INPUT; }
  const int d = o->d, C = o->C, D = d * C, b = cfg->bits;
  const int64_t n = o->n;
  const int64_t T = oq_resolve_inner_steps(cfg, n);
  if (T < 1) { set_err("optimizer: epoch length must be >= 1"); return OQ_INVALID_INPUT; }
  oq_rng sample, rounder;
  oq_rng_init(&sample, cfg->seed, 0);
  oq_rng_init(&rounder, cfg->seed, 1);
  double* wt = (double*)calloc((size_t)D, sizeof(double));
  if (cfg->init) memcpy(wt, cfg->init, sizeof(double) * (size_t)D);
  double* phi = (double*)malloc(sizeof(double) * (size_t)(n * C));
  double* g = (double*)malloc(sizeof(double) * (size_t)D);
  int64_t* z = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  int64_t* h = (int64_t*)calloc((size_t)D, sizeof(int64_t));
  rec->rows_n = 0;
  rec->status = OQ_STATUS_OK;
  rec->steps_taken = 0;
  rec->inner_fp_vector_ops = 0;
  rec->inner_lp_vector_ops = 0;
  rec->fullgrad_seconds = 0.0;
  rec->inner_seconds = 0.0;
  recorder r = {cfg, rec, now_s(), 0.0, D, 0.0, 0.0};
  int64_t steps = 0, traced = 0, hashed = 0;
  int converged = 0;
  rc = OQ_OK;
  for (int k = 0; k < cfg->epochs && !converged; ++k) {
    double loss = 0.0, dm, di, daux;
    const double t0 = now_s();
    const double gn = lm_epoch_stats(o, q, wt, plan, phi, g, &loss);
    rec->fullgrad_seconds += now_s() - t0;
    rc = lm_scales(gn, cfg, q->delta, &dm, &di, &daux, 1);
    if (rc) goto done;
    r.delta_inner = di;
    r.delta_aux = daux;
    rc = rec_boundary(&r, (double)steps / (double)n, wt, loss, gn, dm, k == 0 || gn == 0.0);
    if (rc) goto done;
    if (gn == 0.0) { rec->status = OQ_STATUS_CONVERGED; converged = 1; break; }
    /* zcols = Q_m(0): D draws (class-major), codes 0 */
    for (int kk = 0; kk < D; ++kk) { (void)oq_next_uniform(&rounder); z[kk] = 0; }
    /* h_wide = widen_range(Q_i(alpha * g_c), b) */
    for (int kk = 0; kk < D; ++kk) {
      const double a = cfg->alpha * g[kk];
      int err = 0;
      h[kk] = oq_quantize_code(a, di, b, oq_next_uniform(&rounder), &err);
      if (err) { set_err("quantize: input must be finite"); rc = OQ_INVALID_INPUT; goto done; }
    }
    const double sc = q->delta * dm; /* dot_lp: (double)acc * (delta_x * delta_z) */
    const double ti0 = now_s();
    double lg[64], ph[64], dl[64], dl0[64];
    for (int64_t t = 0; t < T; ++t) {
      const int64_t i = (int64_t)oq_next_index(&sample, (uint64_t)n);
      const int64_t* xr = q->codes + i * d;
      for (int c = 0; c < C; ++c) {
        __int128 acc = 0;
        for (int j = 0; j < d; ++j) acc += (__int128)xr[j] * (__int128)z[(size_t)c * d + j];
        lg[c] = phi[i * C + c] + (double)acc * sc;
        ph[c] = phi[i * C + c];
      }
      lm_link_dl(o, i, lg, dl, plan != NULL);
      lm_link_dl(o, i, ph, dl0, plan != NULL);
      for (int c = 0; c < C; ++c) {
        const double beta = cfg->alpha * (dl[c] - dl0[c]);
        int err = 0;
        const int64_t gam = oq_quantize_code(beta, daux, b, oq_next_uniform(&rounder), &err);
        if (err) { set_err("quantize: input must be finite"); rc = OQ_INVALID_INPUT; goto done; }
        for (int j = 0; j < d; ++j) {
          const size_t kk = (size_t)c * d + j;
          const int64_t wz = z[kk] * ((int64_t)1 << b);          /* widen_shift */
          const int64_t u1 = lm_sub(wz, xr[j] * gam, 2 * b);     /* - mul_scalar */
          const int64_t u = lm_sub(u1, h[kk], 2 * b);            /* - h_wide */
          z[kk] = lm_requant(u, b, b, oq_next_uniform(&rounder)); /* requantize_shift */
        }
      }
      if (rec->trace_codes && traced + D <= rec->trace_cap) {
        memcpy(rec->trace_codes + traced, z, sizeof(int64_t) * (size_t)D);
        traced += D;
      }
      if (rec->step_hash && hashed < rec->step_hash_cap) rec->step_hash[hashed++] = oq_code_hash(z, D);
    }
    rec->inner_seconds += now_s() - ti0;
    rec->inner_lp_vector_ops += (uint64_t)(6 * C) * (uint64_t)T;
    for (int kk = 0; kk < D; ++kk) wt[kk] += (double)z[kk] * dm;
    steps += T;
  }
  if (!converged) {
    double loss = 0.0, dm, di, daux;
    const double gn = lm_epoch_stats(o, q, wt, plan, phi, g, &loss);
    lm_scales(gn, cfg, q->delta, &dm, &di, &daux, 0);
    r.delta_inner = di;
    r.delta_aux = daux;
    rc = rec_boundary(&r, (double)steps / (double)n, wt, loss, gn, dm, 1);
    if (rc) goto done;
    if (gn == 0.0) rec->status = OQ_STATUS_CONVERGED;
  }
  memcpy(rec->final_iterate, wt, sizeof(double) * (size_t)D);
  rec->steps_taken = steps;
done:
  if (rc == OQ_DIVERGED) rec->steps_taken = 0;
  free(wt); free(phi); free(g); free(z); free(h);
  return rc;
}
