/*
 * datagen.c -- host restatement of the K6 synthetic-data generator
 * (paper_1803_03383_b200/csrc/k_datagen.cu), byte for byte.
 *
 * TEST INFRASTRUCTURE ONLY (see halp_oracle.h): it lets the tests and the
 * CPU arms of bench.py (cpu_baseline, --impl reference) build the BASELINE
 * configs' datasets -- or any row range of them -- without loading the
 * product library.  tests/test_gpu_datagen.py checks it against K6.
 *
 * The generator uses only integer hashing, IEEE-exact float/double
 * operations (compiled with -ffp-contract=off, like the kernel's
 * -fmad=false) and the oracle's deterministic exp/log (oq_mexp / oq_mlog =
 * the device hexp / hlog), so both sides produce identical bits.
 *
 * kind 0: x ~ N(0, x_scale^2), w* ~ N(0,1), y = x.w* + noise_sd N(0,1)   (C3, C5)
 * kind 1: x ~ U[0,1) kept w.p. density, teacher W ~ N(0,1) (d x C),
 *         label = argmax_c (x.W_c + Gumbel)                              (C2)
 * kind 2: x ~ N(0, x_scale^2), w* ~ N(0,1), label ~ Bernoulli(sigmoid(x.w*)) (C4)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "halp_oracle.h"

static uint64_t dg_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
static uint64_t dg_ctr(uint64_t seed, uint64_t stream, uint64_t i) {
  return dg_mix64(dg_mix64(seed ^ (stream * 0xD1B54A32D192ED03ULL)) + i * 0x9E3779B97F4A7C15ULL);
}
static double dg_unif64(uint64_t seed, uint64_t stream, uint64_t i) {
  return (double)(dg_ctr(seed, stream, i) >> 11) * 0x1.0p-53;
}
static float dg_logf(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  int e = (int)((b >> 23) & 255u) - 127;
  const uint32_t mb = (b & 0x7FFFFFu) | 0x3F800000u;
  float m;
  memcpy(&m, &mb, 4);
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e += 1;
  }
  const float f = (m - 1.0f) / (m + 1.0f);
  const float f2 = f * f;
  float q = 0.0909090909f;
  q = q * f2 + 0.111111111f;
  q = q * f2 + 0.142857143f;
  q = q * f2 + 0.2f;
  q = q * f2 + 0.333333333f;
  const float tf = 2.0f * f;
  const float lnm = tf + tf * (f2 * q);
  const float ef = (float)e;
  return ef * 0.693145752f + (ef * 1.42860677e-06f + lnm);
}
static float dg_cos2pi(uint32_t k) {
  const uint32_t qu = (k + (1u << 21)) >> 22;
  const int r = (int)k - (int)(qu << 22);
  const float a = (float)r * 3.74507028e-07f;
  const float a2 = a * a;
  const float c = 1.0f + a2 * (-0.5f + a2 * (0.0416666667f + a2 * (-0.00138888889f + a2 * 2.48015873e-05f)));
  const float s = a + (a * a2) * (-0.166666667f + a2 * (0.00833333333f + a2 * (-0.000198412698f + a2 * 2.75573192e-06f)));
  const uint32_t q = qu & 3u;
  return q == 0 ? c : q == 1 ? -s : q == 2 ? -c : s;
}
static float dg_normal32(uint64_t seed, uint64_t stream, uint64_t i) {
  const uint64_t h = dg_ctr(seed, stream, i);
  const float u1 = ((float)(h >> 40) + 0.5f) * 0x1.0p-24f;
  return sqrtf(-2.0f * dg_logf(u1)) * dg_cos2pi((uint32_t)((h >> 16) & 0xFFFFFFu));
}
static uint16_t dg_bf16(float v) { /* __float2bfloat16_rn for finite v */
  uint32_t u;
  memcpy(&u, &v, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
static double dg_bf16_to_d(uint16_t b) {
  const uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

typedef struct {
  const oq_datagen_desc* g;
  int64_t r0, r1; /* global rows [r0, r1) of this worker */
  int64_t row_base;
  void* X;
  double* y;
  int32_t* labels;
  const double* wsm;
} dg_job;

static void* dg_worker(void* arg) {
  const dg_job* j = (const dg_job*)arg;
  const oq_datagen_desc* g = j->g;
  const int d = g->d, C = g->kind == 1 ? g->num_classes : 1;
  const float sc = (float)g->x_scale;
  double* xr = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t i = j->r0; i < j->r1; ++i) {
    const int64_t li = i - j->row_base;
    for (int jj = 0; jj < d; ++jj) { /* k_gen_x */
      const uint64_t e = (uint64_t)i * (uint64_t)d + (uint64_t)jj;
      float v;
      if (g->kind == 1) {
        const uint64_t h = dg_ctr(g->seed, 1, e);
        const float u = (float)(h >> 40) * 0x1.0p-24f;
        const float keep = (float)((h >> 16) & 0xFFFFFF) * 0x1.0p-24f;
        v = keep < (float)g->density ? u : 0.0f;
      } else {
        v = dg_normal32(g->seed, 1, e) * sc;
      }
      const size_t at = (size_t)li * d + jj;
      if (g->dtype == OQ_F64) { ((double*)j->X)[at] = (double)v; xr[jj] = (double)v; }
      else if (g->dtype == OQ_F32) { ((float*)j->X)[at] = v; xr[jj] = (double)v; }
      else { const uint16_t b = dg_bf16(v); ((uint16_t*)j->X)[at] = b; xr[jj] = dg_bf16_to_d(b); }
    }
    /* k_gen_y: lane l accumulates features l, l+32, ... with fma; warp_allsum butterfly */
    double acc[64];
    for (int c = 0; c < C; ++c) {
      double v[32];
      for (int l = 0; l < 32; ++l) {
        double a = 0.0;
        for (int jj = l; jj < d; jj += 32) a = fma(xr[jj], j->wsm[(size_t)c * d + jj], a);
        v[l] = a;
      }
      for (int o = 16; o >= 1; o >>= 1) {
        double nv[32];
        for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
        memcpy(v, nv, sizeof v);
      }
      acc[c] = v[0];
    }
    if (g->kind == 0) {
      j->y[li] = acc[0] + g->noise_sd * (double)dg_normal32(g->seed, 3, (uint64_t)i);
    } else if (g->kind == 1) {
      int best = 0;
      double bv = -1e300;
      for (int c = 0; c < C; ++c) {
        const double u = dg_unif64(g->seed, 4, (uint64_t)i * C + c) + 0x1.0p-54;
        const double v = acc[c] - oq_mlog(-oq_mlog(u));
        if (v > bv) { bv = v; best = c; }
      }
      j->labels[li] = best;
    } else {
      const double pr = 1.0 / (1.0 + oq_mexp(-acc[0]));
      j->labels[li] = dg_unif64(g->seed, 4, (uint64_t)i) < pr ? 1 : 0;
    }
  }
  free(xr);
  return NULL;
}

int oq_datagen(const oq_datagen_desc* g, int64_t row0, int64_t nrows, int nthreads, void* X, double* y,
               int32_t* labels) {
  if (!g || !X || g->d < 1 || g->n < 1 || row0 < 0 || nrows < 0 || row0 + nrows > g->n || g->kind < 0 || g->kind > 2 ||
      g->dtype < 0 || g->dtype > 2)
    return OQ_INVALID_INPUT;
  if (g->kind == 0 && !y) return OQ_INVALID_INPUT;
  if (g->kind != 0 && !labels) return OQ_INVALID_INPUT;
  if (g->kind == 1 && (g->num_classes < 2 || g->num_classes > 64)) return OQ_INVALID_INPUT;
  const int C = g->kind == 1 ? g->num_classes : 1;
  double* wsm = (double*)malloc(sizeof(double) * (size_t)g->d * C);
  for (int64_t k = 0; k < (int64_t)g->d * C; ++k) wsm[k] = (double)dg_normal32(g->seed, 2, (uint64_t)k);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nrows < nthreads) nthreads = nrows > 0 ? (int)nrows : 1;
  pthread_t th[256];
  dg_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (dg_job){g, row0 + nrows * t / nthreads, row0 + nrows * (t + 1) / nthreads, row0, X, y, labels, wsm};
    if (nthreads > 1) pthread_create(&th[t], NULL, dg_worker, &jobs[t]);
    else dg_worker(&jobs[t]);
  }
  if (nthreads > 1)
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(wsm);
  return OQ_OK;
}
