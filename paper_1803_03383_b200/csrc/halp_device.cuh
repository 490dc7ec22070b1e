// halp_device.cuh -- device-side building blocks shared by the HALP kernels.
//
//  * counter-indexed xorshift64* (reference QuantRng, proj/include/lpopt/rng.hpp:34-51):
//    the state update is GF(2)-linear, so a jump of k draws is a 64x64 bit
//    matrix applied through 8 byte-indexed tables (rng_jump.hpp).
//  * the reference quantizer (proj/src/fixed_point.cpp:30-50), bit-exact.
//  * deterministic exp/log (same operation sequence as oracle/halp_oracle.c
//    oq_mexp/oq_mlog) so softmax results are reproducible on the CPU.
//  * mbarrier / cp.async.bulk helpers for the HBM-streaming full-gradient pass.
//
// This translation unit family is compiled with -fmad=false: no a*b+c is
// contracted unless written as fma(); the reference's element-wise
// arithmetic has no FMA (proj/CMakeLists.txt:27 sets no -march).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace halp {

constexpr uint64_t kXsMul = 0x2545F4914F6CDD1DULL;  // rng.hpp:38

__device__ __forceinline__ uint64_t xs_step(uint64_t s) {  // rng.hpp:35-37
  s ^= s >> 12;
  s ^= s << 25;
  s ^= s >> 27;
  return s;
}

// s' = M s for the GF(2) matrix M encoded as 8 tables of 256 words
__device__ __forceinline__ uint64_t jump_tab(uint64_t s, const uint64_t* __restrict__ tab) {
  uint64_t r = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) r ^= tab[b * 256 + ((s >> (8 * b)) & 255u)];
  return r;
}

// jump by an arbitrary count with the power tables X^(2^b), b = 0..63
__device__ __forceinline__ uint64_t jump_count(uint64_t s, uint64_t count, const uint64_t* __restrict__ pow_tab) {
  for (int b = 0; count; ++b, count >>= 1)
    if (count & 1) s = jump_tab(s, pow_tab + (size_t)b * 2048);
  return s;
}

// next_uniform() given the already-advanced state (rng.hpp:42-44)
__device__ __forceinline__ double uniform_of(uint64_t state) {
  return __ull2double_rn((state * kXsMul) >> 11) * 0x1.0p-53;
}
// next_index(n) given the already-advanced state (rng.hpp:48-51)
__device__ __forceinline__ uint64_t index_of(uint64_t state, uint64_t n) { return __umul64hi(state * kXsMul, n); }

// quantize_code (fixed_point.cpp:30-50).  `u` is always consumed by the caller.
__device__ __forceinline__ long long quantize_code(double x, double delta, double hi, double lo, long long maxc,
                                                   long long minc, double u) {
  const double t = x / delta;
  if (t >= hi) return maxc;
  if (t <= lo) return minc;
  const double snapped = rint(t);
  if (__dmul_rn(snapped, delta) == x) return __double2ll_rn(snapped);
  const double fl = floor(t);
  const double frac = t - fl;
  long long code = __double2ll_rn(fl);
  if (frac > 0.0 && u < frac) ++code;
  return code;
}

// t = x / delta, correctly rounded, from the host's rcp = RN(1/delta):
// q0 = RN(x*rcp), r = x - q0*delta (exact with fma), q1 = RN(q0 + r*rcp)
// is the IEEE quotient (Markstein's theorem; tests/test_division.py checks
// 2e8 cases against x/delta).  Outside the safe range (huge quotient, tiny
// x, non-finite) the IEEE division is used.
__device__ __forceinline__ double div_rcp(double x, double delta, double rcp) {
  const double q0 = __dmul_rn(x, rcp);
  const double r = fma(-q0, delta, x);
  const double q1 = fma(r, rcp, q0);
  const double ax = fabs(x);
  if (fabs(q0) <= 0x1.0p60 && (ax >= 0x1.0p-960 || ax == 0.0)) return q1;
  return x / delta;
}

// quantize_code with the reciprocal division
__device__ __forceinline__ long long quantize_code_rcp(double x, double delta, double rcp, double hi, double lo,
                                                       long long maxc, long long minc, double u) {
  const double t = rcp != 0.0 ? div_rcp(x, delta, rcp) : x / delta;
  if (t >= hi) return maxc;
  if (t <= lo) return minc;
  const double snapped = rint(t);
  if (__dmul_rn(snapped, delta) == x) return __double2ll_rn(snapped);
  const double fl = floor(t);
  const double frac = t - fl;
  long long code = __double2ll_rn(fl);
  if (frac > 0.0 && u < frac) ++code;
  return code;
}

// Branch-free quantize_code returning the code as an exact double
// (|code| < 2^53; callers with bits > 53 use quantize_code).  The
// reference's branches (fixed_point.cpp:37-49) are mutually exclusive, so
// evaluating every candidate and selecting gives the same code; t comes
// from div_rcp's fast path and `slow` reports operands that need the IEEE
// fallback (the caller recomputes those coordinates).
__device__ __forceinline__ double quantize_fast(double x, double delta, double rcp, double hi, double lo, double u,
                                                bool& slow) {
  const double q0 = __dmul_rn(x, rcp);
  const double r = fma(-q0, delta, x);
  const double t = fma(r, rcp, q0);
  const double ax = fabs(x);
  slow = !(fabs(q0) <= 0x1.0p60 && (ax >= 0x1.0p-960 || ax == 0.0));
  const double sn = rint(t);
  const double fl = floor(t);
  const double frac = t - fl;
  const bool onlat = __dmul_rn(sn, delta) == x;
  const bool up = frac > 0.0 && u < frac;
  double c = onlat ? sn : (up ? fl + 1.0 : fl);
  c = (t <= lo) ? lo : c;
  c = (t >= hi) ? hi : c;
  return c;
}

template <class T> __device__ __forceinline__ double to_d(T v);
template <> __device__ __forceinline__ double to_d<double>(double v) { return v; }
template <> __device__ __forceinline__ double to_d<float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 v) {
  return (double)__bfloat162float(v);
}

// ---- deterministic exp / log (oq_mexp / oq_mlog) ----
__device__ __forceinline__ double hexp(double x) {
  if (!(x == x)) return x;
  if (x > 709.782712893384) return __longlong_as_double(0x7FF0000000000000LL);
  if (x < -745.1332191019412) return 0.0;
  const double kf = rint(__dmul_rn(x, 1.4426950408889634));
  const double r1 = fma(-kf, 6.93147180369123816490e-01, x);
  const double r = fma(-kf, 1.90821492927058770002e-10, r1);
  // degree-13 Taylor polynomial by Estrin's scheme (oq_mexp, same order)
  const double r2 = __dmul_rn(r, r), r4 = __dmul_rn(r2, r2), r8 = __dmul_rn(r4, r4);
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
  if (k > -1000) {
    const int k1 = k / 2, k2 = k - k1;
    const double s1 = __longlong_as_double((long long)(k1 + 1023) << 52);
    const double s2 = __longlong_as_double((long long)(k2 + 1023) << 52);
    return __dmul_rn(__dmul_rn(p, s1), s2);
  }
  const double s1 = __longlong_as_double((long long)(k + 600 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(-600 + 1023) << 52);
  return __dmul_rn(__dmul_rn(p, s1), s2);
}

// hexp for x <= 0 (or NaN) without branches: the same operations as hexp on
// that domain (both scalings selected, the underflow cut applied at the end),
// so the results are bit-identical; used where the argument is -|s|.
__device__ __forceinline__ double hexp_nonpos(double x) {
  const double kf = rint(__dmul_rn(x, 1.4426950408889634));
  const double r1 = fma(-kf, 6.93147180369123816490e-01, x);
  const double r = fma(-kf, 1.90821492927058770002e-10, r1);
  const double r2 = __dmul_rn(r, r), r4 = __dmul_rn(r2, r2), r8 = __dmul_rn(r4, r4);
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
  const bool inr = x >= -745.1332191019412;  // false for NaN and the underflow range
  const int k = inr ? (int)kf : 0;
  const bool near = k > -1000;
  const int k1 = near ? k / 2 : k + 600, k2 = near ? k - k / 2 : -600;
  const double s1 = __longlong_as_double((long long)(k1 + 1023) << 52);
  const double s2 = __longlong_as_double((long long)(k2 + 1023) << 52);
  const double v = __dmul_rn(__dmul_rn(p, s1), s2);
  return inr ? v : (x == x ? 0.0 : x);
}

// hlog for x in [1, 2] without branches: the same operations as hlog on that
// domain (bit-identical); used for log(1 + exp(-|s|)).
__device__ __forceinline__ double hlog_1to2(double x) {
  const bool hi = x > 1.4142135623730951;
  const double m = hi ? __dmul_rn(x, 0.5) : x;
  const double num = m - 1.0;
  const double f = num == 0.0 ? 0.0 : (num == 0.0 ? 1.0 : num) / (m + 1.0);
  const double f2 = __dmul_rn(f, f);
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
  const double s = __dmul_rn(__dmul_rn(2.0, f), __dmul_rn(f2, p));
  const double ef = hi ? 1.0 : 0.0;
  const double h = fma(ef, 6.93147180369123816490e-01, __dmul_rn(2.0, f));
  return h + fma(ef, 1.90821492927058770002e-10, s);
}

__device__ __forceinline__ double hlog(double x) {
  if (!(x == x) || x < 0.0) return __longlong_as_double(0x7FF8000000000000LL);
  if (x == 0.0) return __longlong_as_double((long long)0xFFF0000000000000ULL);
  if (isinf(x)) return x;
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7FF);
  if (e == 0) {
    x = __dmul_rn(x, 0x1.0p54);
    b = (unsigned long long)__double_as_longlong(x);
    e = (int)((b >> 52) & 0x7FF) - 54;
  }
  e -= 1023;
  double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL));
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  // (m - 1) / (m + 1) with a zero dividend (x a power of two) would take the
  // IEEE division's slow path: divide a nonzero stand-in and select 0 instead
  const double num = m - 1.0;
  const double f = num == 0.0 ? 0.0 : (num == 0.0 ? 1.0 : num) / (m + 1.0);
  const double f2 = __dmul_rn(f, f);
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
  const double s = __dmul_rn(__dmul_rn(2.0, f), __dmul_rn(f2, p));
  const double ef = (double)e;
  const double hi = fma(ef, 6.93147180369123816490e-01, __dmul_rn(2.0, f));
  return hi + fma(ef, 1.90821492927058770002e-10, s);
}

// softmax derivative in place, the oracle's mirror order (max, exp, sequential sum, divide, -1)
template <int CMAX>
__device__ __forceinline__ void softmax_dl(double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c)
    if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) l[c] = hexp(l[c] - mx);
  for (int c = 0; c < C; ++c) s = s + l[c];
  for (int c = 0; c < C; ++c) l[c] = l[c] / s;
  l[label] = l[label] - 1.0;
}

__device__ __forceinline__ double softmax_loss(const double* l, int C, int label) {
  double mx = l[0];
  for (int c = 1; c < C; ++c)
    if (l[c] > mx) mx = l[c];
  double s = 0.0;
  for (int c = 0; c < C; ++c) s = s + hexp(l[c] - mx);
  return (mx + hlog(s)) - l[label];
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- mbarrier + bulk async copy (sm_90+; SASS UBLKCP / SYNCS) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- cluster helpers ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store a double into CTA `rank`'s shared memory at the same offset as `local`
__device__ __forceinline__ void st_cluster_f64(const double* local, uint32_t rank, double v) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

__device__ __forceinline__ void st_cluster_s32(const int* local, uint32_t rank, int v) {
  uint32_t a = smem_u32(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace halp
