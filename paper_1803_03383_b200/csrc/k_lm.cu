// k_lm.cu -- LM-HALP, the paper's linear-model form of HALP with an
// integer-only inner loop (reference: lpopt::run_lm_halp,
// proj/src/optimizers.cpp:461-627, non-bypass path; the fixed-point ops of
// proj/src/fixed_point.cpp:131-260).
//
// K7 k_lm_stats -- epoch_stats (optimizers.cpp:486-505): one sweep over the
//   dequantized rows x = code * delta_x (to_real, fixed_point.cpp:113-123)
//   giving phi_i = W~^T x_i for every row (kept for the inner loop), the
//   loss and the gradient.  One CTA per split of the problem's split grid;
//   rows of a split in order; row dot = 128-thread order (thread t owns
//   features t, t+128, ..., sequential fma; warp butterfly; the 4 warps in
//   order); gradient (c, j) = sequential fma over the split's rows.  The
//   splits then go through the K1 split tree and k_finalize (g = sum/n +
//   l2 w, |g|, loss) -- MIRROR order of oracle oq_run_lm_halp.
//
// K8 k3_lm -- the T-step inner loop of one epoch, one CTA (persistent),
//   thread tau owning the M flat coordinates [tau*M, tau*M + M) of z
//   (column-major d x C, objectives.hpp:56-58).  Per step i (K4's index
//   stream):
//     acc_c  = sum_j x_ij z_cj               exact int64 (dot_lp's int128 sum;
//                                             |x z| < 2^(2b-2), b <= 16)
//     logit_c = phi_ic + (double)acc_c * (delta_x * delta_m)
//     beta_c = alpha (dl_c(logit) - dl_c(phi_i)), gamma_c = Q_aux(beta_c)
//     u = sat2b(sat2b(z 2^b - x gamma_c) - h_c)   (widen_shift, mul_scalar,
//                                                  sub_same_scale x2)
//     z = requantize_shift(u, b)             stochastic, one draw per coordinate
//   The per-class sums are integer atomics into shared memory, so their
//   order does not matter: the dot is bit-identical to the reference's.
//   Draws: per step and class c, gamma_c then the d coordinate draws
//   (optimizers.cpp:556-563); every thread jumps C(d+1) draws per step with
//   the GF(2) table in shared memory, and the owner of (c, 0) publishes
//   gamma_c's uniform before the step's barrier.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

constexpr int kLmThreads = 128;  // k_lm_stats row-dot order (mirror_fg_dot T=128, V=1)

template <class Tq>
__global__ void __launch_bounds__(kLmThreads) k_lm_stats(LmStatsParams p) {
  extern __shared__ double sm[];  // w~ [D], gradient accumulators [D]
  __shared__ double wsum[2][4][16];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int d = p.d, C = p.C, D = d * C;
  double* w_s = sm;
  double* g_s = sm + D;
  for (int k = tid; k < D; k += kLmThreads) {
    w_s[k] = p.w[k];
    g_s[k] = 0.0;
  }
  __syncthreads();
  const int s = p.split0 + blockIdx.x;
  const int64_t r0 = (int64_t)(((unsigned __int128)p.n * s) / p.S);
  const int64_t r1 = (int64_t)(((unsigned __int128)p.n * (s + 1)) / p.S);
  const Tq* Q = reinterpret_cast<const Tq*>(p.q);
  double la = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const int par = (int)(r & 1);
    const Tq* qr = Q + r * d;
    double acc[kMaxClasses];
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c) acc[c] = 0.0;
    for (int j = tid; j < d; j += kLmThreads) {
      const double x = __dmul_rn((double)qr[j], p.delta_x);
#pragma unroll
      for (int c = 0; c < kMaxClasses; ++c)
        if (c < C) acc[c] = fma(x, w_s[c * d + j], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c)
      if (c < C) {
        const double v = warp_allsum(acc[c]);
        if (lane == 0) wsum[par][wid][c] = v;
      }
    __syncthreads();
    double l[kMaxClasses], dl[kMaxClasses];
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c)
      if (c < C) l[c] = ((wsum[par][0][c] + wsum[par][1][c]) + wsum[par][2][c]) + wsum[par][3][c];
    if (tid == 0)
      for (int c = 0; c < C; ++c) p.phi[r * C + c] = l[c];
    if (p.loss == 0) {
      const double e = l[0] - p.y[r];
      dl[0] = e;
      if (tid == 0) la = la + __dmul_rn(__dmul_rn(0.5, e), e);
    } else {
      const int y = p.labels[r];
      if (tid == 0) la = la + softmax_loss(l, C, y);
      for (int c = 0; c < C; ++c) dl[c] = l[c];
      softmax_dl<kMaxClasses>(dl, C, y);
    }
    for (int j = tid; j < d; j += kLmThreads) {
      const double x = __dmul_rn((double)qr[j], p.delta_x);
      for (int c = 0; c < C; ++c) g_s[c * d + j] = fma(dl[c], x, g_s[c * d + j]);
    }
  }
  __syncthreads();
  double* out = p.partials + (size_t)blockIdx.x * (D + 1);
  for (int k = tid; k < D; k += kLmThreads) out[k] = g_s[k];
  if (tid == 0) out[D] = la;
}

// Q_aux(beta): quantize_code (fixed_point.cpp:30-50) at the auxiliary scale
__device__ __forceinline__ long long lm_quantize_beta(double x, double delta, double hi, double lo, long long maxc,
                                                      long long minc, double u, int* bad) {
  if (!isfinite(x)) {
    *bad = 1;
    return 0;
  }
  return quantize_code(x, delta, hi, lo, maxc, minc, u);
}

template <class Tq, int M>
__global__ void __launch_bounds__(256, 1) k3_lm(LmInnerParams p) {
  __shared__ uint64_t jt[2048];
  __shared__ unsigned long long acc[3][16];
  __shared__ double ug[2][16];
  __shared__ int bad_s;
  const int tid = threadIdx.x;
  const int d = p.d, C = p.C, D = d * C, b = p.bits;
  for (int i = tid; i < 2048; i += blockDim.x) jt[i] = p.jump_tab[i];
  if (tid < 48) (&acc[0][0])[tid] = 0ull;
  if (tid == 0) bad_s = 0;
  const int k0 = tid * M;
  bool valid[M];
  int cls[M], fj[M];
  long long z[M], h[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int k = k0 + i;
    valid[i] = k < D;
    cls[i] = valid[i] ? k / d : 0;
    fj[i] = valid[i] ? k % d : 0;
    z[i] = 0;
    h[i] = valid[i] ? p.h[k] : 0;
  }
  // this thread's first draw in a step: gamma of its first class if it owns (c, 0)
  const int64_t first = valid[0] ? (int64_t)cls[0] * (d + 1) + (fj[0] == 0 ? 0 : 1 + fj[0]) : 0;
  uint64_t rs = jump_count(p.rstate0, (uint64_t)first, p.pow_tab);
  const long long hi2 = (1LL << (2 * b - 1)) - 1, lo2 = -(1LL << (2 * b - 1));
  const long long hib = (1LL << (b - 1)) - 1, lob = -(1LL << (b - 1));
  const double p2mb = ldexp(1.0, -b);
  const Tq* Q = reinterpret_cast<const Tq*>(p.q);
  // raw x codes of the next step's row (one step of prefetch) + its phi / target
  int64_t row = p.idx[0];
  Tq xn[M];
#pragma unroll
  for (int i = 0; i < M; ++i) xn[i] = Q[row * d + fj[i]];
  __syncthreads();
  int bad = 0;
  for (int64_t t = 0; t < p.T; ++t) {
    const int b3 = (int)(t % 3), par = (int)(t & 1);
    long long xq[M];
#pragma unroll
    for (int i = 0; i < M; ++i) xq[i] = (long long)xn[i];
    const int64_t ri = row;
    if (t + 1 < p.T) {
      row = p.idx[t + 1];
#pragma unroll
      for (int i = 0; i < M; ++i) xn[i] = Q[row * d + fj[i]];
    }
    // exact per-class partial dots -> shared int64 atomics
    {
      int cur = cls[0];
      long long loc = 0;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (!valid[i]) continue;
        if (cls[i] != cur) {
          atomicAdd(&acc[b3][cur], (unsigned long long)loc);
          loc = 0;
          cur = cls[i];
        }
        loc += xq[i] * z[i];
      }
      if (valid[0]) atomicAdd(&acc[b3][cur], (unsigned long long)loc);
    }
    // this step's draws (independent of the iterate)
    double U[M];
    {
      uint64_t s = rs;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (!valid[i]) continue;
        if (fj[i] == 0) {
          s = xs_step(s);
          ug[par][cls[i]] = uniform_of(s);
        }
        s = xs_step(s);
        U[i] = uniform_of(s);
      }
      rs = jump_tab(rs, jt);
    }
    __syncthreads();
    if (tid == 0)
      for (int c = 0; c < 16; ++c) acc[(t + 2) % 3][c] = 0ull;
    // logits, link derivatives at (phi + dot) and at phi, beta, gamma per class
    double lg[kMaxClasses], ph[kMaxClasses], dl[kMaxClasses], dl0[kMaxClasses];
    for (int c = 0; c < C; ++c) {
      ph[c] = p.phi[ri * C + c];
      lg[c] = ph[c] + __dmul_rn(__ll2double_rn((long long)acc[b3][c]), p.sc);
    }
    if (p.loss == 0) {
      const double yi = p.y[ri];
      dl[0] = lg[0] - yi;
      dl0[0] = ph[0] - yi;
    } else {
      const int li = p.labels[ri];
      for (int c = 0; c < C; ++c) {
        dl[c] = lg[c];
        dl0[c] = ph[c];
      }
      softmax_dl<kMaxClasses>(dl, C, li);
      softmax_dl<kMaxClasses>(dl0, C, li);
    }
    int gc = -1;
    long long gam = 0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (!valid[i]) continue;
      if (cls[i] != gc) {
        gc = cls[i];
        const double beta = __dmul_rn(p.alpha, dl[gc] - dl0[gc]);
        gam = lm_quantize_beta(beta, p.daux, (double)hib, (double)lob, hib, lob, ug[par][gc], &bad);
      }
      long long u = z[i] * (1LL << b) - xq[i] * gam;  // widen_shift - mul_scalar (no int64 overflow for b <= 16)
      u = u > hi2 ? hi2 : u < lo2 ? lo2 : u;
      u = u - h[i];
      u = u > hi2 ? hi2 : u < lo2 ? lo2 : u;
      long long q = u >> b;  // requantize_shift: floor, stochastic round-up by the exact dyadic low / 2^b
      const long long low = u - q * (1LL << b);
      if (low != 0 && U[i] < __dmul_rn((double)low, p2mb)) ++q;
      z[i] = q > hib ? hib : q < lob ? lob : q;
    }
    if (t < p.trace_steps) {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) p.trace[t * D + k0 + i] = z[i];
    }
  }
  if (bad) atomicOr(&bad_s, 1);
  __syncthreads();
  if (tid == 0) *p.bad = bad_s;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (!valid[i]) continue;
    const int k = k0 + i;
    p.w_out[k] = p.w[k] + __dmul_rn((double)z[i], p.dm);  // w~ += to_real(z)
  }
}

template <class Tq>
static cudaError_t lm_stats_t(const LmStatsParams& p, int nblocks, cudaStream_t st) {
  const size_t smem = sizeof(double) * 2 * (size_t)p.d * p.C;
  cudaError_t e = cudaFuncSetAttribute(k_lm_stats<Tq>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_lm_stats<Tq><<<nblocks, kLmThreads, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_lm_stats(const LmStatsParams& p, int nblocks, int code_bytes, cudaStream_t st) {
  if (p.C > kMaxClasses || (size_t)p.d * p.C * 16 > 200 * 1024) return cudaErrorInvalidConfiguration;
  return code_bytes == 1 ? lm_stats_t<int8_t>(p, nblocks, st) : lm_stats_t<int16_t>(p, nblocks, st);
}

template <class Tq, int M>
static cudaError_t lm_inner_m(const LmInnerParams& p, cudaStream_t st) {
  k3_lm<Tq, M><<<1, 256, 0, st>>>(p);
  return cudaGetLastError();
}
template <class Tq>
static cudaError_t lm_inner_t(const LmInnerParams& p, cudaStream_t st) {
  const int D = p.d * p.C;
  if (D <= 256) return lm_inner_m<Tq, 1>(p, st);
  if (D <= 512) return lm_inner_m<Tq, 2>(p, st);
  if (D <= 1024) return lm_inner_m<Tq, 4>(p, st);
  if (D <= 2048) return lm_inner_m<Tq, 8>(p, st);
  return lm_inner_m<Tq, 16>(p, st);
}

cudaError_t launch_lm_inner(const LmInnerParams& p, int code_bytes, cudaStream_t st) {
  if (p.d * p.C > kLmMaxD || p.C > kMaxClasses || p.bits < 2 || p.bits > 16) return cudaErrorInvalidConfiguration;
  return code_bytes == 1 ? lm_inner_t<int8_t>(p, st) : lm_inner_t<int16_t>(p, st);
}

}  // namespace halp
