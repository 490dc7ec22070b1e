// k_inner.cu -- K3: the b-bit SVRG inner loop of one HALP epoch as ONE
// persistent kernel on one thread-block cluster.
//
// Reference: proj/src/optimizers.cpp:414-442 (z = Q(0), T steps of
//   i = sample.next_index(n); wz = w~ + z;
//   g1 = grad f_i(wz); g2 = grad f_i(w~)            objectives.cpp:225-250
//   u = z - alpha*((g1 - g2) + g~); blowup if !allFinite(u)
//   z = Q(u) with one rounding draw per coordinate   fixed_point.cpp:104-123
// then w~ += z (option I) or the sampled snapshot (option II)).
//
// Layout: the D = d*C flat coordinates (column-major d x C, objectives.hpp:56-58)
// are split over the cluster: thread tau = rank*T3 + tid owns the M
// contiguous coordinates [tau*M, tau*M + M).  w~, g~ and the integer codes
// of z live in registers for the whole epoch; only the sampled row x_i is
// read from memory each step, prefetched two steps ahead in raw form.
//
// Rounding stream: the reference's xorshift64* stream 1, reproduced exactly.
// Coordinate k of step t uses draw  D*(t+1) + k  of the epoch (after the D
// draws of Q(0)); a thread steps its M draws sequentially and jumps D draws
// per step with the GF(2) table of X^D (rng_jump.hpp) held in shared memory.
//
// One cluster barrier per step.  Each warp reduces its partial logits with an
// xor-butterfly reduce-scatter and stores them into every CTA of the cluster
// (DSMEM).  After the barrier EVERY warp redundantly combines the warp
// partials and evaluates the loss derivative (lane-parallel softmax: lane c
// = class c at wz, lane 16+c = at w~), so nothing is broadcast through a
// second barrier.  The non-finite flag of step t is published with the
// partials of step t+1.
//
// Reduction order (mirrored by oracle MIRROR mode): thread partial =
// sequential fma over its coordinates; warp = xor butterfly 16..1; across
// warps, squared loss (C == 1): lane l sums warps l, l+32, ... sequentially,
// then a lane butterfly; softmax (C >= 2): sequential over the warps holding
// the class, in global warp order.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

constexpr int kMaxWarpsPerCluster = 128;

// SPAN2: every warp's 32*M coordinates touch at most two classes (C == 1 or
// 32*M <= d): 4 slots per warp.  Otherwise: 2*C slots per warp (small d).
template <class Tx, int M, bool CL, bool SPAN2>
__global__ void __launch_bounds__(256, 1) k3_inner(InParams p) {
  constexpr int NSLOT = SPAN2 ? 4 : 32;
  __shared__ uint64_t jt[2048];
  extern __shared__ __align__(16) double xbuf_dyn[];  // [2][NGW][NSLOT]
  __shared__ int flagbuf[2][kMaxWarpsPerCluster];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  const uint32_t rank = CL ? cluster_ctarank() : 0u;
  const int NC = CL ? (int)gridDim.x : 1;
  const int NGW = NC * NW;
  const int gw = (int)rank * NW + wid;
  const int d = p.d, C = p.C, D = p.D, ld = p.ld;
  const int64_t k0 = ((int64_t)rank * blockDim.x + tid) * M;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  const double delta = p.delta, alpha = p.alpha, l2 = p.l2, rcp = p.rcp;
  const bool squared = (p.loss == 0);
  const int WC = 32 * M;  // coordinates per warp
  auto XB = [&](int par_, int q_, int slot_) -> double& {
    return xbuf_dyn[((size_t)par_ * NGW + q_) * NSLOT + slot_];
  };

  for (int i = tid; i < 2048; i += blockDim.x) jt[i] = p.jump_tab[i];

  // class of this warp's first coordinate (warp-uniform, SPAN2 split point)
  const int64_t wk0 = (int64_t)gw * WC;
  const int cw0 = (int)(wk0 < D ? wk0 / d : 0);

  // per-lane plan of the cross-warp logit sum (softmax): lane hc (+16 for w~)
  const int hc = lane & 15;
  const int isw = (lane >> 4) & 1;
  int q_first = 0, q_last = -1, slot_first = 0, slot_rest = 0;
  if (!squared && hc < C) {
    q_first = (int)(((int64_t)hc * d) / WC);
    q_last = (int)((((int64_t)hc + 1) * d - 1) / WC);
    if (SPAN2) {
      const int c_of_first = (int)(((int64_t)q_first * WC) / d);
      slot_first = (c_of_first == hc ? 0 : 2) + isw;
      slot_rest = isw;
    } else {
      slot_first = slot_rest = 2 * hc + isw;
    }
  }

  double wt[M], gt[M], up[M], Un[M];
  Tx xa[M], xb[M];
  double code[M], snap[M];  // z codes as exact doubles (|code| <= 2^(bits-1))
  const bool wide = p.hi > 0x1.0p53;
  int cls[M], fj[M];
  bool valid[M];
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int64_t k = k0 + i;
    valid[i] = k < D;
    cls[i] = valid[i] ? (int)(k / d) : 0;
    fj[i] = valid[i] ? (int)(k % d) : 0;
    wt[i] = valid[i] ? p.w[k] : 0.0;
    gt[i] = valid[i] ? p.g[k] : 0.0;
    code[i] = 0.0;
    snap[i] = 0.0;
    up[i] = 0.0;
  }
  const int cA = cls[0];
  int cB = cA;
#pragma unroll
  for (int i = 0; i < M; ++i)
    if (valid[i]) cB = cls[i];
  uint64_t rs = jump_count(p.rstate0, (uint64_t)(k0 < D ? k0 : 0), p.pow_tab);
  {  // uniforms of step 0
    uint64_t s = rs;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      s = xs_step(s);
      Un[i] = uniform_of(s);
    }
  }

  // rows of steps 0 and 1 in flight (raw), the index of step 2 loaded
  const int64_t T = p.T;
  int64_t row0 = p.idx[0];
  int64_t row1 = T > 1 ? p.idx[1] : row0;
  int64_t row2 = T > 2 ? p.idx[2] : row1;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    xa[i] = X[row0 * ld + fj[i]];
    xb[i] = X[row1 * ld + fj[i]];
  }
  double yv = squared ? p.y[row0] : 0.0, ynext = squared ? p.y[row1] : 0.0;
  int lab = squared ? 0 : p.labels[row0], labnext = squared ? 0 : p.labels[row1];

  __syncthreads();
  if (CL) cluster_sync_all();

  int bad_prev = 0;
  for (int64_t t = 0; t <= T; ++t) {
    const bool last = (t == T);
    const int par = (int)(t & 1);
    double xc[M];
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    if (!last) {
      if (t == p.t_pick) {
#pragma unroll
        for (int i = 0; i < M; ++i) snap[i] = code[i];
      }
#pragma unroll
      for (int i = 0; i < M; ++i) {
        xc[i] = to_d<Tx>(xa[i]);
        xa[i] = xb[i];
      }
      if (t + 2 < T) {  // raw prefetch of the row of step t+2
#pragma unroll
        for (int i = 0; i < M; ++i) xb[i] = X[row2 * ld + fj[i]];
      }
      const int cS = SPAN2 ? cw0 : cA;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (!valid[i]) continue;
        const double z = __dmul_rn(code[i], delta);
        const double wz = wt[i] + z;
        if (cls[i] == cS) {
          a0 = fma(xc[i], wz, a0);
          b0 = fma(xc[i], wt[i], b0);
        } else {
          a1 = fma(xc[i], wz, a1);
          b1 = fma(xc[i], wt[i], b1);
        }
      }
    }
    const int anybad = __any_sync(0xffffffffu, bad_prev);
    if constexpr (SPAN2) {
      // warp reduce-scatter of (a0, b0, a1, b1): lanes 0, 8, 16, 24 end with them
      const bool u16 = (lane & 16) != 0;
      const double s0 = (u16 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, u16 ? a0 : a1, 16);
      const double s1 = (u16 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, u16 ? b0 : b1, 16);
      const bool u8 = (lane & 8) != 0;
      double v = (u8 ? s1 : s0) + __shfl_xor_sync(0xffffffffu, u8 ? s0 : s1, 8);
      v = v + __shfl_xor_sync(0xffffffffu, v, 4);
      v = v + __shfl_xor_sync(0xffffffffu, v, 2);
      v = v + __shfl_xor_sync(0xffffffffu, v, 1);
      if ((lane & 7) == 0) {
        const int slot = ((lane >> 4) << 1) | ((lane >> 3) & 1);
        if (CL) {
          for (int r = 0; r < NC; ++r) st_cluster_f64(&XB(par, gw, slot), (uint32_t)r, v);
        } else {
          XB(par, gw, slot) = v;
        }
      }
    } else {
      // 32-slot reduce-scatter (slot 2c = class c at wz, 2c+1 at w~): lane l ends with slot l
      double sl[32];
      const bool v0 = valid[0] && !last;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        double v = 0.0;
        if (v0 && q == 2 * cA) v = a0;
        if (v0 && q == 2 * cA + 1) v = b0;
        if (v0 && cB != cA && q == 2 * cB) v = a1;
        if (v0 && cB != cA && q == 2 * cB + 1) v = b1;
        sl[q] = v;
      }
#pragma unroll
      for (int stp = 0; stp < 5; ++stp) {
        const int h = 16 >> stp;
        const bool up_ = (lane & h) != 0;
#pragma unroll
        for (int q = 0; q < h; ++q) {
          const double send = up_ ? sl[q] : sl[q + h];
          const double keep = up_ ? sl[q + h] : sl[q];
          sl[q] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
      }
      if (lane < 2 * C) {
        if (CL) {
          for (int r = 0; r < NC; ++r) st_cluster_f64(&XB(par, gw, lane), (uint32_t)r, sl[0]);
        } else {
          XB(par, gw, lane) = sl[0];
        }
      }
    }
    if (lane == 1) {
      if (CL) {
        for (int r = 0; r < NC; ++r) st_cluster_s32(&flagbuf[par][gw], (uint32_t)r, anybad);
      } else {
        flagbuf[par][gw] = anybad;
      }
    }
    if (CL) cluster_sync_all();
    else __syncthreads();

    // blowup of step t-1?
    {
      int f = 0;
      for (int q = lane; q < NGW; q += 32) f |= flagbuf[par][q];
      if (__any_sync(0xffffffffu, f)) {
#pragma unroll
        for (int i = 0; i < M; ++i)
          if (valid[i]) p.u_out[k0 + i] = up[i];
        if (rank == 0 && tid == 0) *p.blow_step = (int)(t - 1);
        return;
      }
    }
    if (last) break;
    const double yi = yv;
    const int li = lab;
    row0 = row1;
    row1 = row2;
    yv = ynext;
    lab = labnext;
    if (t + 3 < T) row2 = p.idx[t + 3];
    if (t + 2 < T) {
      if (squared) ynext = p.y[row1];
      else labnext = p.labels[row1];
    }

    // loss derivative at wz (p1) and at w~ (p2) for this thread's classes
    double p1A, p2A, p1B, p2B;
    if (squared) {
      double sa = 0.0, sb = 0.0;
      for (int q = lane; q < NGW; q += 32) {
        sa = sa + XB(par, q, 0);
        sb = sb + XB(par, q, 1);
      }
      // lanes >= NGW hold +0.0: butterfly levels that only add zeros are skipped
      // (the totals then sit in lane 0 and are broadcast)
      for (int o = (NGW >= 32 ? 16 : NGW > 1 ? (1 << (31 - __clz(NGW - 1))) : 0); o >= 1; o >>= 1) {
        sa = sa + __shfl_xor_sync(0xffffffffu, sa, o);
        sb = sb + __shfl_xor_sync(0xffffffffu, sb, o);
      }
      if (NGW < 32) {
        sa = __shfl_sync(0xffffffffu, sa, 0);
        sb = __shfl_sync(0xffffffffu, sb, 0);
      }
      p1A = p1B = sa - yi;
      p2A = p2B = sb - yi;
    } else {
      double lg = 0.0;
      if (hc < C) {
        lg = XB(par, q_first, slot_first);
        for (int q = q_first + 1; q <= q_last; ++q) lg = lg + XB(par, q, slot_rest);
      }
      const bool act = hc < C;
      double mx = act ? lg : -INFINITY;
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const double e = act ? hexp(lg - mx) : 0.0;
      const int base = lane & 16;
      double s = __shfl_sync(0xffffffffu, e, base);  // sequential sum (mirror order)
      for (int c = 1; c < C; ++c) s = s + __shfl_sync(0xffffffffu, e, base + c);
      double pr = e / s;
      if (hc == li) pr = pr - 1.0;
      p1A = __shfl_sync(0xffffffffu, pr, cA);
      p2A = __shfl_sync(0xffffffffu, pr, 16 + cA);
      p1B = __shfl_sync(0xffffffffu, pr, cB);
      p2B = __shfl_sync(0xffffffffu, pr, 16 + cB);
    }

    // ---- element-wise update + stochastic rounding (branch-free) ----
    bool bad = false, slow_any = false;
    bool slow[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const bool inA = cls[i] == cA;
      const double p1 = inA ? p1A : p1B, p2 = inA ? p2A : p2B;
      const double z = __dmul_rn(code[i], delta);
      const double wz = wt[i] + z;
      const double g1 = __dmul_rn(p1, xc[i]) + __dmul_rn(l2, wz);
      const double g2 = __dmul_rn(p2, xc[i]) + __dmul_rn(l2, wt[i]);
      const double u = z - __dmul_rn(alpha, (g1 - g2) + gt[i]);
      up[i] = u;
      bad |= valid[i] && !isfinite(u);
      code[i] = quantize_fast(u, delta, rcp, p.hi, p.lo, Un[i], slow[i]);
      slow_any |= valid[i] && slow[i];
    }
    if (slow_any || wide || rcp == 0.0) {  // IEEE-division path for the rare operands
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i] && (slow[i] || wide || rcp == 0.0))
          code[i] = (double)quantize_code(up[i], delta, p.hi, p.lo, p.maxc, p.minc, Un[i]);
    }
    rs = jump_tab(rs, jt);
    {  // uniforms of the next step, off the critical path
      uint64_t s = rs;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        s = xs_step(s);
        Un[i] = uniform_of(s);
      }
    }
    bad_prev = bad ? 1 : 0;
    if (t < p.trace_steps) {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) p.trace[t * D + k0 + i] = __double2ll_rn(code[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (!valid[i]) continue;
    const double zc = p.t_pick >= 0 ? snap[i] : code[i];
    p.w_out[k0 + i] = wt[i] + __dmul_rn(zc, delta);
    p.codes_out[k0 + i] = __double2ll_rn(code[i]);
  }
}

template <class Tx, int M, bool SPAN2>
static cudaError_t launch_in_t(const InLaunch& L, const InParams& p, cudaStream_t st) {
  if (L.ctas * L.threads / 32 > kMaxWarpsPerCluster) return cudaErrorInvalidConfiguration;
  const size_t smem = sizeof(double) * 2 * (size_t)(L.ctas * L.threads / 32) * (SPAN2 ? 4 : 32);
  if (L.ctas == 1) {
    auto kern = k3_inner<Tx, M, false, SPAN2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<1, L.threads, smem, st>>>(p);
    return cudaGetLastError();
  }
  auto kern = k3_inner<Tx, M, true, SPAN2>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.ctas);
  cfg.blockDim = dim3(L.threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <class Tx, int M>
static cudaError_t launch_in_span(const InLaunch& L, const InParams& p, cudaStream_t st) {
  if (p.C == 1 || 32 * M <= p.d) return launch_in_t<Tx, M, true>(L, p, st);
  return launch_in_t<Tx, M, false>(L, p, st);
}

template <class Tx>
static cudaError_t launch_in_dt(const InLaunch& L, const InParams& p, cudaStream_t st) {
  switch (L.per) {
    case 1: return launch_in_span<Tx, 1>(L, p, st);
    case 2: return launch_in_span<Tx, 2>(L, p, st);
    case 4: return launch_in_span<Tx, 4>(L, p, st);
    default: return launch_in_span<Tx, 8>(L, p, st);
  }
}

cudaError_t launch_inner(const InLaunch& L, const InParams& p, cudaStream_t st) {
  switch (L.dtype) {
    case 0: return launch_in_dt<double>(L, p, st);
    case 1: return launch_in_dt<float>(L, p, st);
    default: return launch_in_dt<__nv_bfloat16>(L, p, st);
  }
}

}  // namespace halp
