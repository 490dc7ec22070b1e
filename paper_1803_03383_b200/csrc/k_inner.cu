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
// read from memory each step (prefetched one step ahead).
//
// Rounding stream: the reference's xorshift64* stream 1, reproduced exactly.
// Coordinate k of step t uses draw  D*(t+1) + k  of the epoch (after the D
// draws of Q(0)); a thread steps its M draws sequentially and jumps D draws
// per step with the GF(2) table of X^D (rng_jump.hpp) held in shared memory.
//
// Per step, the 2C logits (at wz and at w~; C = 1 for squared loss) are
// reduced over the cluster: thread partials (sequential fma) -> warp
// reduce-scatter (xor 16..1) -> warps summed in order -> CTAs summed in order
// through distributed shared memory, one cluster barrier per step.  The
// non-finite flag of step t rides in the reduction of step t+1.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

// xor-butterfly reduce-scatter of NSP slots over a warp: lane l ends with
// the warp sum of slot (l >> (5 - log2 NSP)).  Every addition pairs the same
// operands as the plain butterfly, so each slot's bits equal warp_allsum's.
template <int NSP>
__device__ __forceinline__ double warp_reduce_scatter(double (&v)[NSP], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int off = 16 >> st;
    const int cur = NSP >> st;
    if (cur > 1) {
      const int h = cur >> 1;
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double send = up ? v[i] : v[i + h];
        const double keep = up ? v[i + h] : v[i];
        const double recv = __shfl_xor_sync(0xffffffffu, send, off);
        v[i] = keep + recv;
      }
    } else {
      v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

template <int NSP> struct Log2 { static constexpr int v = NSP <= 1 ? 0 : 1 + Log2<NSP / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

template <class Tx, int M, int NSP, bool CL>
__global__ void __launch_bounds__(256, 1) k3_inner(InParams p) {
  __shared__ uint64_t jt[2048];
  __shared__ double red[8][NSP];
  __shared__ double xbuf[2][16][NSP];
  __shared__ double fin[NSP];
  __shared__ double dla[kMaxClasses + 1], dlb[kMaxClasses + 1];
  __shared__ double flag_s;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  const uint32_t rank = CL ? cluster_ctarank() : 0u;
  const int NC = CL ? (int)gridDim.x : 1;
  const int d = p.d, C = p.C, D = p.D, ld = p.ld;
  const int nslots = 2 * C + 1;
  const int64_t k0 = ((int64_t)rank * blockDim.x + tid) * M;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  const double delta = p.delta, alpha = p.alpha, l2 = p.l2;
  const bool squared = (p.loss == 0);

  for (int i = tid; i < 2048; i += blockDim.x) jt[i] = p.jump_tab[i];

  double wt[M], gt[M], xc[M], xn[M], up[M];
  long long code[M], snap[M];
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
    code[i] = 0;
    snap[i] = 0;
    up[i] = 0.0;
    xn[i] = 0.0;
  }
  const int cA = cls[0];
  int cB = cA;
#pragma unroll
  for (int i = 0; i < M; ++i)
    if (valid[i]) cB = cls[i];
  uint64_t rs = jump_count(p.rstate0, (uint64_t)(k0 < D ? k0 : 0), p.pow_tab);

  int64_t row_next = p.idx[0];
#pragma unroll
  for (int i = 0; i < M; ++i)
    if (valid[i]) xn[i] = to_d<Tx>(X[row_next * ld + fj[i]]);
  int64_t row_next2 = p.T > 1 ? p.idx[1] : 0;

  __syncthreads();
  if (CL) cluster_sync_all();

  double bad_prev = 0.0;
  for (int64_t t = 0; t <= p.T; ++t) {
    const bool last = (t == p.T);
    double sl[NSP];
#pragma unroll
    for (int s = 0; s < NSP; ++s) sl[s] = 0.0;
    int64_t row = 0;
    if (!last) {
      if (t == p.t_pick) {
#pragma unroll
        for (int i = 0; i < M; ++i) snap[i] = code[i];
      }
      row = row_next;
#pragma unroll
      for (int i = 0; i < M; ++i) xc[i] = xn[i];
      if (t + 1 < p.T) {
        row_next = row_next2;
#pragma unroll
        for (int i = 0; i < M; ++i)
          if (valid[i]) xn[i] = to_d<Tx>(X[row_next * ld + fj[i]]);
        if (t + 2 < p.T) row_next2 = p.idx[t + 2];
      }
      double aA = 0.0, bA = 0.0, aB = 0.0, bB = 0.0;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (!valid[i]) continue;
        const double z = __dmul_rn(__ll2double_rn(code[i]), delta);
        const double wz = wt[i] + z;
        if (cls[i] == cA) {
          aA = fma(xc[i], wz, aA);
          bA = fma(xc[i], wt[i], bA);
        } else {
          aB = fma(xc[i], wz, aB);
          bB = fma(xc[i], wt[i], bB);
        }
      }
#pragma unroll
      for (int s = 0; s < NSP; ++s) {
        double v = 0.0;
        if (s == cA) v = aA;
        if (cB != cA && s == cB) v = aB;
        if (s == C + cA) v = bA;
        if (cB != cA && s == C + cB) v = bB;
        sl[s] = v;
      }
    }
#pragma unroll
    for (int s = 0; s < NSP; ++s)
      if (s == 2 * C) sl[s] = bad_prev;

    const double ws = warp_reduce_scatter<NSP>(sl, lane);
    constexpr int SH = 5 - Log2<NSP>::v;
    if ((lane & ((1 << SH) - 1)) == 0) red[wid][lane >> SH] = ws;
    __syncthreads();
    if (wid == 0) {
      if (lane < nslots) {
        double v = red[0][lane];
        for (int w2 = 1; w2 < NW; ++w2) v = v + red[w2][lane];
        if (CL) {
          for (int r = 0; r < NC; ++r) st_cluster_f64(&xbuf[t & 1][rank][lane], (uint32_t)r, v);
        } else {
          fin[lane] = v;
        }
      }
    }
    if (CL) {
      cluster_sync_all();
      if (wid == 0 && lane < nslots) {
        double v = xbuf[t & 1][0][lane];
        for (int r = 1; r < NC; ++r) v = v + xbuf[t & 1][r][lane];
        fin[lane] = v;
      }
    }
    if (wid == 0) {
      __syncwarp();
      if (lane == 0) {
        flag_s = fin[2 * C];
        if (!last) {
          if (squared) {
            const double yi = p.y[row];
            dla[0] = fin[0] - yi;
            dlb[0] = fin[1] - yi;
          } else {
            double lg[kMaxClasses];
            for (int c = 0; c < C; ++c) lg[c] = fin[c];
            softmax_dl<kMaxClasses>(lg, C, p.labels[row]);
            for (int c = 0; c < C; ++c) dla[c] = lg[c];
          }
        }
      } else if (lane == 1 && !last && !squared) {
        double lg[kMaxClasses];
        for (int c = 0; c < C; ++c) lg[c] = fin[C + c];
        softmax_dl<kMaxClasses>(lg, C, p.labels[row]);
        for (int c = 0; c < C; ++c) dlb[c] = lg[c];
      }
    }
    __syncthreads();
    if (flag_s > 0.0) {
      // step t-1 produced a non-finite update: hand its u to the host
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) p.u_out[k0 + i] = up[i];
      if (rank == 0 && tid == 0) *p.blow_step = (int)(t - 1);
      return;
    }
    if (last) break;

    // ---- element-wise update + stochastic rounding ----
    bool bad = false;
    uint64_t s = rs;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      s = xs_step(s);
      const double U = uniform_of(s);
      if (!valid[i]) continue;
      const double z = __dmul_rn(__ll2double_rn(code[i]), delta);
      const double wz = wt[i] + z;
      const double p1 = dla[cls[i]], p2 = dlb[cls[i]];
      const double g1 = __dmul_rn(p1, xc[i]) + __dmul_rn(l2, wz);
      const double g2 = __dmul_rn(p2, xc[i]) + __dmul_rn(l2, wt[i]);
      const double u = z - __dmul_rn(alpha, (g1 - g2) + gt[i]);
      up[i] = u;
      if (!isfinite(u)) bad = true;
      code[i] = quantize_code(u, delta, p.hi, p.lo, p.maxc, p.minc, U);
    }
    rs = jump_tab(rs, jt);
    bad_prev = bad ? 1.0 : 0.0;
    if (t < p.trace_steps) {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) p.trace[t * D + k0 + i] = code[i];
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (!valid[i]) continue;
    const long long zc = p.t_pick >= 0 ? snap[i] : code[i];
    p.w_out[k0 + i] = wt[i] + __dmul_rn(__ll2double_rn(zc), delta);
    p.codes_out[k0 + i] = code[i];
  }
}

template <class Tx, int M, int NSP>
static cudaError_t launch_in_t(const InLaunch& L, const InParams& p, cudaStream_t st) {
  if (L.ctas == 1) {
    k3_inner<Tx, M, NSP, false><<<1, L.threads, 0, st>>>(p);
    return cudaGetLastError();
  }
  auto kern = k3_inner<Tx, M, NSP, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.ctas);
  cfg.blockDim = dim3(L.threads);
  cfg.dynamicSmemBytes = 0;
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
static cudaError_t launch_in_nsp(const InLaunch& L, const InParams& p, cudaStream_t st) {
  switch (L.nslot_pow2) {
    case 4: return launch_in_t<Tx, M, 4>(L, p, st);
    case 8: return launch_in_t<Tx, M, 8>(L, p, st);
    case 16: return launch_in_t<Tx, M, 16>(L, p, st);
    default: return launch_in_t<Tx, M, 32>(L, p, st);
  }
}

template <class Tx>
static cudaError_t launch_in_dt(const InLaunch& L, const InParams& p, cudaStream_t st) {
  switch (L.per) {
    case 1: return launch_in_nsp<Tx, 1>(L, p, st);
    case 2: return launch_in_nsp<Tx, 2>(L, p, st);
    case 4: return launch_in_nsp<Tx, 4>(L, p, st);
    default: return launch_in_nsp<Tx, 8>(L, p, st);
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
