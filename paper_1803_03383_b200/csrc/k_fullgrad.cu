// k_fullgrad.cu -- K1: fused full-gradient + loss pass over X, streamed from
// HBM with cp.async.bulk (TMA bulk copies) into a shared-memory ring.
//
// Replaces, in one HBM pass, the reference's three passes per epoch:
//   Objective::full_gradient  (two GEMVs per 1024-row block)  proj/src/objectives.cpp:258-311
//   Objective::loss           (a third blocked pass)          proj/src/objectives.cpp:193-223
// g~ = (1/n) sum_i grad f_i(w~) + l2 w~, loss = (1/n) sum_i l_i + (l2/2)|w~|^2.
//
// Reduction order (mirrored by oracle MIRROR mode):
//   * rows are cut into S splits (power of two), split s = rows [s*n/S, (s+1)*n/S);
//     one CTA per split;
//   * row dot x_r . w_c: thread t owns 16-byte feature groups t, t+T1, ...;
//     sequential fma over its features, warp xor-butterfly (16..1), warps
//     summed in order;
//   * gradient column (j,c): sequential fma over the split's rows;
//   * loss: per-row terms summed sequentially over the split's rows;
//   * splits combined by a pairwise tree (k1_split_tree), ranks by the same
//     tree (k_finalize), so the result is independent of the GPU count.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

template <class Tx> struct VecT;
template <> struct VecT<float> { static constexpr int V = 4; };
template <> struct VecT<__nv_bfloat16> { static constexpr int V = 8; };
template <> struct VecT<double> { static constexpr int V = 2; };

// load one 16-byte group from shared memory and upcast exactly
template <class Tx>
__device__ __forceinline__ void load_group(const Tx* p, double* out) {
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  if constexpr (sizeof(Tx) == 4) {
    out[0] = (double)__uint_as_float(raw.x);
    out[1] = (double)__uint_as_float(raw.y);
    out[2] = (double)__uint_as_float(raw.z);
    out[3] = (double)__uint_as_float(raw.w);
  } else if constexpr (sizeof(Tx) == 2) {
    const uint32_t wds[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      out[2 * q] = (double)__uint_as_float(wds[q] << 16);
      out[2 * q + 1] = (double)__uint_as_float(wds[q] & 0xFFFF0000u);
    }
  } else {
    out[0] = __longlong_as_double(((long long)raw.y << 32) | raw.x);
    out[1] = __longlong_as_double(((long long)raw.w << 32) | raw.z);
  }
}

template <class Tx, int NG, int CT, int R, int STAGES>
__global__ void __launch_bounds__(256) k1_fullgrad(FgParams p) {
  constexpr int V = VecT<Tx>::V;
  extern __shared__ __align__(128) unsigned char smem[];
  const int T1 = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = T1 >> 5;
  const int d = p.d, C = p.C, D = d * C, ld = p.ld;
  const size_t stage_bytes = (size_t)R * ld * sizeof(Tx);
  Tx* stages = reinterpret_cast<Tx*>(smem);
  double* w_s = reinterpret_cast<double*>(smem + STAGES * stage_bytes);
  double* red = w_s + D;                 // [NW][R*C]
  double* dl_s = red + NW * R * C;       // [R][C]
  double* lterm = dl_s + R * C;          // [R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(lterm + R);

  const int s = p.split0 + blockIdx.x;
  const int64_t r0 = (int64_t)(((unsigned long long)p.n * (unsigned long long)s) / (unsigned long long)p.S);
  const int64_t r1 = (int64_t)(((unsigned long long)p.n * (unsigned long long)(s + 1)) / (unsigned long long)p.S);
  const int64_t ntile = (r1 - r0 + R - 1) / R;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);

  for (int k = tid; k < D; k += T1) w_s[k] = p.w[k];
  if (tid == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t tile) {
    const int st = (int)(tile % STAGES);
    const int64_t row = r0 + tile * R;
    const int64_t rows = (r1 - row) < R ? (r1 - row) : R;
    const uint32_t bytes = (uint32_t)(rows * ld * sizeof(Tx));
    mbar_expect_tx(&bars[st], bytes);
    bulk_g2s(stages + (size_t)st * R * ld, X + row * ld, bytes, &bars[st]);
  };
  if (tid == 0)
    for (int64_t t = 0; t < ntile && t < STAGES; ++t) issue(t);

  double gacc[NG][V][CT];
#pragma unroll
  for (int k = 0; k < NG; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q)
#pragma unroll
      for (int cc = 0; cc < CT; ++cc) gacc[k][q][cc] = 0.0;
  double la = 0.0;

  for (int64_t i = 0; i < ntile; ++i) {
    const int st = (int)(i % STAGES);
    mbar_wait(&bars[st], (uint32_t)((i / STAGES) & 1));
    const Tx* xs = stages + (size_t)st * R * ld;
    const int64_t rowb = r0 + i * R;
    const int nr = (int)((r1 - rowb) < R ? (r1 - rowb) : R);

    // ---- dot phase: logits of the nr rows for every class ----
    for (int c = 0; c < C; ++c) {
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
      for (int k = 0; k < NG; ++k) {
        const int g = tid + k * T1;
        if (g * V < d) {
          double wv[V];
#pragma unroll
          for (int q = 0; q < V; ++q) wv[q] = (g * V + q < d) ? w_s[c * d + g * V + q] : 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (r < nr) {
              double xv[V];
              load_group<Tx>(xs + (size_t)r * ld + g * V, xv);
#pragma unroll
              for (int q = 0; q < V; ++q)
                if (g * V + q < d) acc[r] = fma(xv[q], wv[q], acc[r]);
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double v = warp_allsum(acc[r]);
        if (lane == 0) red[wid * R * C + r * C + c] = v;
      }
    }
    __syncthreads();
    // the previous stage is now free (everyone finished its gradient phase)
    if (tid == 0 && i >= 1 && i - 1 + STAGES < ntile) issue(i - 1 + STAGES);
    if (tid < nr) {
      double lg[kMaxClasses];
      for (int c = 0; c < C; ++c) {
        double v = red[tid * C + c];
        for (int w2 = 1; w2 < NW; ++w2) v = v + red[w2 * R * C + tid * C + c];
        lg[c] = v;
      }
      const int64_t row = rowb + tid;
      if (p.loss == 0) {
        const double e = lg[0] - p.y[row];
        lterm[tid] = __dmul_rn(__dmul_rn(0.5, e), e);
        dl_s[tid * C] = e;
      } else {
        const int lab = p.labels[row];
        lterm[tid] = softmax_loss(lg, C, lab);
        softmax_dl<kMaxClasses>(lg, C, lab);
        for (int c = 0; c < C; ++c) dl_s[tid * C + c] = lg[c];
      }
    }
    __syncthreads();

    // ---- gradient phase: column accumulators, sequential over rows ----
    for (int r = 0; r < nr; ++r) {
      double dlr[CT];
#pragma unroll
      for (int cc = 0; cc < CT; ++cc) dlr[cc] = (p.c0 + cc < C) ? dl_s[r * C + p.c0 + cc] : 0.0;
#pragma unroll
      for (int k = 0; k < NG; ++k) {
        const int g = tid + k * T1;
        if (g * V < d) {
          double xv[V];
          load_group<Tx>(xs + (size_t)r * ld + g * V, xv);
#pragma unroll
          for (int q = 0; q < V; ++q)
#pragma unroll
            for (int cc = 0; cc < CT; ++cc) gacc[k][q][cc] = fma(dlr[cc], xv[q], gacc[k][q][cc]);
        }
      }
    }
    if (tid == 0 && p.write_loss)
      for (int r = 0; r < nr; ++r) la = la + lterm[r];
  }

  double* out = p.partials + (size_t)blockIdx.x * (D + 1);
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const int g = tid + k * T1;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int j = g * V + q;
      if (j < d)
#pragma unroll
        for (int cc = 0; cc < CT; ++cc)
          if (p.c0 + cc < C) out[(size_t)(p.c0 + cc) * d + j] = gacc[k][q][cc];
    }
  }
  if (tid == 0 && p.write_loss) out[D] = la;
}

// pairwise tree over the splits, in passes: thread (group o, coordinate k)
// combines G = 2^m consecutive splits with a register tree (pairs, then
// pairs of pairs, ...), i.e. one complete subtree of the global pairwise
// tree; the next pass combines the subtree roots the same way.
template <int G>
__global__ void k1_tree_pass(const double* __restrict__ in, int ngroups_out, int D1, double* __restrict__ out) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int k = (int)(id % D1);
  const int o = (int)(id / D1);
  if (o >= ngroups_out) return;
  double v[G];
#pragma unroll
  for (int i = 0; i < G; ++i) v[i] = in[((size_t)o * G + i) * D1 + k];
#pragma unroll
  for (int h = 1; h < G; h *= 2)
#pragma unroll
    for (int i = 0; i < G; i += 2 * h) v[i] = v[i] + v[i + h];
  out[(size_t)o * D1 + k] = v[0];
}

// centering: tree over ranks, g = sum/n + l2 w, |g|, delta, loss (one CTA of 256)
__global__ void __launch_bounds__(256) k_finalize(FinParams p) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int D = p.D, D1 = D + 1;
  __shared__ double red_g[8], red_w[8];
  __shared__ double lsum;
  double ag = 0.0, aw = 0.0;
  for (int k = tid; k < D1; k += 256) {
    double stk[32];
    int cnt = 0;
    for (int r = 0; r < p.G; ++r) {
      double v = p.rank_sums[(size_t)r * D1 + k];
      for (int c = r; c & 1; c >>= 1) v = stk[--cnt] + v;
      stk[cnt++] = v;
    }
    const double tot = stk[0];
    if (k < D) {
      const double wk = p.w[k];
      const double g = tot / (double)p.n + __dmul_rn(p.l2, wk);
      p.g_out[k] = g;
      ag = fma(g, g, ag);
      aw = fma(wk, wk, aw);
    } else {
      lsum = tot;
    }
  }
  ag = warp_allsum(ag);
  aw = warp_allsum(aw);
  if (lane == 0) {
    red_g[wid] = ag;
    red_w[wid] = aw;
  }
  __syncthreads();
  if (tid == 0) {
    double sg = red_g[0], sw = red_w[0];
    for (int w2 = 1; w2 < 8; ++w2) {
      sg = sg + red_g[w2];
      sw = sw + red_w[w2];
    }
    const double gn = sqrt(sg);
    double delta = 0.0;
    if (isfinite(gn) && gn > 0.0) {
      const double span = ldexp(1.0, p.bits - 1) - 1.0;
      const double sc = gn / __dmul_rn(p.mu, span);
      delta = (sc < p.delta_min) ? p.delta_min : sc;
    }
    p.stats[0] = gn;
    p.stats[1] = delta;
    p.stats[2] = lsum / (double)p.n + __dmul_rn(__dmul_rn(0.5, p.l2), sw);
  }
}

// K4: sample indices of one epoch by counter-indexed jump-ahead.
// Draw j of the epoch (j = 0 is t_pick under option II) is the state after
// j+1 steps from state0 (rng.hpp:48-51, optimizers.cpp:418-424).
__global__ void k_samples(uint64_t state0, int64_t total, int opt2, uint64_t T, uint64_t n,
                          const uint64_t* __restrict__ pow_tab, int64_t per_thread, int64_t* __restrict__ idx,
                          int64_t* __restrict__ tpick) {
  const int64_t first = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * per_thread;
  if (first >= total) return;
  uint64_t s = jump_count(state0, (uint64_t)first, pow_tab);
  for (int64_t q = 0; q < per_thread; ++q) {
    const int64_t j = first + q;
    if (j >= total) return;
    s = xs_step(s);
    if (opt2 && j == 0) *tpick = (int64_t)index_of(s, T);
    else idx[j - opt2] = (int64_t)index_of(s, n);
  }
}

// ---------------------------------------------------------------- dispatch
template <class Tx, int NG, int CT>
static cudaError_t launch_fg_t(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  constexpr int R = 2, STAGES = 4;
  if constexpr (NG * VecT<Tx>::V * CT > 64) {
    return cudaErrorInvalidConfiguration;  // never planned (register budget, see choose_plans)
  } else {
  auto kern = k1_fullgrad<Tx, NG, CT, R, STAGES>;
  const size_t smem = fg_smem_bytes(L.ld, (int)sizeof(Tx), p.d * p.C, p.C, L.threads, R, STAGES);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (L.dry) return cudaSuccess;
  kern<<<L.nsplit_local, L.threads, smem, st>>>(p);
  return cudaGetLastError();
  }
}

template <class Tx, int NG>
static cudaError_t launch_fg_ct(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.ct) {
    case 1: return launch_fg_t<Tx, NG, 1>(L, p, st);
    case 2: return launch_fg_t<Tx, NG, 2>(L, p, st);
    case 4: return launch_fg_t<Tx, NG, 4>(L, p, st);
    default: return launch_fg_t<Tx, NG, 8>(L, p, st);
  }
}

template <class Tx>
static cudaError_t launch_fg_dt(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.ng) {
    case 1: return launch_fg_ct<Tx, 1>(L, p, st);
    case 2: return launch_fg_ct<Tx, 2>(L, p, st);
    case 4: return launch_fg_ct<Tx, 4>(L, p, st);
    default: return launch_fg_ct<Tx, 8>(L, p, st);
  }
}

size_t fg_smem_bytes(int ld, int elem, int D, int C, int threads, int R, int stages) {
  size_t b = (size_t)stages * R * ld * elem;
  b += (size_t)D * 8 + (size_t)(threads / 32) * R * C * 8 + (size_t)R * C * 8 + (size_t)R * 8;
  b = (b + 7) / 8 * 8 + stages * 8;
  return b;
}

cudaError_t launch_fullgrad(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if (L.fast == 3) return launch_fullgrad_smx(L, p, st);
  if (L.fast == 4) return launch_fullgrad_stream(L, p, st);
  switch (L.dtype) {
    case 0: return launch_fg_dt<double>(L, p, st);
    case 1: return launch_fg_dt<float>(L, p, st);
    default: return launch_fg_dt<__nv_bfloat16>(L, p, st);
  }
}

cudaError_t launch_split_tree(const double* partials, int nsplit, int D1, double* out, double* scratch,
                              cudaStream_t st) {
  // nsplit is a power of two; each pass folds up to 64 splits
  const double* in = partials;
  int n = nsplit;
  while (n > 1) {
    int g = n >= 64 ? 64 : n;
    const int nout = n / g;
    double* dst = (nout == 1) ? out : (in == scratch ? const_cast<double*>(partials) : scratch);
    const int64_t threads = (int64_t)nout * D1;
    const int blocks = (int)((threads + 255) / 256);
    switch (g) {
      case 64: k1_tree_pass<64><<<blocks, 256, 0, st>>>(in, nout, D1, dst); break;
      case 32: k1_tree_pass<32><<<blocks, 256, 0, st>>>(in, nout, D1, dst); break;
      case 16: k1_tree_pass<16><<<blocks, 256, 0, st>>>(in, nout, D1, dst); break;
      case 8: k1_tree_pass<8><<<blocks, 256, 0, st>>>(in, nout, D1, dst); break;
      case 4: k1_tree_pass<4><<<blocks, 256, 0, st>>>(in, nout, D1, dst); break;
      default: k1_tree_pass<2><<<blocks, 256, 0, st>>>(in, nout, D1, dst); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    in = dst;
    n = nout;
  }
  if (nsplit == 1) return cudaMemcpyAsync(out, partials, sizeof(double) * D1, cudaMemcpyDeviceToDevice, st);
  return cudaSuccess;
}

cudaError_t launch_finalize(const FinParams& p, cudaStream_t st) {
  k_finalize<<<1, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_samples(uint64_t state0, int64_t total, int opt2, uint64_t T, uint64_t n, const uint64_t* pow_tab,
                           int64_t* idx, int64_t* tpick, cudaStream_t st) {
  const int64_t threads = 148 * 256;
  int64_t per = (total + threads - 1) / threads;
  if (per < 16) per = 16;
  const int64_t nthr = (total + per - 1) / per;
  const int blocks = (int)((nthr + 255) / 256);
  k_samples<<<blocks, 256, 0, st>>>(state0, total, opt2, T, n, pow_tab, per, idx, tpick);
  return cudaGetLastError();
}

}  // namespace halp
