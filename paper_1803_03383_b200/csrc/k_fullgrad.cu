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

// Fast path for C <= 2 classes: the iterate lives in registers, rows are
// zero-padded to whole 16-byte groups (so only the group index is tested),
// R rows are reduced at once with a warp reduce-scatter, and the
// per-row finishing work runs on different warps.  Same floating-point order
// as k1_fullgrad (and as the oracle's MIRROR mode).
template <int NV>
__device__ __forceinline__ void reduce_scatter_n(double (&v)[NV], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int off = 16 >> st;
    constexpr int dummy = 0;
    (void)dummy;
    const int cur = NV >> st;
    if (cur > 1) {
      const int h = cur >> 1;
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double send = up ? v[i] : v[i + h];
        const double keep = up ? v[i + h] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    } else {
      v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
}

template <class Tx, int NG, int CC, int R, int STAGES>
__global__ void __launch_bounds__(256, 2) k1_fast(FgParams p) {
  constexpr int V = VecT<Tx>::V;
  constexpr int NV = R * CC;  // slots per warp (power of two <= 32)
  constexpr int LG = NV <= 1 ? 0 : NV <= 2 ? 1 : NV <= 4 ? 2 : NV <= 8 ? 3 : NV <= 16 ? 4 : 5;
  extern __shared__ __align__(128) unsigned char smem[];
  const int T1 = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = T1 >> 5;
  const int d = p.d, D = d * CC, ld = p.ld;
  const int ngroups = (d + V - 1) / V;
  const size_t stage_elems = (size_t)R * ld;
  Tx* stages = reinterpret_cast<Tx*>(smem);
  double* red = reinterpret_cast<double*>(smem + STAGES * stage_elems * sizeof(Tx));  // [2][NW][NV]
  double* dl_s = red + 2 * NW * NV;                                                    // [2][R][CC]
  double* lterm = dl_s + 2 * NV;                                                       // [2][R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(lterm + 2 * R);

  const int s = p.split0 + blockIdx.x;
  const int64_t r0 = (int64_t)(((unsigned long long)p.n * (unsigned long long)s) / (unsigned long long)p.S);
  const int64_t r1 = (int64_t)(((unsigned long long)p.n * (unsigned long long)(s + 1)) / (unsigned long long)p.S);
  const int64_t ntile = (r1 - r0 + R - 1) / R;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);

  double wr[NG][V][CC];
#pragma unroll
  for (int k = 0; k < NG; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q)
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const int j = (tid + k * T1) * V + q;
        wr[k][q][c] = j < d ? p.w[c * d + j] : 0.0;
      }
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
    bulk_g2s(stages + (size_t)st * stage_elems, X + row * ld, bytes, &bars[st]);
  };
  if (tid == 0)
    for (int64_t t = 0; t < ntile && t < STAGES; ++t) issue(t);

  // dot phase of tile i: per-warp slot sums into red[i & 1]
  auto dot_tile = [&](int64_t i) {
    const int st = (int)(i % STAGES);
    mbar_wait(&bars[st], (uint32_t)((i / STAGES) & 1));
    const Tx* xs = stages + (size_t)st * stage_elems;
    const int nr = (int)((r1 - (r0 + i * R)) < R ? (r1 - (r0 + i * R)) : R);
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const int g = tid + k * T1;
      if (g < ngroups) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < nr) {
            double xv[V];
            load_group<Tx>(xs + (size_t)r * ld + g * V, xv);
#pragma unroll
            for (int q = 0; q < V; ++q)
#pragma unroll
              for (int c = 0; c < CC; ++c) acc[r * CC + c] = fma(xv[q], wr[k][q][c], acc[r * CC + c]);
          }
        }
      }
    }
    reduce_scatter_n<NV>(acc, lane);
    if ((lane & ((32 >> LG) - 1)) == 0) red[(i & 1) * NW * NV + wid * NV + (lane >> (5 - LG))] = acc[0];
  };

  double gacc[NG][V][CC];
#pragma unroll
  for (int k = 0; k < NG; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q)
#pragma unroll
      for (int c = 0; c < CC; ++c) gacc[k][q][c] = 0.0;
  double la = 0.0;

  // finisher targets (lane 0 of warp r % NW owns row r of a tile): prefetched y / label
  double ypre[(R + 7) / 8 + 1];
  int lpre[(R + 7) / 8 + 1];
  auto prefetch_targets = [&](int64_t i) {
    if (lane == 0 && i < ntile) {
      int slot = 0;
      for (int r = wid; r < R; r += NW, ++slot) {
        const int64_t row = r0 + i * R + r;
        if (row < r1) {
          if (p.loss == 0) ypre[slot] = p.y[row];
          else lpre[slot] = p.labels[row];
        }
      }
    }
  };

  prefetch_targets(0);
  dot_tile(0);
  for (int64_t i = 0; i < ntile; ++i) {
    __syncthreads();  // red[i&1] complete; grad(i-1) done everywhere; dl[i&1] free
    // stage of tile i-1 is free: refill it
    if (tid == 0 && i >= 1 && i - 1 + STAGES < ntile) issue(i - 1 + STAGES);
    const int64_t rowb = r0 + i * R;
    const int nr = (int)((r1 - rowb) < R ? (r1 - rowb) : R);
    // finishers: logits -> loss term and loss derivative of tile i
    if (lane == 0) {
      int slot = 0;
      for (int r = wid; r < nr; r += NW, ++slot) {
        double lg[CC];
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          const double* rb = red + (i & 1) * NW * NV;
          double v = rb[r * CC + c];
          for (int w2 = 1; w2 < NW; ++w2) v = v + rb[w2 * NV + r * CC + c];
          lg[c] = v;
        }
        double* dls = dl_s + (i & 1) * NV;
        if (p.loss == 0) {
          const double e = lg[0] - ypre[slot];
          lterm[(i & 1) * R + r] = __dmul_rn(__dmul_rn(0.5, e), e);
          dls[r * CC] = e;
        } else {
          const int lab = lpre[slot];
          lterm[(i & 1) * R + r] = softmax_loss(lg, CC, lab);
          softmax_dl<CC>(lg, CC, lab);
#pragma unroll
          for (int c = 0; c < CC; ++c) dls[r * CC + c] = lg[c];
        }
      }
    }
    prefetch_targets(i + 1);
    // dot phase of the next tile overlaps the finishers
    if (i + 1 < ntile) dot_tile(i + 1);
    __syncthreads();  // dl[i&1] ready
    // gradient phase of tile i, sequential over its rows
    const Tx* xs = stages + (size_t)(i % STAGES) * stage_elems;
    const double* dls = dl_s + (i & 1) * NV;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr) {
        double dlr[CC];
#pragma unroll
        for (int c = 0; c < CC; ++c) dlr[c] = dls[r * CC + c];
#pragma unroll
        for (int k = 0; k < NG; ++k) {
          const int g = tid + k * T1;
          if (g < ngroups) {
            double xv[V];
            load_group<Tx>(xs + (size_t)r * ld + g * V, xv);
#pragma unroll
            for (int q = 0; q < V; ++q)
#pragma unroll
              for (int c = 0; c < CC; ++c) gacc[k][q][c] = fma(dlr[c], xv[q], gacc[k][q][c]);
          }
        }
      }
    }
    if (tid == 0 && p.write_loss)
      for (int r = 0; r < nr; ++r) la = la + lterm[(i & 1) * R + r];
  }

  double* out = p.partials + (size_t)blockIdx.x * (D + 1);
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const int g = tid + k * T1;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int j = g * V + q;
      if (g < ngroups && j < d)
#pragma unroll
        for (int c = 0; c < CC; ++c) out[(size_t)c * d + j] = gacc[k][q][c];
    }
  }
  if (tid == 0 && p.write_loss) out[D] = la;
}

// Register-tile variant: each thread converts its R x (NG*V) slice of a tile
// ONCE into fp64 registers and uses it for both the dot and the gradient
// phase; full tiles run without per-row / per-group predicates.  Same
// floating-point order as k1_fullgrad / k1_fast (oracle MIRROR mode).
template <class Tx, int NG, int CC, int R, int STAGES, bool FULLG, int TB>
__global__ void __launch_bounds__(TB, TB <= 128 ? 3 : 1) k1_reg(FgParams p) {
  constexpr int V = VecT<Tx>::V;
  constexpr int NV = R * CC;
  constexpr int LG = NV <= 1 ? 0 : NV <= 2 ? 1 : NV <= 4 ? 2 : NV <= 8 ? 3 : NV <= 16 ? 4 : 5;
  extern __shared__ __align__(128) unsigned char smem[];
  const int T1 = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = T1 >> 5;
  const int d = p.d, D = d * CC, ld = p.ld;
  const int ngroups = (d + V - 1) / V;
  const size_t stage_elems = (size_t)R * ld;
  Tx* stages = reinterpret_cast<Tx*>(smem);
  double* red = reinterpret_cast<double*>(smem + STAGES * stage_elems * sizeof(Tx));  // [2][NW][NV]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * NW * NV);
  double* ysm = reinterpret_cast<double*>(bars + STAGES);  // targets of the split

  const int s = p.split0 + blockIdx.x;
  const int64_t r0 = (int64_t)(((unsigned long long)p.n * (unsigned long long)s) / (unsigned long long)p.S);
  const int64_t r1 = (int64_t)(((unsigned long long)p.n * (unsigned long long)(s + 1)) / (unsigned long long)p.S);
  const int64_t ntile = (r1 - r0 + R - 1) / R;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  for (int64_t q = tid; q < r1 - r0; q += T1)
    ysm[q] = p.loss == 0 ? p.y[r0 + q] : (double)p.labels[r0 + q];

  double wr[NG][V][CC];
#pragma unroll
  for (int k = 0; k < NG; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q)
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const int j = (tid + k * T1) * V + q;
        wr[k][q][c] = j < d ? p.w[c * d + j] : 0.0;
      }
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
    bulk_g2s(stages + (size_t)st * stage_elems, X + row * ld, bytes, &bars[st]);
  };
  if (tid == 0)
    for (int64_t t = 0; t < ntile && t < STAGES; ++t) issue(t);

  double gacc[NG][V][CC];
#pragma unroll
  for (int k = 0; k < NG; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q)
#pragma unroll
      for (int c = 0; c < CC; ++c) gacc[k][q][c] = 0.0;
  double la = 0.0;
  bool gval[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) gval[k] = FULLG || (tid + k * T1 < ngroups);
  // every warp evaluates the loss derivatives itself: lane (fr, fc) = (row, class)
  const int fr = lane / CC, fc = lane % CC;

  for (int64_t i = 0; i < ntile; ++i) {
    const int st = (int)(i % STAGES);
    const int64_t rowb = r0 + i * R;
    const int nr = (int)((r1 - rowb) < R ? (r1 - rowb) : R);
    const bool act = (lane < NV) && (fr < nr);
    const double tgt = act ? ysm[rowb - r0 + fr] : 0.0;
    mbar_wait(&bars[st], (uint32_t)((i / STAGES) & 1));
    const Tx* xs = stages + (size_t)st * stage_elems;
    double xr[R][NG][V];
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool rv = (r < nr);
#pragma unroll
      for (int k = 0; k < NG; ++k) {
        if (rv && gval[k]) {
          load_group<Tx>(xs + (size_t)r * ld + (tid + k * T1) * V, xr[r][k]);
        } else {
#pragma unroll
          for (int q = 0; q < V; ++q) xr[r][k][q] = 0.0;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < NG; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q)
#pragma unroll
          for (int c = 0; c < CC; ++c) acc[r * CC + c] = fma(xr[r][k][q], wr[k][q][c], acc[r * CC + c]);
    reduce_scatter_n<NV>(acc, lane);
    double* rb = red + (size_t)(i & 1) * NW * NV;
    if ((lane & ((32 >> LG) - 1)) == 0) rb[wid * NV + (lane >> (5 - LG))] = acc[0];
    __syncthreads();
    // x of this tile now lives in registers: its stage can be refilled
    if (tid == 0 && i + STAGES < ntile) issue(i + STAGES);

    // logit of (fr, fc): warps summed in order (same in every warp)
    double lg = 0.0;
    if (lane < NV) {
      // all loads first (independent), then the in-order chain of adds
      lg = rb[lane];
      for (int w2 = 1; w2 < NW; ++w2) lg = lg + rb[w2 * NV + lane];
    }
    double pr, lt = 0.0;
    if (p.loss == 0) {
      pr = lg - tgt;
      lt = __dmul_rn(__dmul_rn(0.5, pr), pr);
    } else {
      const int lab = (int)tgt;
      const int base = (fr * CC) & 31;
      double mx = 0.0;
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const double v = __shfl_sync(0xffffffffu, lg, (base + c) & 31);
        mx = c == 0 ? v : (v > mx ? v : mx);
      }
      const double e = hexp(lg - mx);
      double ssum = __shfl_sync(0xffffffffu, e, base);
#pragma unroll
      for (int c = 1; c < CC; ++c) ssum = ssum + __shfl_sync(0xffffffffu, e, (base + c) & 31);
      const double lab_logit = __shfl_sync(0xffffffffu, lg, (base + lab) & 31);
      pr = e / ssum;
      if (fc == lab) pr = pr - 1.0;
      if (wid == 0 && fc == 0) lt = (mx + hlog(ssum)) - lab_logit;
    }
    double dlr[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) dlr[v] = __shfl_sync(0xffffffffu, pr, v);
    if (wid == 0 && p.write_loss) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = __shfl_sync(0xffffffffu, lt, r * CC);
        if (r < nr) la = la + t;
      }
    }
    // rows beyond nr: skipped
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr) {
#pragma unroll
        for (int k = 0; k < NG; ++k)
#pragma unroll
          for (int q = 0; q < V; ++q)
#pragma unroll
            for (int c = 0; c < CC; ++c) gacc[k][q][c] = fma(dlr[r * CC + c], xr[r][k][q], gacc[k][q][c]);
      }
    }
  }

  double* out = p.partials + (size_t)blockIdx.x * (D + 1);
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    const int g = tid + k * T1;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int j = g * V + q;
      if (g < ngroups && j < d)
#pragma unroll
        for (int c = 0; c < CC; ++c) out[(size_t)c * d + j] = gacc[k][q][c];
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
size_t fast_smem_bytes(int ld, int elem, int threads, int R, int CC, int stages) {
  size_t b = (size_t)stages * R * ld * elem;
  b += 2 * ((size_t)(threads / 32) * R * CC * 8 + (size_t)R * CC * 8 + (size_t)R * 8);
  return (b + 7) / 8 * 8 + stages * 8;
}

template <class Tx, int NG, int CC, int R, int STAGES>
static cudaError_t launch_fast_t(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  auto kern = k1_fast<Tx, NG, CC, R, STAGES>;
  const size_t smem = fast_smem_bytes(L.ld, (int)sizeof(Tx), L.threads, R, CC, STAGES);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<L.nsplit_local, L.threads, smem, st>>>(p);
  return cudaGetLastError();
}

// fast-path shapes: (NG, R, STAGES); R rows per tile, STAGES-deep bulk-copy ring
template <class Tx, int CC>
static cudaError_t launch_fast_cc(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.ng * 1000 + L.rows * 10 + L.stages) {
    case 1086: return launch_fast_t<Tx, 1, CC, 8, 6>(L, p, st);
    case 1046: return launch_fast_t<Tx, 1, CC, 4, 6>(L, p, st);
    case 1026: return launch_fast_t<Tx, 1, CC, 2, 6>(L, p, st);
    case 1016: return launch_fast_t<Tx, 1, CC, 1, 6>(L, p, st);
    case 2046: return launch_fast_t<Tx, 2, CC, 4, 6>(L, p, st);
    case 2026: return launch_fast_t<Tx, 2, CC, 2, 6>(L, p, st);
    case 2016: return launch_fast_t<Tx, 2, CC, 1, 6>(L, p, st);
    case 4026: return launch_fast_t<Tx, 4, CC, 2, 6>(L, p, st);
    case 4016: return launch_fast_t<Tx, 4, CC, 1, 6>(L, p, st);
    case 4013: return launch_fast_t<Tx, 4, CC, 1, 3>(L, p, st);
    case 4023: return launch_fast_t<Tx, 4, CC, 2, 3>(L, p, st);
    case 8013: return launch_fast_t<Tx, 8, CC, 1, 3>(L, p, st);
    case 8016: return launch_fast_t<Tx, 8, CC, 1, 6>(L, p, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

template <class Tx, int NG, int CC, int R, int STAGES, int TB>
static cudaError_t launch_reg_tb(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  const size_t smem = (size_t)STAGES * R * L.ld * sizeof(Tx) + 2 * (size_t)(L.threads / 32) * R * CC * 8 +
                      STAGES * 8 + 8 * (size_t)((p.n + p.S - 1) / p.S + 1);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  const bool fullg = ((p.d + VecT<Tx>::V - 1) / VecT<Tx>::V) == NG * L.threads;
  cudaError_t e;
  if (fullg) {
    auto kern = k1_reg<Tx, NG, CC, R, STAGES, true, TB>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<L.nsplit_local, L.threads, smem, st>>>(p);
  } else {
    auto kern = k1_reg<Tx, NG, CC, R, STAGES, false, TB>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<L.nsplit_local, L.threads, smem, st>>>(p);
  }
  return cudaGetLastError();
}

template <class Tx, int NG, int CC, int R, int STAGES>
static cudaError_t launch_reg_t(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if (L.threads <= 128) return launch_reg_tb<Tx, NG, CC, R, STAGES, 128>(L, p, st);
  return launch_reg_tb<Tx, NG, CC, R, STAGES, 512>(L, p, st);
}

template <class Tx, int CC>
static cudaError_t launch_reg_cc(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.ng * 1000 + L.rows * 10 + L.stages) {
    case 1084: return launch_reg_t<Tx, 1, CC, 8, 4>(L, p, st);
    case 1044: return launch_reg_t<Tx, 1, CC, 4, 4>(L, p, st);
    case 1024: return launch_reg_t<Tx, 1, CC, 2, 4>(L, p, st);
    case 2044: return launch_reg_t<Tx, 2, CC, 4, 4>(L, p, st);
    case 2024: return launch_reg_t<Tx, 2, CC, 2, 4>(L, p, st);
    case 2014: return launch_reg_t<Tx, 2, CC, 1, 4>(L, p, st);
    case 4024: return launch_reg_t<Tx, 4, CC, 2, 4>(L, p, st);
    case 4014: return launch_reg_t<Tx, 4, CC, 1, 4>(L, p, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

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
  if (L.fast == 2) {
    switch (L.dtype * 10 + p.C) {
      case 1: return launch_reg_cc<double, 1>(L, p, st);
      case 2: return launch_reg_cc<double, 2>(L, p, st);
      case 11: return launch_reg_cc<float, 1>(L, p, st);
      case 12: return launch_reg_cc<float, 2>(L, p, st);
      case 21: return launch_reg_cc<__nv_bfloat16, 1>(L, p, st);
      case 22: return launch_reg_cc<__nv_bfloat16, 2>(L, p, st);
      default: return cudaErrorInvalidConfiguration;
    }
  }
  if (L.fast) {
    const int cc = p.C;
    switch (L.dtype * 10 + cc) {
      case 1: return launch_fast_cc<double, 1>(L, p, st);
      case 2: return launch_fast_cc<double, 2>(L, p, st);
      case 11: return launch_fast_cc<float, 1>(L, p, st);
      case 12: return launch_fast_cc<float, 2>(L, p, st);
      case 21: return launch_fast_cc<__nv_bfloat16, 1>(L, p, st);
      case 22: return launch_fast_cc<__nv_bfloat16, 2>(L, p, st);
      default: return cudaErrorInvalidConfiguration;
    }
  }
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
