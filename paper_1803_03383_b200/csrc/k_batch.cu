// k_batch.cu -- K5: many independent HALP problems (BASELINE config C5, and the
// reference's grid / conditioning-sweep workloads, harness.cpp:379-518, which
// run one lpopt::run_prepared per configuration sequentially).  One CTA of
// four warps owns one problem and runs the WHOLE lpopt::run_halp
// (optimizers.cpp:387-459) for it in a single launch: every epoch's full
// gradient + loss, centering, the T-step inner loop, the Recorder rows
// (pass, loss, grad norm, delta, FNV-1a iterate hash, optimizers.cpp:104-167,
// 218-227), divergence / blow-up and convergence.  Problems are independent:
// no collective, shard them across GPUs.
//
// Floating-point order = the single-problem kernels', so the oracle's MIRROR
// mode (plan of halp_plan_for(n, d, 1)) checks K5 bit for bit:
//   * full gradient: the K1 split tree -- S splits (power of two), warp w
//     owns the aligned subtree of splits [w*S/4, (w+1)*S/4) and merges them
//     in order with a binary-counter stack; the 4 warp roots are combined as
//     the top of the pairwise tree.  Row dot: lane l owns the 16-byte groups
//     l, l+32, ... (K1 with fg_threads = 32, which is what the plan picks
//     for d <= 128 fp32); gradient column = sequential fma over the split's rows.
//   * finalize: k_finalize's 256-strided order for |g| and |w|.
//   * inner loop: K3's single-CTA order (KIND 0) with 128 threads, M = D/128
//     coordinates per thread: thread partial, warp reduce-scatter butterfly,
//     the 4 warp records combined by every warp (lane l reads warp l, lane
//     butterfly) -- halp_batch_plan reports {1 CTA, 128 threads, M}.
// Squared loss only (the C5 / sweep workloads); d*C <= 256.
//
// Inner-loop latency (the whole cost of a problem, one chain per step):
//   * the sample stream does not depend on the iterate, so every thread runs
//     it kP steps ahead and keeps the sampled rows (its M features + y) in a
//     register ring: the HBM round trip of a row is off the serial chain;
//   * all four warps work: one exchange through shared memory + one barrier
//     per step (the blow-up flag of the previous step rides in the record);
//   * the X^D jump table of the rounding stream lives in shared memory.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

constexpr int kBatchMaxM = 4;     // D <= 256 over 64 threads
constexpr int kP = 4;             // sample-row prefetch distance (steps)
constexpr int kBatchMaxLev = 16;  // splits per warp <= 2^15

template <class Tx> struct BVec;
template <> struct BVec<float> { static constexpr int V = 4; };
template <> struct BVec<double> { static constexpr int V = 2; };
template <> struct BVec<__nv_bfloat16> { static constexpr int V = 8; };

template <class Tx>
__device__ __forceinline__ void load_group_g(const Tx* p, double* out) {
  const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p));
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

template <class Tx>
__device__ __forceinline__ Tx zero_raw() {
  Tx z;
  memset(&z, 0, sizeof z);
  return z;
}

__device__ __forceinline__ uint64_t fnv1a_doubles(const double* v, int len) {
  uint64_t h = 1469598103934665603ULL;
  for (int k = 0; k < len; ++k) {
    const uint64_t b = (uint64_t)__double_as_longlong(v[k]);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      h ^= (b >> (8 * q)) & 0xFF;
      h *= 1099511628211ULL;
    }
  }
  return h;
}

// NG groups of V features per lane (NG*V*32 >= d)
template <class Tx, int NG, int M, int NWP>
__global__ void __launch_bounds__(32 * NWP, 4) k5_batch(BatchParams p) {
  static_assert(NWP == 2 || NWP == 4, "2 or 4 warps per problem");
  constexpr int NTH = 32 * NWP;
  constexpr int V = BVec<Tx>::V;
  const int prob = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int d = p.d, D = d, ld = p.ld;
  const int64_t n = p.n;
  const int S = p.splits;
  // own dataset per problem, or one dataset shared by all (grid searches: x_rows_per_prob = 0)
  const Tx* X = reinterpret_cast<const Tx*>(p.X) + (size_t)prob * p.x_rows_per_prob * ld;
  const double* y = p.y + (size_t)prob * p.x_rows_per_prob;

  __shared__ double w_s[264], g_s[264], wsum[4][257];  // iterate, g~, warp subtree roots (+loss)
  __shared__ double stats[4];
  __shared__ int sh_stop, sh_blew;
  __shared__ uint64_t jt[2048];                 // X^D jump table of the rounding stream
  __shared__ __align__(32) double rec[2][4][4];  // [parity][warp]: a-sum, b-sum, blow-up flag of step t-1

  const double alpha = p.alpha[prob], mu = p.mu[prob], dmin = p.delta_min[prob], divl = p.div_limit[prob];
  const int bits = p.bits[prob], epochs = p.epochs[prob], opt2 = p.option[prob];
  const int64_t T = p.T[prob];
  const double l2 = p.l2;
  const double hi = bits == 64 ? 9223372036854775807.0 : (double)((1LL << (bits - 1)) - 1);
  const double lo = bits == 64 ? -9223372036854775808.0 : (double)(-(1LL << (bits - 1)));
  const long long maxc = bits == 64 ? 0x7FFFFFFFFFFFFFFFLL : (1LL << (bits - 1)) - 1;
  const long long minc = bits == 64 ? (long long)0x8000000000000000ULL : -(1LL << (bits - 1));
  const bool wide = hi > 0x1.0p53;
  double* rows = p.rows + (size_t)prob * p.max_rows * 5;
  uint64_t* rhash = p.rhash + (size_t)prob * p.max_rows;
  const uint64_t t_start = globaltimer_ns();

  for (int k = tid; k < 264; k += NTH) w_s[k] = (k < D && p.init) ? p.init[(size_t)prob * D + k] : 0.0;
  if (tid == 0) {
    sh_stop = 0;
    sh_blew = 0;
  }
  __syncthreads();

  // RNG states (seeding as rng.hpp:29-32, done on the host: p.seed holds the
  // stream-0 / stream-1 initial states interleaved)
  uint64_t s_sample = p.seed[2 * prob];   // stream 0 state (thread-uniform)
  const uint64_t s_round0 = p.seed[2 * prob + 1];
  for (int i = tid; i < 2048; i += NTH) jt[i] = p.jump_tab[i];

  int nrow = 0;
  int status = 0;  // 0 ok, 1 converged, 2 diverged
  int64_t steps = 0;
  double next_pass = 0.0;
  const double metric_every = p.metric_every[prob];

  auto boundary = [&](double pass, const double* wv, double loss, double gn, double delta, bool forced) -> bool {
    // Recorder::boundary (optimizers.cpp:125-152), lane 0 of warp 0; returns "bad"
    const bool bad = !(isfinite(loss) && isfinite(gn)) || loss > divl || gn > divl;
    const bool due = forced || metric_every <= 0.0 || pass + 1e-9 >= next_pass;
    if ((due || bad) && nrow < p.max_rows) {
      double* r = rows + (size_t)nrow * 5;
      r[0] = pass;
      r[1] = (double)(globaltimer_ns() - t_start) * 1e-9;
      r[2] = loss;
      r[3] = gn;
      r[4] = delta;
      rhash[nrow] = fnv1a_doubles(wv, D);
      ++nrow;
      if (metric_every > 0.0) next_pass = pass + metric_every;
    }
    return bad;
  };

  // ---- full gradient + loss in the K1 order; result -> g_s, stats ----
  auto full_pass = [&]() {
    // warp w: splits [w*S/NWP, (w+1)*S/NWP), binary-counter tree
    const int sw = S / NWP;
    double stk[kBatchMaxLev][NG * V + 1];
    int cnt = 0;
    for (int si = 0; si < sw; ++si) {
      const int s = wid * sw + si;
      const int64_t r0 = (int64_t)(((unsigned long long)n * s) / S);
      const int64_t r1 = (int64_t)(((unsigned long long)n * (s + 1)) / S);
      double acc[NG * V + 1];
#pragma unroll
      for (int q = 0; q < NG * V + 1; ++q) acc[q] = 0.0;
      for (int64_t r = r0; r < r1; ++r) {
        double xv[NG][V];
        double dot = 0.0;
#pragma unroll
        for (int k = 0; k < NG; ++k) {
          const int g = lane + 32 * k;
          if (g * V < d) {
            load_group_g<Tx>(X + r * ld + g * V, xv[k]);
#pragma unroll
            for (int q = 0; q < V; ++q) dot = fma(xv[k][q], w_s[g * V + q], dot);
          } else {
#pragma unroll
            for (int q = 0; q < V; ++q) xv[k][q] = 0.0;
          }
        }
        dot = warp_allsum(dot);
        const double e = dot - y[r];
        acc[NG * V] = acc[NG * V] + __dmul_rn(__dmul_rn(0.5, e), e);
#pragma unroll
        for (int k = 0; k < NG; ++k)
#pragma unroll
          for (int q = 0; q < V; ++q) acc[k * V + q] = fma(e, xv[k][q], acc[k * V + q]);
      }
      // merge split si into the stack (pairwise tree over the warp's splits)
      int c = si;
      while (c & 1) {
        --cnt;
#pragma unroll
        for (int q = 0; q < NG * V + 1; ++q) acc[q] = stk[cnt][q] + acc[q];
        c >>= 1;
      }
#pragma unroll
      for (int q = 0; q < NG * V + 1; ++q) stk[cnt][q] = acc[q];
      ++cnt;
    }
#pragma unroll
    for (int k = 0; k < NG; ++k)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const int j = (lane + 32 * k) * V + q;
        if (j < D) wsum[wid][j] = stk[0][k * V + q];
      }
    if (lane == 0) wsum[wid][256] = stk[0][NG * V];
    __syncthreads();
    // top of the tree: ((w0 + w1) + (w2 + w3)) or (w0 + w1); g = sum/n + l2 w; norms (k_finalize order)
    double ag = 0.0, aw = 0.0;
    for (int k = tid; k < 256; k += NTH) {
      if (k < D) {
        const double tot = NWP == 4 ? (wsum[0][k] + wsum[1][k]) + (wsum[2][k] + wsum[3][k]) : wsum[0][k] + wsum[1][k];
        const double g = tot / (double)n + __dmul_rn(l2, w_s[k]);
        g_s[k] = g;
      }
    }
    __syncthreads();
    if (wid == 0) {
      // 256 virtual threads: v[t] = g[t]^2 (t < D), 8 virtual warps of 32 in order
      double sg = 0.0, sw2 = 0.0;
      for (int vw = 0; vw < 8; ++vw) {
        const int t = vw * 32 + lane;
        ag = t < D ? fma(g_s[t], g_s[t], 0.0) : 0.0;
        aw = t < D ? fma(w_s[t], w_s[t], 0.0) : 0.0;
        ag = warp_allsum(ag);
        aw = warp_allsum(aw);
        sg = vw == 0 ? ag : sg + ag;
        sw2 = vw == 0 ? aw : sw2 + aw;
      }
      if (lane == 0) {
        const double ltot = NWP == 4 ? (wsum[0][256] + wsum[1][256]) + (wsum[2][256] + wsum[3][256])
                                     : wsum[0][256] + wsum[1][256];
        const double gn = sqrt(sg);
        double delta = 0.0;
        if (isfinite(gn) && gn > 0.0) {
          const double span = ldexp(1.0, bits - 1) - 1.0;
          const double sc = gn / __dmul_rn(mu, span);
          delta = (sc < dmin) ? dmin : sc;
        }
        stats[0] = gn;
        stats[1] = delta;
        stats[2] = ltot / (double)n + __dmul_rn(__dmul_rn(0.5, l2), sw2);
      }
    }
    __syncthreads();
  };

  // inner-loop state: thread tid owns coordinates [tid*M, tid*M + M)
  double wt[M], gtl[M], l2w[M], code[M], snap[M], up[M];
  bool valid[M];
  const int k0 = tid * M;
#pragma unroll
  for (int i = 0; i < M; ++i) valid[i] = (k0 + i) < D;
  const bool vecx = (M * sizeof(Tx) == 8 || M * sizeof(Tx) == 16) && (ld % M == 0);
  // rounding stream after Q(0) of epoch 0, at this thread's first draw
  uint64_t rs = jump_count(s_round0, (uint64_t)(D + k0), p.pow_tab);

  bool converged = false;
  for (int k = 0; k < epochs && !converged; ++k) {
    full_pass();
    const double gn = stats[0], delta = stats[1], loss = stats[2];
    if (tid == 0) {
      const bool bad = boundary((double)steps / (double)n, w_s, loss, gn, delta, k == 0 || gn == 0.0);
      if (bad) {
        status = 2;
        sh_stop = 2;
      } else if (gn == 0.0) {
        status = 1;
        sh_stop = 1;
      } else if (!(isfinite(delta) && delta > 0.0)) {
        status = 3;
        sh_stop = 3;
      }
    }
    __syncthreads();
    if (sh_stop) {
      converged = sh_stop == 1;
      break;
    }
    const double rcp = 1.0 / delta;
    const bool fast_q = isfinite(rcp) && rcp != 0.0 && !wide;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      wt[i] = valid[i] ? w_s[k0 + i] : 0.0;
      gtl[i] = valid[i] ? g_s[k0 + i] : 0.0;
      l2w[i] = __dmul_rn(l2, wt[i]);
      code[i] = 0.0;
      snap[i] = 0.0;
      up[i] = 0.0;
    }
    int64_t t_pick = -1;
    if (opt2) {
      s_sample = xs_step(s_sample);
      t_pick = (int64_t)index_of(s_sample, (uint64_t)T);
    }
    // sample-row ring: slot j holds the row of steps j, j + kP, ... (raw x + y)
    Tx xr[kP][M];
    double yr[kP];
    auto issue = [&](Tx (&dst)[M], double& ydst) {
      s_sample = xs_step(s_sample);
      const int64_t row = (int64_t)index_of(s_sample, (uint64_t)n);
      const Tx* xp = X + row * ld + k0;
      if (vecx && M > 1) {
        if constexpr (M * sizeof(Tx) == 16) {
          const uint4 r = __ldg(reinterpret_cast<const uint4*>(xp));
          const Tx* q = reinterpret_cast<const Tx*>(&r);
#pragma unroll
          for (int i = 0; i < M; ++i) dst[i] = q[i];
        } else if constexpr (M * sizeof(Tx) == 8) {
          const uint2 r = __ldg(reinterpret_cast<const uint2*>(xp));
          const Tx* q = reinterpret_cast<const Tx*>(&r);
#pragma unroll
          for (int i = 0; i < M; ++i) dst[i] = q[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i) dst[i] = valid[i] ? __ldg(xp + i) : zero_raw<Tx>();
      }
      ydst = __ldg(y + row);
    };
#pragma unroll
    for (int j = 0; j < kP; ++j)
      if (j < T) issue(xr[j], yr[j]);
    int bad_prev = 0;
    int64_t blow = -1;
    for (int64_t t0 = 0; t0 < T && blow < 0; t0 += kP) {
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        const int64_t t = t0 + j;
        if (t >= T) break;
        const int par = (int)(t & 1);
        double xc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xc[i] = to_d<Tx>(xr[j][i]);
        const double yi = yr[j];
        if (t + kP < T) issue(xr[j], yr[j]);  // the row of step t + kP
        if (t == t_pick) {
#pragma unroll
          for (int i = 0; i < M; ++i) snap[i] = code[i];
        }
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
          if (!valid[i]) continue;
          const double z = __dmul_rn(code[i], delta);
          a = fma(xc[i], wt[i] + z, a);
          b = fma(xc[i], wt[i], b);
        }
        // warp reduce-scatter: a on lanes 0..15, b on lanes 16..31 (K3 KIND 0)
        const bool u16 = (lane & 16) != 0;
        double v = (u16 ? b : a) + __shfl_xor_sync(0xffffffffu, u16 ? a : b, 16);
        v = v + __shfl_xor_sync(0xffffffffu, v, 8);
        v = v + __shfl_xor_sync(0xffffffffu, v, 4);
        v = v + __shfl_xor_sync(0xffffffffu, v, 2);
        v = v + __shfl_xor_sync(0xffffffffu, v, 1);
        const double vp = __shfl_xor_sync(0xffffffffu, v, 16);
        const int flag = __any_sync(0xffffffffu, bad_prev);
        if (lane == 0)
          *reinterpret_cast<double4*>(&rec[par][wid][0]) = make_double4(v, vp, flag ? 1.0 : 0.0, 0.0);
        // rounding draws of this step, independent of the exchange
        double U[M];
        {
          uint64_t sr = rs;
#pragma unroll
          for (int i = 0; i < M; ++i) {
            sr = xs_step(sr);
            U[i] = uniform_of(sr);
          }
          rs = jump_tab(rs, jt);
        }
        __syncthreads();
        // lane l < NWP holds warp l's record; lane butterfly over the NWP records
        double sa = 0.0, sb = 0.0, fl = 0.0;
        if (lane < NWP) {
          const double4 r = *reinterpret_cast<const double4*>(&rec[par][lane][0]);
          sa = sa + r.x;
          sb = sb + r.y;
          fl = r.z;
        }
        if (__any_sync(0xffffffffu, fl != 0.0)) {
          blow = t - 1;  // step t-1's update was non-finite; up[] still holds it
          break;
        }
        if (NWP == 4) {
          sa = sa + __shfl_xor_sync(0xffffffffu, sa, 2);
          sb = sb + __shfl_xor_sync(0xffffffffu, sb, 2);
        }
        sa = sa + __shfl_xor_sync(0xffffffffu, sa, 1);
        sb = sb + __shfl_xor_sync(0xffffffffu, sb, 1);
        sa = __shfl_sync(0xffffffffu, sa, 0);
        sb = __shfl_sync(0xffffffffu, sb, 0);
        const double e1 = sa - yi, e2 = sb - yi;
        bool bad = false, slow_any = false;
        bool slow[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          const double z = __dmul_rn(code[i], delta);
          const double wz = wt[i] + z;
          const double g1 = __dmul_rn(e1, xc[i]) + __dmul_rn(l2, wz);
          const double g2 = __dmul_rn(e2, xc[i]) + l2w[i];
          const double u = z - __dmul_rn(alpha, (g1 - g2) + gtl[i]);
          up[i] = u;
          bad |= valid[i] && !isfinite(u);
          slow[i] = false;
          if (fast_q) {
            code[i] = quantize_fast(u, delta, rcp, hi, lo, U[i], slow[i]);
            slow_any |= valid[i] && slow[i];
          } else {
            code[i] = (double)quantize_code(u, delta, hi, lo, maxc, minc, U[i]);
          }
        }
        if (slow_any) {
#pragma unroll
          for (int i = 0; i < M; ++i)
            if (valid[i] && slow[i]) code[i] = (double)quantize_code(up[i], delta, hi, lo, maxc, minc, U[i]);
        }
        bad_prev = bad ? 1 : 0;
      }
    }
    // the last step's finiteness (no further exchange carries it)
    if (blow < 0 && __syncthreads_or(bad_prev)) blow = T - 1;
    if (blow >= 0) {
      // Recorder::blowup: row (inf, inf, delta) hashed over u (optimizers.cpp:156-160)
      __syncthreads();
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) g_s[k0 + i] = up[i];
      __syncthreads();
      if (tid == 0) {
        boundary((double)(steps + blow + 1) / (double)n, g_s, INFINITY, INFINITY, delta, true);
        status = 2;
        sh_stop = 2;
        sh_blew = 1;
        for (int q = 0; q < D; ++q) p.w_out[(size_t)prob * D + q] = g_s[q];
      }
    } else {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) w_s[k0 + i] = wt[i] + __dmul_rn(t_pick >= 0 ? snap[i] : code[i], delta);
      // next epoch: skip its Q(0) draws
      rs = jump_tab(rs, jt);
    }
    __syncthreads();
    if (sh_stop) break;
    steps += T;
  }
  if (!sh_stop && !converged) {
    full_pass();
    if (tid == 0) {
      const bool bad = boundary((double)steps / (double)n, w_s, stats[2], stats[0], stats[1], true);
      if (bad) status = 2;
      else if (stats[0] == 0.0) status = 1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    p.rows_n[prob] = nrow;
    p.status[prob] = status;
    p.steps[prob] = (status >= 2) ? 0 : steps;
  }
  if (!sh_blew)
    for (int q = tid; q < D; q += NTH) p.w_out[(size_t)prob * D + q] = w_s[q];
}

// ---------------------------------------------------------------------------
// k5_batch_w1: ONE WARP per problem (one warp per CTA), the default plan.
// Same floating-point order as k5_batch for the full pass (one warp walks all
// S splits through the binary-counter stack = the same pairwise tree) and the
// single-warp K3 order for the inner loop (plan {1 CTA, 32 threads, M = D/32}):
// lane partials, the warp butterfly (reduce-scatter: a on lanes 0..15, b on
// 16..31).  Per problem this issues about a third of the 4-warp kernel's
// instructions (one sample-index chain, one jump per M draws, no barrier), and
// the full pass computes kR rows' dots at once (their butterflies interleave)
// before accumulating them in row order.
constexpr int kR = 4;  // rows per full-pass chunk

template <class Tx, int NG, int M>
__global__ void __launch_bounds__(32, 8) k5_batch_w1(BatchParams p) {
  constexpr int V = BVec<Tx>::V;
  constexpr int NF = NG * V;  // features per lane in the full pass
  const int prob = blockIdx.x;
  const int lane = threadIdx.x;
  const int d = p.d, D = d, ld = p.ld;
  const int64_t n = p.n;
  const int S = p.splits;
  const Tx* X = reinterpret_cast<const Tx*>(p.X) + (size_t)prob * p.x_rows_per_prob * ld;
  const double* y = p.y + (size_t)prob * p.x_rows_per_prob;

  __shared__ double w_s[264], g_s[264];
  __shared__ uint64_t jt[2048];

  const double alpha = p.alpha[prob], mu = p.mu[prob], dmin = p.delta_min[prob], divl = p.div_limit[prob];
  const int bits = p.bits[prob], epochs = p.epochs[prob], opt2 = p.option[prob];
  const int64_t T = p.T[prob];
  const double l2 = p.l2;
  const double hi = bits == 64 ? 9223372036854775807.0 : (double)((1LL << (bits - 1)) - 1);
  const double lo = bits == 64 ? -9223372036854775808.0 : (double)(-(1LL << (bits - 1)));
  const long long maxc = bits == 64 ? 0x7FFFFFFFFFFFFFFFLL : (1LL << (bits - 1)) - 1;
  const long long minc = bits == 64 ? (long long)0x8000000000000000ULL : -(1LL << (bits - 1));
  const bool wide = hi > 0x1.0p53;
  double* rows = p.rows + (size_t)prob * p.max_rows * 5;
  uint64_t* rhash = p.rhash + (size_t)prob * p.max_rows;
  const uint64_t t_start = globaltimer_ns();

  for (int k = lane; k < 264; k += 32) w_s[k] = (k < D && p.init) ? p.init[(size_t)prob * D + k] : 0.0;
  for (int i = lane; i < 2048; i += 32) jt[i] = p.jump_tab[i];
  __syncwarp();
  uint64_t s_sample = p.seed[2 * prob];
  const uint64_t s_round0 = p.seed[2 * prob + 1];

  int nrow = 0, status = 0;
  int64_t steps = 0;
  double next_pass = 0.0;
  const double metric_every = p.metric_every[prob];
  double st_gn = 0.0, st_delta = 0.0, st_loss = 0.0;

  auto boundary = [&](double pass, const double* wv, double loss, double gn, double delta, bool forced) -> bool {
    const bool bad = !(isfinite(loss) && isfinite(gn)) || loss > divl || gn > divl;
    const bool due = forced || metric_every <= 0.0 || pass + 1e-9 >= next_pass;
    if ((due || bad) && nrow < p.max_rows) {
      if (lane == 0) {
        double* r = rows + (size_t)nrow * 5;
        r[0] = pass;
        r[1] = (double)(globaltimer_ns() - t_start) * 1e-9;
        r[2] = loss;
        r[3] = gn;
        r[4] = delta;
        rhash[nrow] = fnv1a_doubles(wv, D);
      }
      ++nrow;
      if (metric_every > 0.0) next_pass = pass + metric_every;
    }
    return bad;
  };

  // full gradient + loss (K1 order), g -> g_s, stats in registers (all lanes)
  auto full_pass = [&]() {
    double stk[kBatchMaxLev][NF + 1];
    int cnt = 0;
    for (int s = 0; s < S; ++s) {
      const int64_t r0 = (int64_t)(((unsigned long long)n * s) / S);
      const int64_t r1 = (int64_t)(((unsigned long long)n * (s + 1)) / S);
      double acc[NF + 1];
#pragma unroll
      for (int q = 0; q < NF + 1; ++q) acc[q] = 0.0;
      for (int64_t rb = r0; rb < r1; rb += kR) {
        double xv[kR][NF];
        double e[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const int64_t r = rb + u;
          double dot = 0.0;
#pragma unroll
          for (int k = 0; k < NG; ++k) {
            const int g = lane + 32 * k;
            if (r < r1 && g * V < d) {
              load_group_g<Tx>(X + r * ld + g * V, &xv[u][k * V]);
#pragma unroll
              for (int q = 0; q < V; ++q) dot = fma(xv[u][k * V + q], w_s[g * V + q], dot);
            } else {
#pragma unroll
              for (int q = 0; q < V; ++q) xv[u][k * V + q] = 0.0;
            }
          }
          e[u] = dot;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
          for (int u = 0; u < kR; ++u) e[u] = e[u] + __shfl_xor_sync(0xffffffffu, e[u], o);
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const int64_t r = rb + u;
          if (r >= r1) break;
          const double ee = e[u] - y[r];
          acc[NF] = acc[NF] + __dmul_rn(__dmul_rn(0.5, ee), ee);
#pragma unroll
          for (int q = 0; q < NF; ++q) acc[q] = fma(ee, xv[u][q], acc[q]);
        }
      }
      int c = s;
      while (c & 1) {
        --cnt;
#pragma unroll
        for (int q = 0; q < NF + 1; ++q) acc[q] = stk[cnt][q] + acc[q];
        c >>= 1;
      }
#pragma unroll
      for (int q = 0; q < NF + 1; ++q) stk[cnt][q] = acc[q];
      ++cnt;
    }
    // root of the pairwise tree -> g = sum/n + l2 w (k_finalize), loss
#pragma unroll
    for (int k = 0; k < NG; ++k)
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const int j = (lane + 32 * k) * V + q;
        if (j < D) g_s[j] = stk[0][k * V + q] / (double)n + __dmul_rn(l2, w_s[j]);
      }
    __syncwarp();
    double sg = 0.0, sw2 = 0.0;
    for (int vw = 0; vw < 8; ++vw) {
      const int t = vw * 32 + lane;
      double ag = t < D ? fma(g_s[t], g_s[t], 0.0) : 0.0;
      double aw = t < D ? fma(w_s[t], w_s[t], 0.0) : 0.0;
      ag = warp_allsum(ag);
      aw = warp_allsum(aw);
      sg = vw == 0 ? ag : sg + ag;
      sw2 = vw == 0 ? aw : sw2 + aw;
    }
    const double ltot = __shfl_sync(0xffffffffu, stk[0][NF], 0);
    st_gn = sqrt(sg);
    st_delta = 0.0;
    if (isfinite(st_gn) && st_gn > 0.0) {
      const double span = ldexp(1.0, bits - 1) - 1.0;
      const double sc = st_gn / __dmul_rn(mu, span);
      st_delta = (sc < dmin) ? dmin : sc;
    }
    st_loss = ltot / (double)n + __dmul_rn(__dmul_rn(0.5, l2), sw2);
  };

  double wt[M], gtl[M], l2w[M], code[M], snap[M], up[M];
  bool valid[M];
  const int k0 = lane * M;
#pragma unroll
  for (int i = 0; i < M; ++i) valid[i] = (k0 + i) < D;
  const bool vecx = (M * sizeof(Tx) == 8 || M * sizeof(Tx) == 16) && (ld % M == 0);
  uint64_t rs = jump_count(s_round0, (uint64_t)(D + k0), p.pow_tab);
  bool blew = false;

  for (int k = 0; k < epochs; ++k) {
    full_pass();
    const double gn = st_gn, delta = st_delta, loss = st_loss;
    const bool bad = boundary((double)steps / (double)n, w_s, loss, gn, delta, k == 0 || gn == 0.0);
    if (bad) { status = 2; break; }
    if (gn == 0.0) { status = 1; break; }
    if (!(isfinite(delta) && delta > 0.0)) { status = 3; break; }
    const double rcp = 1.0 / delta;
    const bool fast_q = isfinite(rcp) && rcp != 0.0 && !wide;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      wt[i] = valid[i] ? w_s[k0 + i] : 0.0;
      gtl[i] = valid[i] ? g_s[k0 + i] : 0.0;
      l2w[i] = __dmul_rn(l2, wt[i]);
      code[i] = 0.0;
      snap[i] = 0.0;
      up[i] = 0.0;
    }
    int64_t t_pick = -1;
    if (opt2) {
      s_sample = xs_step(s_sample);
      t_pick = (int64_t)index_of(s_sample, (uint64_t)T);
    }
    Tx xr[kP][M];
    double yr[kP];
    auto issue = [&](Tx (&dst)[M], double& ydst) {
      s_sample = xs_step(s_sample);
      const int64_t row = (int64_t)index_of(s_sample, (uint64_t)n);
      const Tx* xp = X + row * ld + k0;
      if (vecx && M > 1) {
        if constexpr (M * sizeof(Tx) == 16) {
          const uint4 r = __ldg(reinterpret_cast<const uint4*>(xp));
          const Tx* q = reinterpret_cast<const Tx*>(&r);
#pragma unroll
          for (int i = 0; i < M; ++i) dst[i] = q[i];
        } else if constexpr (M * sizeof(Tx) == 8) {
          const uint2 r = __ldg(reinterpret_cast<const uint2*>(xp));
          const Tx* q = reinterpret_cast<const Tx*>(&r);
#pragma unroll
          for (int i = 0; i < M; ++i) dst[i] = q[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i) dst[i] = valid[i] ? __ldg(xp + i) : zero_raw<Tx>();
      }
      ydst = __ldg(y + row);
    };
#pragma unroll
    for (int j = 0; j < kP; ++j)
      if (j < T) issue(xr[j], yr[j]);
    int64_t blow = -1;
    for (int64_t t0 = 0; t0 < T && blow < 0; t0 += kP) {
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        const int64_t t = t0 + j;
        if (t >= T) break;
        double xc[M];
#pragma unroll
        for (int i = 0; i < M; ++i) xc[i] = to_d<Tx>(xr[j][i]);
        const double yi = yr[j];
        if (t + kP < T) issue(xr[j], yr[j]);
        if (t == t_pick) {
#pragma unroll
          for (int i = 0; i < M; ++i) snap[i] = code[i];
        }
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
          if (!valid[i]) continue;
          const double z = __dmul_rn(code[i], delta);
          a = fma(xc[i], wt[i] + z, a);
          b = fma(xc[i], wt[i], b);
        }
        const bool u16 = (lane & 16) != 0;
        double v = (u16 ? b : a) + __shfl_xor_sync(0xffffffffu, u16 ? a : b, 16);
        v = v + __shfl_xor_sync(0xffffffffu, v, 8);
        v = v + __shfl_xor_sync(0xffffffffu, v, 4);
        v = v + __shfl_xor_sync(0xffffffffu, v, 2);
        v = v + __shfl_xor_sync(0xffffffffu, v, 1);
        double U[M];
        {
          uint64_t sr = rs;
#pragma unroll
          for (int i = 0; i < M; ++i) {
            sr = xs_step(sr);
            U[i] = uniform_of(sr);
          }
          rs = jump_tab(rs, jt);
        }
        const double e1 = __shfl_sync(0xffffffffu, v, 0) - yi;
        const double e2 = __shfl_sync(0xffffffffu, v, 16) - yi;
        bool bad = false, slow_any = false;
        bool slow[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          const double z = __dmul_rn(code[i], delta);
          const double wz = wt[i] + z;
          const double g1 = __dmul_rn(e1, xc[i]) + __dmul_rn(l2, wz);
          const double g2 = __dmul_rn(e2, xc[i]) + l2w[i];
          const double u = z - __dmul_rn(alpha, (g1 - g2) + gtl[i]);
          up[i] = u;
          bad |= valid[i] && !isfinite(u);
          slow[i] = false;
          if (fast_q) {
            code[i] = quantize_fast(u, delta, rcp, hi, lo, U[i], slow[i]);
            slow_any |= valid[i] && slow[i];
          } else {
            code[i] = (double)quantize_code(u, delta, hi, lo, maxc, minc, U[i]);
          }
        }
        if (__any_sync(0xffffffffu, slow_any)) {
#pragma unroll
          for (int i = 0; i < M; ++i)
            if (valid[i] && slow[i]) code[i] = (double)quantize_code(up[i], delta, hi, lo, maxc, minc, U[i]);
        }
        if (__any_sync(0xffffffffu, bad)) {
          blow = t;
          break;
        }
      }
    }
    if (blow >= 0) {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) g_s[k0 + i] = up[i];
      __syncwarp();
      boundary((double)(steps + blow + 1) / (double)n, g_s, INFINITY, INFINITY, delta, true);
      status = 2;
      blew = true;
      for (int q = lane; q < D; q += 32) p.w_out[(size_t)prob * D + q] = g_s[q];
      break;
    }
#pragma unroll
    for (int i = 0; i < M; ++i)
      if (valid[i]) w_s[k0 + i] = wt[i] + __dmul_rn(t_pick >= 0 ? snap[i] : code[i], delta);
    __syncwarp();
    rs = jump_tab(rs, jt);
    steps += T;
  }
  if (status == 0) {
    full_pass();
    const bool bad = boundary((double)steps / (double)n, w_s, st_loss, st_gn, st_delta, true);
    if (bad) status = 2;
    else if (st_gn == 0.0) status = 1;
  }
  if (lane == 0) {
    p.rows_n[prob] = nrow;
    p.status[prob] = status;
    p.steps[prob] = (status >= 2) ? 0 : steps;
  }
  if (!blew)
    for (int q = lane; q < D; q += 32) p.w_out[(size_t)prob * D + q] = w_s[q];
}

template <class Tx, int NG>
static cudaError_t launch_b_ng(const BatchParams& p, cudaStream_t st) {
  if (batch_warps_per_problem(p.d) == 1) {
    const int M = (p.d + 31) / 32;
    if (M <= 1) k5_batch_w1<Tx, NG, 1><<<p.nprob, 32, 0, st>>>(p);
    else if (M <= 2) k5_batch_w1<Tx, NG, 2><<<p.nprob, 32, 0, st>>>(p);
    else if (M <= 4) k5_batch_w1<Tx, NG, 4><<<p.nprob, 32, 0, st>>>(p);
    else k5_batch_w1<Tx, NG, 8><<<p.nprob, 32, 0, st>>>(p);
  } else if (batch_warps_per_problem(p.d) == 2) {
    const int M = (p.d + 63) / 64;
    if (M <= 1) k5_batch<Tx, NG, 1, 2><<<p.nprob, 64, 0, st>>>(p);
    else if (M <= 2) k5_batch<Tx, NG, 2, 2><<<p.nprob, 64, 0, st>>>(p);
    else k5_batch<Tx, NG, 4, 2><<<p.nprob, 64, 0, st>>>(p);
  } else if (p.d <= 128) {
    k5_batch<Tx, NG, 1, 4><<<p.nprob, 128, 0, st>>>(p);
  } else {
    k5_batch<Tx, NG, 2, 4><<<p.nprob, 128, 0, st>>>(p);
  }
  return cudaGetLastError();
}

template <class Tx>
static cudaError_t launch_b_dt(const BatchParams& p, cudaStream_t st) {
  constexpr int V = BVec<Tx>::V;
  const int ngroups = (p.d + V - 1) / V;
  const int NG = (ngroups + 31) / 32;
  switch (NG) {
    case 1: return launch_b_ng<Tx, 1>(p, st);
    case 2: return launch_b_ng<Tx, 2>(p, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

cudaError_t launch_batch(const BatchParams& p, int /*threads*/, cudaStream_t st) {
  if (p.d > 256 || p.d < 1 || (p.splits & (p.splits - 1)) || p.splits < 4) return cudaErrorInvalidConfiguration;
  switch (p.dtype) {
    case 0: return launch_b_dt<double>(p, st);
    case 1: return launch_b_dt<float>(p, st);
    default: return launch_b_dt<__nv_bfloat16>(p, st);
  }
}

}  // namespace halp
