// k_fullgrad_ws.cu -- K1 for two-class softmax (BASELINE C4: bf16,
// 16,777,216 x 1024): the streaming pass with a warp-specialized, one-tile
// software pipeline.
//
// Reference: Objective::full_gradient + Objective::loss, softmax rows
// (proj/src/objectives.cpp:258-311, :193-223, :277-283), evaluated in the
// logistic form of oracle mirror_logistic_row (one dot with w1 - w0, the
// class-1 column the exact negation of class 0).
//
// Why a separate kernel: per row the loss derivative is a ~60-deep chain of
// dependent fp64 ops (exp, an IEEE division, log for the loss) that the
// streaming kernel leaves exposed once per tile (k_fullgrad_stream.cu: 44% of
// HBM at C4, stalls dominated by fixed-latency waits).  Here
//   * NWC compute warps stream tiles: wait the tile's mbarrier, convert x once
//     into registers, row dots, warp reduce-scatter -> shared partials, and
//     arrive on P(j);  then wait D(j-1) and run tile j-1's gradient with the
//     x they still hold (two x buffers, statically unrolled);
//   * one finisher warp waits P(j), refills tile j's stage (cp.async.bulk),
//     sums the warp partials, evaluates the derivative and the loss of the
//     tile's rows (lane r = row r), publishes dl and arrives on D(j).
// So the finisher's latency chain overlaps the compute warps' next tile.
// Named barriers (bar.sync / bar.arrive): P(j) = 1 + (j & 1), D(j) = 3 + (j & 1).
//
// Floating-point order = oracle MIRROR mode (identical to k1_stream): row
// dot = sequential fma over the thread's groups, xor butterfly, warps summed
// in order; gradient column and loss sequential over the split's rows.
#include <type_traits>

#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

namespace {

template <class Tx> struct VecW;
template <> struct VecW<float> { static constexpr int V = 4; };
template <> struct VecW<__nv_bfloat16> { static constexpr int V = 8; };
template <> struct VecW<double> { static constexpr int V = 2; };

template <class Tx>
__device__ __forceinline__ void load_group_w(const Tx* p, double* out) {
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

// bf16 -> x * 2^-896 by integer ops (k_fullgrad_stream.cu load_group_scaled)
template <class Tx>
__device__ __forceinline__ void load_group_ws(const Tx* p, double* out) {
  static_assert(sizeof(Tx) == 2, "bf16 only");
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  const uint32_t wds[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t w = wds[q];
    const uint32_t hlo = ((w << 16) & 0x80000000u) | ((w << 13) & 0x0FFFE000u);
    const uint32_t hhi = (w & 0x80000000u) | ((w >> 3) & 0x0FFFE000u);
    out[2 * q] = __hiloint2double((int)hlo, 0);
    out[2 * q + 1] = __hiloint2double((int)hhi, 0);
  }
}

template <int NV>
__device__ __forceinline__ void reduce_scatter_w(double (&v)[NV], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int off = 16 >> st;
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

template <int N> struct Lg2 { static constexpr int v = 1 + Lg2<N / 2>::v; };
template <> struct Lg2<1> { static constexpr int v = 0; };
template <bool B> struct WTag { static constexpr bool value = B; };

__device__ __forceinline__ void nb_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// position in a CTA's tile sequence (its splits ls = blockIdx.x + k*gridDim.x)
struct TileCursor {
  int ls;
  int64_t i, r0, r1, ntile;
  __device__ void split(const FgParams& p, int nloc, int R) {
    i = 0;
    if (ls < nloc) {
      const unsigned long long nn = (unsigned long long)p.n, SS = (unsigned long long)p.S;
      r0 = (int64_t)(nn * (unsigned long long)(p.split0 + ls) / SS);
      r1 = (int64_t)(nn * (unsigned long long)(p.split0 + ls + 1) / SS);
      ntile = (r1 - r0 + R - 1) / R;
    }
  }
  __device__ void next(const FgParams& p, int nloc, int R) {
    if (++i >= ntile) {
      ls += gridDim.x;
      split(p, nloc, R);
    }
  }
};

}  // namespace

template <class Tx, int NWC, int NG, int R, int STAGES, bool FULLG>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k1_ws(FgParams p, int nloc) {
  constexpr int V = VecW<Tx>::V;
  constexpr int T1 = NWC * 32;
  constexpr int NT = (NWC + 1) * 32;
  constexpr int LG = Lg2<R>::v;
  static_assert((R & (R - 1)) == 0 && R <= 32, "R must be a power of two <= 32");
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool finisher = wid == NWC;
  const int d = p.d, D = 2 * d, ld = p.ld;
  const int ngroups = (d + V - 1) / V;
  const int64_t stage_elems = (int64_t)R * ld;
  Tx* stages = reinterpret_cast<Tx*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)STAGES * stage_elems * sizeof(Tx));  // [2][NWC][R]
  double* dls = red + 2 * NWC * R;                                                             // [2][R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(dls + 2 * R);
  const Tx* X = reinterpret_cast<const Tx*>(p.X);

  // compute warps: w1 - w0 of their feature groups in registers
  double wr[NG][V];
  bool gval[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    gval[k] = !finisher && (FULLG || tid + k * T1 < ngroups);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int j = (tid + k * T1) * V + q;
      wr[k][q] = (finisher || j >= d) ? 0.0 : p.w[d + j] - p.w[j];
    }
  }
  constexpr bool SCALE_OK = std::is_same<Tx, __nv_bfloat16>::value;
  bool ok = SCALE_OK && p.x_finite;
#pragma unroll
  for (int k = 0; k < NG; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q) ok = ok && fabs(wr[k][q]) < 0x1.0p126;
  if (tid == 0) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  const bool scaled = __syncthreads_and(ok) != 0;
  if (scaled) {
#pragma unroll
    for (int k = 0; k < NG; ++k)
#pragma unroll
      for (int q = 0; q < V; ++q) wr[k][q] = __dmul_rn(wr[k][q], 0x1.0p896);
  }
  // the CTA's tile count
  int64_t ntiles = 0;
  {
    TileCursor c{(int)blockIdx.x, 0, 0, 0, 0};
    for (; c.ls < nloc; c.ls += gridDim.x) {
      c.split(p, nloc, R);
      ntiles += c.ntile;
    }
  }

  auto run = [&](auto scaled_tag) {
    constexpr bool SC = SCALE_OK && decltype(scaled_tag)::value;
    if (finisher) {
      // ---------------- finisher warp (+ producer on lane 0) ----------------
      TileCursor pc{(int)blockIdx.x, 0, 0, 0, 0};  // producer
      pc.split(p, nloc, R);
      auto issue = [&](int64_t j) {
        if (pc.ls >= nloc) return;
        const int st = (int)(j % STAGES);
        const int64_t row = pc.r0 + pc.i * R;
        const int64_t rows = (pc.r1 - row) < R ? (pc.r1 - row) : R;
        const uint32_t bytes = (uint32_t)(rows * ld * (int64_t)sizeof(Tx));
        mbar_expect_tx(&bars[st], bytes);
        bulk_g2s(stages + st * stage_elems, X + row * ld, bytes, &bars[st]);
        pc.next(p, nloc, R);
      };
      if (lane == 0)
        for (int64_t j = 0; j < STAGES && j < ntiles; ++j) issue(j);
      TileCursor fc{(int)blockIdx.x, 0, 0, 0, 0};
      fc.split(p, nloc, R);
      double la = 0.0;
      int lab_next = 0;
      if (lane < R && fc.ls < nloc && fc.r0 + lane < fc.r1) lab_next = p.labels[fc.r0 + lane];
#pragma unroll 1
      for (int64_t j = 0; j < ntiles; ++j) {
        const int64_t rowb = fc.r0 + fc.i * R;
        const int nr = (int)((fc.r1 - rowb) < R ? (fc.r1 - rowb) : R);
        const int lab = lab_next;
        const bool last_of_split = fc.i + 1 == fc.ntile;
        const int ls_cur = fc.ls;
        fc.next(p, nloc, R);
        if (lane < R && fc.ls < nloc) {
          const int64_t rn = fc.r0 + fc.i * R + lane;
          if (rn < fc.r1) lab_next = p.labels[rn];
        }
        nb_sync(1 + (int)(j & 1), NT);  // P(j): the tile's partials are in shared memory
        if (lane == 0 && j + STAGES < ntiles) issue(j + STAGES);
        const double* rb = red + (j & 1) * (NWC * R);
        double pv[NWC];
#pragma unroll
        for (int w2 = 0; w2 < NWC; ++w2) pv[w2] = lane < R ? rb[w2 * R + lane] : 0.0;
        double s = pv[0];
#pragma unroll
        for (int w2 = 1; w2 < NWC; ++w2) s = s + pv[w2];
        // logistic form (mirror_logistic_row)
        const double q = hexp(-fabs(s));
        const double den = 1.0 + q;
        const double p0 = (s > 0.0 ? q : 1.0) / den;
        double dl = lab == 0 ? p0 - 1.0 : p0;
        if constexpr (SC) dl = __dmul_rn(dl, 0x1.0p896);  // |dl| <= 1: exact
        if (lane < R) dls[(j & 1) * R + lane] = lane < nr ? dl : 0.0;
        nb_arrive(3 + (int)(j & 1), NT);  // D(j)
        const double a = lab == 0 ? s : -s;
        const double lt = (a > 0.0 ? a : 0.0) + hlog(den);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double t = __shfl_sync(0xffffffffu, lt, r);
          if (r < nr) la = la + t;
        }
        if (last_of_split) {
          if (lane == 0) p.partials[(size_t)ls_cur * (D + 1) + D] = la;
          la = 0.0;
        }
      }
    } else {
      // ---------------- compute warps ----------------
      TileCursor dc{(int)blockIdx.x, 0, 0, 0, 0};  // dot position (one tile ahead)
      dc.split(p, nloc, R);
      TileCursor gc = dc;  // gradient position
      double gacc[NG][V];
#pragma unroll
      for (int k = 0; k < NG; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q) gacc[k][q] = 0.0;
      double xa[R][NG][V], xb[R][NG][V];
      // load + dot of tile j (position dc) into x; partials -> red[j & 1]; arrive P(j)
      auto dot_tile = [&](int64_t j, double(&x)[R][NG][V]) {
        const int64_t rowb = dc.r0 + dc.i * R;
        const int nr = (int)((dc.r1 - rowb) < R ? (dc.r1 - rowb) : R);
        const int st = (int)(j % STAGES);
        mbar_wait(&bars[st], (uint32_t)((j / STAGES) & 1));
        const Tx* xs = stages + st * stage_elems;
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < NG; ++k) {
            if (r < nr && gval[k]) {
              if constexpr (SC) load_group_ws<Tx>(xs + (int64_t)r * ld + (tid + k * T1) * V, x[r][k]);
              else load_group_w<Tx>(xs + (int64_t)r * ld + (tid + k * T1) * V, x[r][k]);
            } else {
#pragma unroll
              for (int q = 0; q < V; ++q) x[r][k][q] = 0.0;
            }
          }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < NG; ++k)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[r] = fma(x[r][k][q], wr[k][q], acc[r]);
        reduce_scatter_w<R>(acc, lane);
        double* rb = red + (j & 1) * (NWC * R);
        if ((lane & ((32 >> LG) - 1)) == 0) rb[wid * R + (lane >> (5 - LG))] = acc[0];
        nb_arrive(1 + (int)(j & 1), NT);  // P(j)
        dc.next(p, nloc, R);
      };
      // gradient of tile j (position gc) with its x; split end -> partial columns
      auto grad_tile = [&](int64_t j, const double(&x)[R][NG][V]) {
        nb_sync(3 + (int)(j & 1), NT);  // D(j)
        const double* dp = dls + (j & 1) * R;
        double dlr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) dlr[r] = dp[r];
        // rows beyond the tile's end have dl = 0 and x = 0: adding +0 leaves gacc unchanged
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < NG; ++k)
#pragma unroll
            for (int q = 0; q < V; ++q) gacc[k][q] = fma(dlr[r], x[r][k][q], gacc[k][q]);
        if (gc.i + 1 == gc.ntile) {
          double* out = p.partials + (size_t)gc.ls * (D + 1);
#pragma unroll
          for (int k = 0; k < NG; ++k) {
            const int g = tid + k * T1;
            if (gval[k]) {
#pragma unroll
              for (int q = 0; q < V; ++q) {
                const int jj = g * V + q;
                if (jj < d) {
                  out[jj] = gacc[k][q];
                  out[(size_t)d + jj] = -gacc[k][q];  // class 1 = -class 0, exactly
                }
                gacc[k][q] = 0.0;
              }
            }
          }
        }
        gc.next(p, nloc, R);
      };
      if (ntiles > 0) dot_tile(0, xa);
#pragma unroll 1
      for (int64_t j = 0; j < ntiles; j += 2) {
        if (j + 1 < ntiles) dot_tile(j + 1, xb);
        grad_tile(j, xa);
        if (j + 1 >= ntiles) break;
        if (j + 2 < ntiles) dot_tile(j + 2, xa);
        grad_tile(j + 1, xb);
      }
    }
  };
  if (scaled) run(WTag<true>{});
  else run(WTag<false>{});
}

// ------------------------------------------------------------------ dispatch
size_t ws_smem_bytes(int ld, int elem, int warps, int R, int stages) {
  size_t b = (size_t)stages * R * ld * elem;
  b = (b + 15) / 16 * 16;
  b += (size_t)2 * warps * R * 8 + (size_t)2 * R * 8 + (size_t)stages * 8;
  return b;
}

namespace {

template <class Tx, int NWC, int NG, int R, int STAGES, bool FULLG>
cudaError_t launch_ws_k(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  auto kern = k1_ws<Tx, NWC, NG, R, STAGES, FULLG>;
  const size_t smem = ws_smem_bytes(L.ld, (int)sizeof(Tx), NWC, R, STAGES);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (NWC + 1) * 32, smem)) != cudaSuccess)
    return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int grid = sms * per_sm;
  if (grid > L.nsplit_local) grid = L.nsplit_local;
  kern<<<grid, (NWC + 1) * 32, smem, st>>>(p, L.nsplit_local);
  return cudaGetLastError();
}

template <class Tx, int NWC, int NG, int R, int STAGES>
cudaError_t launch_ws_f(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  constexpr int V = VecW<Tx>::V;
  if (((p.d + V - 1) / V) == NG * NWC * 32) return launch_ws_k<Tx, NWC, NG, R, STAGES, true>(L, p, st);
  return launch_ws_k<Tx, NWC, NG, R, STAGES, false>(L, p, st);
}

template <class Tx>
cudaError_t launch_ws_t(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  const int nw = L.threads / 32;
  switch (nw * 10000 + L.ng * 1000 + L.rows * 10 + L.stages) {
#define HALP_WS_CASE(NW, NG, R, ST) \
  case NW * 10000 + NG * 1000 + R * 10 + ST: return launch_ws_f<Tx, NW, NG, R, ST>(L, p, st);
    HALP_WS_SHAPES(HALP_WS_CASE)
#undef HALP_WS_CASE
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace

cudaError_t launch_fullgrad_ws(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if (p.C != 2) return cudaErrorInvalidConfiguration;
  switch (L.dtype) {
    case 0: return launch_ws_t<double>(L, p, st);
    case 1: return launch_ws_t<float>(L, p, st);
    default: return launch_ws_t<__nv_bfloat16>(L, p, st);
  }
}

}  // namespace halp
