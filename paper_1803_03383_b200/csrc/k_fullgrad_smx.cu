// k_fullgrad_smx.cu -- K1 for softmax objectives with 3..16 classes (the
// MNIST-shaped C2 workload): one HBM pass computing g~ and the loss.
//
// Reference: Objective::full_gradient / Objective::loss for LossFamily::Softmax
// (proj/src/objectives.cpp:258-311, :193-223, softmax rows :277-283).
//
// Same reduction order as k1_fullgrad / k1_reg (oracle MIRROR mode): thread t
// owns the 16-byte feature group t (NG = 1), row logits = sequential fma over
// the group, warp xor-butterfly (done as a 32-slot reduce-scatter: slot
// r*C + c = (row r, class c)), warps summed in order; softmax per row with a
// sequential max and sum; gradient columns by sequential fma over the split's
// rows; per-row losses summed sequentially.
//
// Layout: R = 32 / C rows per tile streamed by cp.async.bulk into a 4-deep
// shared ring; the iterate (d*C doubles) in shared memory; every thread keeps
// its V x C gradient accumulators in registers for the whole split.
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

namespace {
template <class Tx> struct VecS;
template <> struct VecS<float> { static constexpr int V = 4; };
template <> struct VecS<__nv_bfloat16> { static constexpr int V = 8; };
template <> struct VecS<double> { static constexpr int V = 2; };

template <class Tx>
__device__ __forceinline__ void load_group_s(const Tx* p, double* out) {
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

// 32-slot reduce-scatter: lane l ends with the butterfly sum of slot l
__device__ __forceinline__ void reduce_scatter_32(double (&v)[32], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int off = 16 >> st, h = 16 >> st;
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
}
}  // namespace

constexpr int kSmxStages = 4;

template <class Tx, int CC>
__global__ void __launch_bounds__(256, 1) k1_smx(FgParams p) {
  constexpr int V = VecS<Tx>::V;
  constexpr int R = 32 / CC;
  constexpr int NV = R * CC;
  constexpr int STAGES = kSmxStages;
  extern __shared__ __align__(128) unsigned char smem[];
  const int T1 = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = T1 >> 5;
  const int d = p.d, D = d * CC, ld = p.ld;
  const int ngroups = (d + V - 1) / V;
  const size_t stage_elems = (size_t)R * ld;
  Tx* stages = reinterpret_cast<Tx*>(smem);
  double* w_s = reinterpret_cast<double*>(smem + STAGES * stage_elems * sizeof(Tx));
  double* red = w_s + D;  // [2][NW][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * NW * 32);
  int* lsm = reinterpret_cast<int*>(bars + STAGES);  // labels of the split

  const int s = p.split0 + blockIdx.x;
  const int64_t r0 = (int64_t)(((unsigned long long)p.n * (unsigned long long)s) / (unsigned long long)p.S);
  const int64_t r1 = (int64_t)(((unsigned long long)p.n * (unsigned long long)(s + 1)) / (unsigned long long)p.S);
  const int64_t ntile = (r1 - r0 + R - 1) / R;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  for (int64_t q = tid; q < r1 - r0; q += T1) lsm[q] = p.labels[r0 + q];
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
    bulk_g2s(stages + (size_t)st * stage_elems, X + row * ld, bytes, &bars[st]);
  };
  if (tid == 0)
    for (int64_t t = 0; t < ntile && t < STAGES; ++t) issue(t);

  const bool gv = tid < ngroups;
  const int j0 = tid * V;
  // this thread's slice of the iterate, zero beyond d (x is zero there too)
  bool jv[V];
#pragma unroll
  for (int q = 0; q < V; ++q) jv[q] = gv && (j0 + q < d);
  double gacc[V][CC];
#pragma unroll
  for (int q = 0; q < V; ++q)
#pragma unroll
    for (int c = 0; c < CC; ++c) gacc[q][c] = 0.0;
  double la = 0.0;
  const int fr = lane / CC, fc = lane % CC;
  const int base = (fr * CC) & 31;

  for (int64_t i = 0; i < ntile; ++i) {
    const int st = (int)(i % STAGES);
    const int64_t rowb = r0 + i * R;
    const int nr = (int)((r1 - rowb) < R ? (r1 - rowb) : R);
    const bool act = (lane < NV) && (fr < nr);
    const int lab = act ? lsm[rowb - r0 + fr] : 0;
    mbar_wait(&bars[st], (uint32_t)((i / STAGES) & 1));
    const Tx* xs = stages + (size_t)st * stage_elems;
    double xr[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr && gv) {
        load_group_s<Tx>(xs + (size_t)r * ld + j0, xr[r]);
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) xr[r][q] = 0.0;
      }
    }
    double acc[32];
#pragma unroll
    for (int v = 0; v < 32; ++v) acc[v] = 0.0;
#pragma unroll
    for (int c = 0; c < CC; ++c) {
      double wv[V];
#pragma unroll
      for (int q = 0; q < V; ++q) wv[q] = jv[q] ? w_s[c * d + j0 + q] : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < V; ++q)
          if (jv[q]) acc[r * CC + c] = fma(xr[r][q], wv[q], acc[r * CC + c]);
    }
    reduce_scatter_32(acc, lane);
    double* rb = red + (size_t)(i & 1) * NW * 32;
    rb[wid * 32 + lane] = acc[0];
    __syncthreads();
    // x of this tile now lives in registers: its stage can be refilled
    if (tid == 0 && i + STAGES < ntile) issue(i + STAGES);

    // logit of (row fr, class fc): warps summed in order (same in every warp)
    double lg = rb[lane];
    for (int w2 = 1; w2 < NW; ++w2) lg = lg + rb[w2 * 32 + lane];
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
    double pr = e / ssum;
    if (fc == lab) pr = pr - 1.0;
    double lt = 0.0;
    if (wid == 0 && fc == 0) lt = (mx + hlog(ssum)) - lab_logit;
    if (wid == 0 && p.write_loss) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double t = __shfl_sync(0xffffffffu, lt, r * CC);
        if (r < nr) la = la + t;
      }
    }
    // gradient columns: sequential fma over the rows
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nr) {
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          const double dl = __shfl_sync(0xffffffffu, pr, r * CC + c);
#pragma unroll
          for (int q = 0; q < V; ++q) gacc[q][c] = fma(dl, xr[r][q], gacc[q][c]);
        }
      }
    }
  }

  double* out = p.partials + (size_t)blockIdx.x * (D + 1);
#pragma unroll
  for (int q = 0; q < V; ++q)
    if (jv[q])
#pragma unroll
      for (int c = 0; c < CC; ++c) out[(size_t)c * d + j0 + q] = gacc[q][c];
  if (tid == 0 && p.write_loss) out[D] = la;
}

size_t smx_smem_bytes(int ld, int elem, int d, int C, int threads, int64_t split_rows) {
  const int R = 32 / C;
  return (size_t)kSmxStages * R * ld * elem + (size_t)d * C * 8 + 2 * (size_t)(threads / 32) * 32 * 8 +
         kSmxStages * 8 + 4 * (size_t)split_rows;
}

template <class Tx, int CC>
static cudaError_t launch_smx_t(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if constexpr (VecS<Tx>::V * CC > 64) {
    return cudaErrorInvalidConfiguration;  // never planned (register budget)
  } else {
    const int64_t split_rows = (p.n + p.S - 1) / p.S + 1;
    const size_t smem = smx_smem_bytes(L.ld, (int)sizeof(Tx), p.d, CC, L.threads, split_rows);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    auto kern = k1_smx<Tx, CC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (L.dry) return cudaSuccess;
    kern<<<L.nsplit_local, L.threads, smem, st>>>(p);
    return cudaGetLastError();
  }
}

template <class Tx>
static cudaError_t launch_smx_dt(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (p.C) {
    case 3: return launch_smx_t<Tx, 3>(L, p, st);
    case 4: return launch_smx_t<Tx, 4>(L, p, st);
    case 5: return launch_smx_t<Tx, 5>(L, p, st);
    case 6: return launch_smx_t<Tx, 6>(L, p, st);
    case 7: return launch_smx_t<Tx, 7>(L, p, st);
    case 8: return launch_smx_t<Tx, 8>(L, p, st);
    case 9: return launch_smx_t<Tx, 9>(L, p, st);
    case 10: return launch_smx_t<Tx, 10>(L, p, st);
    case 11: return launch_smx_t<Tx, 11>(L, p, st);
    case 12: return launch_smx_t<Tx, 12>(L, p, st);
    case 13: return launch_smx_t<Tx, 13>(L, p, st);
    case 14: return launch_smx_t<Tx, 14>(L, p, st);
    case 15: return launch_smx_t<Tx, 15>(L, p, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

cudaError_t launch_fullgrad_smx(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.dtype) {
    case 0: return launch_smx_dt<double>(L, p, st);
    case 1: return launch_smx_dt<float>(L, p, st);
    default: return launch_smx_dt<__nv_bfloat16>(L, p, st);
  }
}

}  // namespace halp
