// k_fullgrad_rows.cu -- K1 for narrow rows (<= 32 x 4 sixteen-byte groups:
// d <= 1024 bf16 / 512 f32 / 256 f64; least squares and two classes, e.g.
// BASELINE C4): one WARP per row, no block barrier on the row path.
//
// Reference: Objective::full_gradient + Objective::loss in one HBM pass
// (proj/src/objectives.cpp:258-311, :193-223).
//
// Structure:
//   * a CTA of NWC warps owns NWC consecutive splits of the MIRROR split
//     grid (S' = S * NWC); warp w walks split s*NWC + w row by row from its
//     own cp.async.bulk ring (STAGES tiles of RT rows, issued by lane 0,
//     mbarrier completion), so warps never wait for each other inside a split;
//   * lane l owns the 16-byte feature groups l, l + 32, ... (GPL of them):
//     the iterate (w, or w1 - w0 for two classes) and the split's gradient
//     column live in registers; the row dot is a 5-level butterfly all-reduce,
//     after which EVERY lane holds the row's logit and evaluates the loss
//     derivative itself (no broadcast);
//   * at the end of a CTA split the NWC warp partials are combined in shared
//     memory by the pairwise tree -- exactly the first log2(NWC) levels of
//     the global split tree -- and one (D+1) partial is written per CTA split.
//
// Floating-point order = oracle MIRROR mode with fg_threads = 32: row dot =
// sequential fma over the lane's groups, xor butterfly 16..1; gradient column
// and loss sequential over the split's rows; splits combined pairwise.  Two
// classes use the logistic form (mirror_logistic_row), bf16 two-class sweeps
// the integer 2^-896-scaled conversion (see k_fullgrad_stream.cu).
#include <type_traits>

#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

namespace {

template <class Tx> struct VecR;
template <> struct VecR<float> { static constexpr int V = 4; };
template <> struct VecR<__nv_bfloat16> { static constexpr int V = 8; };
template <> struct VecR<double> { static constexpr int V = 2; };

template <class Tx>
__device__ __forceinline__ void load_group_r(const Tx* p, double* out) {
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
__device__ __forceinline__ void load_group_rs(const Tx* p, double* out) {
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

template <bool B> struct Tag { static constexpr bool value = B; };

}  // namespace

template <class Tx, int CC, int GPL, int NWC, int RT, int STAGES>
__global__ void __launch_bounds__(NWC * 32, 1) k1_rows(FgParams p, int nloc) {
  constexpr int V = VecR<Tx>::V;
  static_assert(CC == 1 || CC == 2, "least squares or two classes");
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, tid = threadIdx.x;
  const int d = p.d, D = d * CC, ld = p.ld;
  const int ngroups = (d + V - 1) / V;
  const int64_t tile_elems = (int64_t)RT * ld;
  // layout: rings [NWC][STAGES][RT*ld] | comb [NWC][d] doubles | comb_l [NWC] | bars [NWC][STAGES]
  Tx* ring = reinterpret_cast<Tx*>(smem) + (int64_t)wid * STAGES * tile_elems;
  const size_t ring_bytes = ((size_t)NWC * STAGES * tile_elems * sizeof(Tx) + 15) / 16 * 16;
  double* comb = reinterpret_cast<double*>(smem + ring_bytes);
  double* comb_l = comb + (size_t)NWC * d;
  uint64_t* bars = reinterpret_cast<uint64_t*>(comb_l + NWC) + wid * STAGES;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  const unsigned long long nn = (unsigned long long)p.n;
  const unsigned long long SS = (unsigned long long)p.S;  // MIRROR splits (NWC per CTA split)

  double wr[GPL][V];
  bool gval[GPL];
#pragma unroll
  for (int k = 0; k < GPL; ++k) {
    gval[k] = lane + 32 * k < ngroups;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int j = (lane + 32 * k) * V + q;
      wr[k][q] = j >= d ? 0.0 : CC == 1 ? p.w[j] : p.w[d + j] - p.w[j];
    }
  }
  constexpr bool SCALE_OK = std::is_same<Tx, __nv_bfloat16>::value && CC == 2;
  bool ok = SCALE_OK && p.x_finite;
#pragma unroll
  for (int k = 0; k < GPL; ++k)
#pragma unroll
    for (int q = 0; q < V; ++q) ok = ok && fabs(wr[k][q]) < 0x1.0p126;
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  const bool scaled = __syncthreads_and(ok) != 0;
  if (scaled) {
#pragma unroll
    for (int k = 0; k < GPL; ++k)
#pragma unroll
      for (int q = 0; q < V; ++q) wr[k][q] = __dmul_rn(wr[k][q], 0x1.0p896);
  }

  // ---- per-warp producer (lane 0): this warp's tiles across its splits ----
  int ls_p = blockIdx.x;
  int64_t pt = 0, pr0 = 0, pr1 = 0;
  auto sub_rows = [&](int ls, int64_t& a, int64_t& b) {
    const unsigned long long s = (unsigned long long)p.split0 + (unsigned long long)ls * NWC + wid;
    a = (int64_t)(nn * s / SS);
    b = (int64_t)(nn * (s + 1) / SS);
  };
  auto advance_split = [&]() {
    // next split of this CTA with at least one row for this warp
    for (;;) {
      if (ls_p >= nloc) return;
      sub_rows(ls_p, pr0, pr1);
      if (pr1 > pr0) return;
      ls_p += gridDim.x;
    }
  };
  if (lane == 0) advance_split();
  auto issue = [&](int64_t j) {
    if (ls_p >= nloc) return;
    const int st = (int)(j % STAGES);
    const int64_t row = pr0 + pt * RT;
    const int64_t rows = (pr1 - row) < RT ? (pr1 - row) : RT;
    const uint32_t bytes = (uint32_t)(rows * ld * (int64_t)sizeof(Tx));
    mbar_expect_tx(&bars[st], bytes);
    bulk_g2s(ring + st * tile_elems, X + row * ld, bytes, &bars[st]);
    if (row + RT >= pr1) {
      ls_p += gridDim.x;
      pt = 0;
      advance_split();
    } else {
      ++pt;
    }
  };
  if (lane == 0)
#pragma unroll 1
    for (int j = 0; j < STAGES; ++j) issue(j);

  int64_t jseq = 0;  // this warp's consumer position in its tile sequence
  auto run = [&](auto scaled_tag) {
    constexpr bool SC = SCALE_OK && decltype(scaled_tag)::value;
#pragma unroll 1
    for (int ls = blockIdx.x; ls < nloc; ls += gridDim.x) {
      int64_t r0, r1;
      sub_rows(ls, r0, r1);
      double gacc[GPL][V];
#pragma unroll
      for (int k = 0; k < GPL; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q) gacc[k][q] = 0.0;
      double la = 0.0;
      using TgtT = std::conditional_t<CC == 1, double, int32_t>;
      TgtT tnext = 0;
      if (r0 < r1) tnext = CC == 1 ? (TgtT)p.y[r0] : (TgtT)p.labels[r0];
#pragma unroll 1
      for (int64_t row = r0; row < r1; row += RT, ++jseq) {
        const int st = (int)(jseq % STAGES);
        mbar_wait(&bars[st], (uint32_t)((jseq / STAGES) & 1));
        const Tx* xt = ring + st * tile_elems;
        const int nr = (int)((r1 - row) < RT ? (r1 - row) : RT);
#pragma unroll 1
        for (int r = 0; r < nr; ++r) {
          const TgtT tcur = tnext;
          if (row + r + 1 < r1) tnext = CC == 1 ? (TgtT)p.y[row + r + 1] : (TgtT)p.labels[row + r + 1];
          double x[GPL][V];
#pragma unroll
          for (int k = 0; k < GPL; ++k) {
            if (gval[k]) {
              if constexpr (SC) load_group_rs<Tx>(xt + (int64_t)r * ld + (lane + 32 * k) * V, x[k]);
              else load_group_r<Tx>(xt + (int64_t)r * ld + (lane + 32 * k) * V, x[k]);
            } else {
#pragma unroll
              for (int q = 0; q < V; ++q) x[k][q] = 0.0;
            }
          }
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < GPL; ++k)
#pragma unroll
            for (int q = 0; q < V; ++q) s = fma(x[k][q], wr[k][q], s);
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s = s + __shfl_xor_sync(0xffffffffu, s, o);
          // the tile's last row is consumed by every lane (the butterfly needs
          // all lanes' dots): its stage can be refilled
          if (r == nr - 1 && lane == 0) issue(jseq + STAGES);
          double dl;
          if constexpr (CC == 1) {
            dl = s - tcur;
            la = la + __dmul_rn(__dmul_rn(0.5, dl), dl);
          } else {
            const int lab = (int)tcur;
            const double q = hexp(-fabs(s));
            const double den = 1.0 + q;
            const double p0 = (s > 0.0 ? q : 1.0) / den;
            dl = lab == 0 ? p0 - 1.0 : p0;
            const double a = lab == 0 ? s : -s;
            la = la + ((a > 0.0 ? a : 0.0) + hlog(den));
            if constexpr (SC) dl = __dmul_rn(dl, 0x1.0p896);  // |dl| <= 1: exact
          }
#pragma unroll
          for (int k = 0; k < GPL; ++k)
#pragma unroll
            for (int q = 0; q < V; ++q) gacc[k][q] = fma(dl, x[k][q], gacc[k][q]);
        }
      }
      // ---- combine the NWC warp partials: pairwise tree (first levels of the split tree) ----
      double* cw = comb + (size_t)wid * d;
#pragma unroll
      for (int k = 0; k < GPL; ++k)
        if (gval[k])
#pragma unroll
          for (int q = 0; q < V; ++q) {
            const int j = (lane + 32 * k) * V + q;
            if (j < d) cw[j] = gacc[k][q];
          }
      if (lane == 0) comb_l[wid] = la;
      __syncthreads();
      double* out = p.partials + (size_t)ls * (D + 1);
      for (int j = tid; j <= d; j += NWC * 32) {
        const double* src = j < d ? comb + j : comb_l;
        const size_t stride = j < d ? (size_t)d : 1;
        double v[NWC];
#pragma unroll
        for (int i = 0; i < NWC; ++i) v[i] = src[i * stride];
#pragma unroll
        for (int h = 1; h < NWC; h *= 2)
#pragma unroll
          for (int i = 0; i < NWC; i += 2 * h) v[i] = v[i] + v[i + h];
        if (j < d) {
          out[j] = v[0];
          if (CC == 2) out[(size_t)d + j] = -v[0];  // class 1 = -class 0, exactly
        } else {
          out[D] = v[0];
        }
      }
      __syncthreads();  // comb is reused by the next split
    }
  };
  if (scaled) run(Tag<true>{});
  else run(Tag<false>{});
}

// ------------------------------------------------------------------ dispatch
size_t rows_smem_bytes(int ld, int elem, int d, int warps, int RT, int stages) {
  size_t b = ((size_t)warps * stages * RT * ld * elem + 15) / 16 * 16;
  b += (size_t)warps * d * 8 + (size_t)warps * 8 + (size_t)warps * stages * 8;
  return b;
}

namespace {

template <class Tx, int CC, int GPL, int NWC, int RT, int STAGES>
cudaError_t launch_rows_k(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  auto kern = k1_rows<Tx, CC, GPL, NWC, RT, STAGES>;
  const size_t smem = rows_smem_bytes(L.ld, (int)sizeof(Tx), p.d, NWC, RT, STAGES);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NWC * 32, smem)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int grid = sms * per_sm;
  if (grid > L.nsplit_local) grid = L.nsplit_local;
  kern<<<grid, NWC * 32, smem, st>>>(p, L.nsplit_local);
  return cudaGetLastError();
}

template <class Tx, int CC>
cudaError_t launch_rows_cc(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.ng * 10000 + L.sub * 100 + L.rows * 10 + L.stages) {
#define HALP_ROWS_CASE(GPL, NWC, RT, ST) \
  case GPL * 10000 + NWC * 100 + RT * 10 + ST: return launch_rows_k<Tx, CC, GPL, NWC, RT, ST>(L, p, st);
    HALP_ROWS_SHAPES(HALP_ROWS_CASE)
#undef HALP_ROWS_CASE
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace

cudaError_t launch_fullgrad_rows(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.dtype * 10 + p.C) {
    case 1: return launch_rows_cc<double, 1>(L, p, st);
    case 2: return launch_rows_cc<double, 2>(L, p, st);
    case 11: return launch_rows_cc<float, 1>(L, p, st);
    case 12: return launch_rows_cc<float, 2>(L, p, st);
    case 21: return launch_rows_cc<__nv_bfloat16, 1>(L, p, st);
    case 22: return launch_rows_cc<__nv_bfloat16, 2>(L, p, st);
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace halp
