// k_fullgrad_stream.cu -- K1 for the HBM-bound shapes (least squares and
// 2-class softmax; BASELINE C1/C3/C4): a persistent streaming kernel.
//
// Reference: Objective::full_gradient + Objective::loss in one HBM pass
// (proj/src/objectives.cpp:258-311 and :193-223; squared rows :274-276,
// softmax rows :277-283).
//
// Structure (everything that decides the instruction count is compile-time):
//   * one CTA per SM (or two), each walking its splits s = blockIdx.x,
//     blockIdx.x + gridDim.x, ... with ONE continuous cp.async.bulk ring of
//     STAGES tiles of R rows -- the ring runs across split boundaries, so the
//     copy engine never drains between splits;
//   * thread t owns the 16-byte feature groups t, t + T1, ... (NG of them):
//     its slice of w~ and of the split's gradient columns live in registers,
//     the tile's x slice is converted to fp64 once and reused by the dot and
//     the gradient phase;
//   * per tile ONE __syncthreads: warp reduce-scatter of the R partial row
//     dots -> shared (parity double-buffered) -> every warp sums the NW warp
//     partials of its lane's row (fully unrolled) and evaluates the loss
//     derivative itself, so no second barrier broadcasts it;
//   * two classes (CC == 2) use the logistic form: the softmax depends only
//     on s = x.(w1 - w0), so ONE dot and ONE gradient column per row (the
//     other column is its exact negation) -- half the fp64 work and half the
//     registers of two softmax logits, which is what lets the bf16 C4 sweep
//     stream at HBM speed.  Formulas: oracle/halp_oracle.c mirror_logistic_row.
//
// Floating-point order = k1_reg / k1_fullgrad = oracle MIRROR mode (DESIGN.md
// "Reduction orders"): row dot = sequential fma over the thread's groups,
// warp xor butterfly 16..1, warps summed in order; gradient column =
// sequential fma over the split's rows; loss = sequential over the rows.
#include <type_traits>

#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

namespace {

template <class Tx> struct VecK;
template <> struct VecK<float> { static constexpr int V = 4; };
template <> struct VecK<__nv_bfloat16> { static constexpr int V = 8; };
template <> struct VecK<double> { static constexpr int V = 2; };

// one 16-byte group from shared memory, upcast exactly
template <class Tx>
__device__ __forceinline__ void load_group_k(const Tx* p, double* out) {
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

// bf16 group -> fp64 with the conversion split between two pipes.  ODD
// features (the high bf16 of each 32-bit word) go through integer ops only:
// the f32 pattern of a bf16 maps to the double with the same sign, exponent
// FIELD and leading mantissa bits, i.e. exactly x * 2^-896 for every finite x
// (normal, subnormal, zero); with w' = w * 2^896 and dl' = dl * 2^896 the
// products x'*w' and dl'*x' equal x*w and dl*x exactly, so every fma rounds
// as with the F2F-converted x.  EVEN features use F2F (unscaled, w and dl
// unscaled).  Requires finite x (checked at problem creation) and |w|, |dl| <
// 2^126 (checked per launch / bounded by 1 for the two-class derivative).
#ifndef HALP_K1_OF
#define HALP_K1_OF 0  // odd features of the first OF words of a group also via F2F
#endif
#ifndef HALP_K1_EF
#define HALP_K1_EF 4  // even features of the first EF words of a group via F2F (the rest integer-upcast)
#endif
__device__ __forceinline__ bool k1_scaled_feature(int j) {
  return (j & 1) ? (j >> 1) >= HALP_K1_OF : (j >> 1) >= HALP_K1_EF;
}

// exact bf16 -> fp64 of the low / high half of a 32-bit word (F2F.F64.BF16 reads the half directly)
__device__ __forceinline__ double bf16_lo_to_f64(uint32_t w) {
  double r;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f64.bf16 %0, l;\n\t}" : "=d"(r) : "r"(w));
  return r;
}
__device__ __forceinline__ double bf16_hi_to_f64(uint32_t w) {
  double r;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f64.bf16 %0, h;\n\t}" : "=d"(r) : "r"(w));
  return r;
}

template <class Tx>
__device__ __forceinline__ void load_group_scaled(const Tx* p, double* out) {
  static_assert(sizeof(Tx) == 2, "bf16 only");
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  const uint32_t wds[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t w = wds[q];
    // arithmetic >> 3 puts the exponent field at bits 27..20 and copies the sign
    // into bits 31..28; the mask keeps bit 31 and the 15 exponent/mantissa bits
    if (q < HALP_K1_EF) {
      out[2 * q] = bf16_lo_to_f64(w);  // even features: one F2F.F64.BF16, unscaled
    } else {
      const uint32_t hlo = (uint32_t)((int32_t)(w << 16) >> 3) & 0x8FFFE000u;
      out[2 * q] = __hiloint2double((int)hlo, 0);
    }
    if (q < HALP_K1_OF) {
      out[2 * q + 1] = bf16_hi_to_f64(w);
    } else {
      const uint32_t hhi = (uint32_t)((int32_t)w >> 3) & 0x8FFFE000u;
      out[2 * q + 1] = __hiloint2double((int)hhi, 0);
    }
  }
}

// xor-butterfly reduce-scatter of NV slots (NV a power of two <= 32): lane l
// ends with the full warp sum of slot l >> (5 - log2 NV).  The pairs added at
// every level are the butterfly's, so each slot's value equals a plain
// xor-butterfly all-reduce (addition is commutative).
// PRE: the first PRE levels need no selects because the caller filled the slots in a
// lane-dependent order (slot i of a lane holds row i ^ p, p = the lane's bits 4.. mapped
// to the slot's top bits), so every lane keeps its low half and sends its high half.
template <int NV, int PRE = 0>
__device__ __forceinline__ void reduce_scatter_k(double (&v)[NV], int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int off = 16 >> st;
    const int cur = NV >> st;
    if (cur > 1) {
      const int h = cur >> 1;
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        if (st < PRE) {
          v[i] = v[i] + __shfl_xor_sync(0xffffffffu, v[i + h], off);
        } else {
          const double send = up ? v[i] : v[i + h];
          const double keep = up ? v[i + h] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
    } else {
      v[0] = v[0] + __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
}

template <int N> struct Log2 { static constexpr int v = 1 + Log2<N / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

template <bool B> struct BoolTag { static constexpr bool value = B; };

}  // namespace

// Minimum resident CTAs per SM the register allocator must allow.  The bf16 two-class
// 16-row shape (C4: 4 warps) fits 168 registers with no spills, so 3 CTAs per SM
// (12 warps) instead of 2 at 243 registers: same-box A/B 8.29 -> 7.60 ms per C4 pass
// (profiles/r01_k1_minb3_ab.txt), bit-identical.  Forcing 3 on the 256-thread fp32
// shapes spills (C3 86% -> 32%).  Current C4 figures: DESIGN.md section 7.
#ifndef HALP_K1_MINB_BF16_2C
#define HALP_K1_MINB_BF16_2C 3
#endif
template <class Tx, int CC, int NW, int R>
struct K1MinBlocks {
  static constexpr int value = (sizeof(Tx) == 2 && CC == 2 && NW == 4 && R == 16) ? HALP_K1_MINB_BF16_2C : 1;
};

template <class Tx, int CC, int NW, int NG, int R, int STAGES, bool FULLG>
__global__ void __launch_bounds__(NW * 32, (K1MinBlocks<Tx, CC, NW, R>::value)) k1_stream(FgParams p, int nloc) {
  constexpr int V = VecK<Tx>::V;
  constexpr int T1 = NW * 32;
  constexpr int NV = R;  // one dot per row (squared: x.w; two classes: x.(w1 - w0))
  constexpr int LG = Log2<NV>::v;
  // RR: tiles of 16+ rows keep x in shared memory only and re-read it for the
  // gradient phase (registers for the row dots instead of an R x 8 fp64 slice)
#ifndef HALP_K1_RR_MIN
#define HALP_K1_RR_MIN 16
#endif
  constexpr bool RR = R >= HALP_K1_RR_MIN;
  // DW: two classes on several warps: ONE warp per tile (rotating over warps 1..) evaluates
  // the rows' softmax derivative (exp + division) and publishes it through shared memory
  // behind a second barrier, instead of every warp repeating it for the same R rows -- the
  // sweep is issue-bound; the loss terms (log) and their running sum
  // trail by one / two tiles and run in the same window on other warps
#ifndef HALP_K1_DW
#define HALP_K1_DW 1
#endif
  constexpr bool DW = HALP_K1_DW && CC == 2 && NW > 1;
  // RL: 16-row tiles fill the dot slots in a lane-dependent row order (slot i = row
  // i ^ p, p = 8 * lane bit 4 + 4 * lane bit 3 [+ 2 * lane bit 2]), which makes the first
  // two [three] levels of the reduce-scatter select-free; four [eight] lane-dependent row
  // bases keep the shared-memory offsets immediate
#ifndef HALP_K1_RELABEL
#define HALP_K1_RELABEL 2  // relabeled levels (0: off; 3 uses eight row bases)
#endif
  constexpr bool RL = HALP_K1_RELABEL > 0 && RR && NV == 16;
  constexpr int RLN = RL ? HALP_K1_RELABEL : 0;
  static_assert(CC == 1 || CC == 2, "least squares or two classes");
  static_assert((NV & (NV - 1)) == 0 && NV <= 32, "R must be a power of two <= 32");
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // FULLG: every group of the padded row is owned, so the row pitch is a
  // compile-time constant (ld = ngroups * V) and tile offsets fold into immediates
  const int d = p.d, D = d * CC, ld = FULLG ? NG * T1 * V : p.ld;
  const int ngroups = (d + V - 1) / V;
  const int64_t stage_elems = (int64_t)R * ld;
  Tx* stages = reinterpret_cast<Tx*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)STAGES * stage_elems * sizeof(Tx));  // [2][NW][NV]
  double* lts = red + 2 * NW * NV;  // [2][NW][R] per-row losses (two classes), parity double-buffered
  double* dsh = lts + 2 * NW * R;  // [R][2] {dl, dl * 2^896} + [2][R][2] {a, 1 + q} by tile parity (two classes, DW)
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsh + 6 * R);
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  const unsigned long long nn = (unsigned long long)p.n, SS = (unsigned long long)p.S;

  double wr[NG][V];  // w (squared) or w1 - w0 (two classes)
  bool gval[NG];
#pragma unroll
  for (int k = 0; k < NG; ++k) {
    gval[k] = FULLG || (tid + k * T1 < ngroups);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const int j = (tid + k * T1) * V + q;
      wr[k][q] = j >= d ? 0.0 : CC == 1 ? p.w[j] : p.w[d + j] - p.w[j];
    }
  }
  // bf16 two-class sweeps convert x with integer ops in the 2^-896-scaled
  // domain (load_group_scaled) when X is known finite and |w1 - w0| < 2^126
  constexpr bool SCALE_OK = std::is_same<Tx, __nv_bfloat16>::value && CC == 2;
  // even features F2F-converted (unscaled, conversion pipe), odd ones integer-
  // upcast (scaled, ALU): the two pipes share the conversion work (C4 58% -> 62%)
  constexpr bool MIXED = true;
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
      for (int q = 0; q < V; ++q)
        if (!MIXED || k1_scaled_feature(q)) wr[k][q] = __dmul_rn(wr[k][q], 0x1.0p896);
  }

  // ---- producer (thread 0): the CTA's tile sequence across its splits ----
  int ls_p = blockIdx.x;
  int64_t pt = 0, pr0 = 0, pr1 = 0;
  if (tid == 0 && ls_p < nloc) {
    pr0 = (int64_t)(nn * (unsigned long long)(p.split0 + ls_p) / SS);
    pr1 = (int64_t)(nn * (unsigned long long)(p.split0 + ls_p + 1) / SS);
  }
  auto issue = [&](int64_t j) {
    if (ls_p >= nloc) return;
    const int st = (int)(j % STAGES);
    const int64_t row = pr0 + pt * R;
    const int64_t rows = (pr1 - row) < R ? (pr1 - row) : R;
    const uint32_t bytes = (uint32_t)(rows * ld * (int64_t)sizeof(Tx));
    mbar_expect_tx(&bars[st], bytes);
    bulk_g2s(stages + st * stage_elems, X + row * ld, bytes, &bars[st]);
    if (row + R >= pr1) {
      ls_p += gridDim.x;
      pt = 0;
      if (ls_p < nloc) {
        pr0 = (int64_t)(nn * (unsigned long long)(p.split0 + ls_p) / SS);
        pr1 = (int64_t)(nn * (unsigned long long)(p.split0 + ls_p + 1) / SS);
      }
    } else {
      ++pt;
    }
  };
  if (tid == 0)
#pragma unroll 1
    for (int j = 0; j < STAGES; ++j) issue(j);

  // lane fr < R evaluates the loss derivative of row fr of every tile
  const int fr = lane;
  int64_t jseq = 0;  // consumer position in the CTA's tile sequence

  int rot = 0;  // DW: rotation of the derivative / loss-term warps over warps 1 .. NW - 1
  auto run = [&](auto scaled_tag) {
  constexpr bool SC = SCALE_OK && decltype(scaled_tag)::value;
#pragma unroll 1
  for (int ls = blockIdx.x; ls < nloc; ls += gridDim.x) {
    const int64_t r0 = (int64_t)(nn * (unsigned long long)(p.split0 + ls) / SS);
    const int64_t r1 = (int64_t)(nn * (unsigned long long)(p.split0 + ls + 1) / SS);
    const int64_t ntile = (r1 - r0 + R - 1) / R;
    double gacc[NG][V];
#pragma unroll
    for (int k = 0; k < NG; ++k)
#pragma unroll
      for (int q = 0; q < V; ++q) gacc[k][q] = 0.0;
    double la = 0.0;
    // targets of the slot rows, one tile ahead (kept raw: used one tile later)
    using TgtT = std::conditional_t<CC == 1, double, int32_t>;
    TgtT tgt = 0;
    if (lane < NV && r0 + fr < r1) tgt = CC == 1 ? (TgtT)p.y[r0 + fr] : (TgtT)p.labels[r0 + fr];

#pragma unroll 1
    for (int64_t i = 0; i < ntile; ++i, ++jseq) {
      const int64_t rowb = r0 + i * R;
      const int nr = (int)((r1 - rowb) < R ? (r1 - rowb) : R);
      const TgtT tcur = tgt;
      if (lane < NV && rowb + R + fr < r1)
        tgt = CC == 1 ? (TgtT)p.y[rowb + R + fr] : (TgtT)p.labels[rowb + R + fr];
      const int st = (int)(jseq % STAGES);
      mbar_wait(&bars[st], (uint32_t)((jseq / STAGES) & 1));
      const Tx* xs = stages + st * stage_elems;
      double* rb = red + (jseq & 1) * (NW * NV);

      auto body = [&](auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        // row r's x slice of this thread, upcast exactly (zeros past the tile / row end)
        auto load_row_at = [&](const Tx* rowp, bool valid, double (&xg)[NG][V]) {
#pragma unroll
          for (int k = 0; k < NG; ++k) {
            if ((FULL || valid) && gval[k]) {
              if constexpr (SC) load_group_scaled<Tx>(rowp + (tid + k * T1) * V, xg[k]);
              else load_group_k<Tx>(rowp + (tid + k * T1) * V, xg[k]);
            } else {
#pragma unroll
              for (int q = 0; q < V; ++q) xg[k][q] = 0.0;
            }
          }
        };
        auto load_row = [&](int r, double (&xg)[NG][V]) { load_row_at(xs + (int64_t)r * ld, r < nr, xg); };
        // RL: slot r's row is r ^ p = r +- p8 +- p4 (signs by slot bits 3, 2): base[bits] + r * ld
        const int pl = RL ? ((lane >> 1) & (16 - (16 >> RLN))) : 0;  // lane bits 4.. -> slot bits 3..
        const Tx* xb[RL ? (1 << RLN) : 1];
        if constexpr (RL) {
#pragma unroll
          for (int bi = 0; bi < (1 << RLN); ++bi) {
            int off = 0;
#pragma unroll
            for (int b = 0; b < RLN; ++b) {
              const int pb = pl & (8 >> b);  // the lane's flip of slot bit 3 - b
              off += ((bi >> (RLN - 1 - b)) & 1) ? -pb : pb;
            }
            xb[bi] = xs + (int64_t)off * ld;
          }
        }
        double xr[RR ? 1 : R][NG][V];
        double acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = 0.0;
        if constexpr (!RR) {
#pragma unroll
          for (int r = 0; r < R; ++r) load_row(r, xr[RR ? 0 : r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (RL) load_row_at(xb[RL ? (r >> (4 - RLN)) : 0] + (int64_t)r * ld, (r ^ pl) < nr, xr[0]);
          else if constexpr (RR) load_row(r, xr[0]);
#pragma unroll
          for (int k = 0; k < NG; ++k)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[r] = fma(xr[RR ? 0 : r][k][q], wr[k][q], acc[r]);
        }
        reduce_scatter_k<NV, RLN>(acc, lane);
        if ((lane & ((32 >> LG) - 1)) == 0) rb[wid * NV + (lane >> (5 - LG))] = acc[0];
        __syncthreads();
        // x in registers: this tile's stage can be refilled now; x re-read in the
        // gradient phase (RR): every warp has finished the PREVIOUS tile, refill that
        if (tid == 0) {
          if constexpr (RR) {
            if (jseq > 0) issue(jseq - 1 + STAGES);
          } else {
            issue(jseq + STAGES);
          }
        }

        // logit of slot (fr, fc): the NW warp partials summed in warp order
        auto row_logit = [&]() {
          double lg = 0.0;
          if (lane < NV) {
            double pv[NW];
#pragma unroll
            for (int w2 = 0; w2 < NW; ++w2) pv[w2] = rb[w2 * NV + lane];
            lg = pv[0];
#pragma unroll
            for (int w2 = 1; w2 < NW; ++w2) lg = lg + pv[w2];
          }
          return lg;
        };
        double pr = 0.0, lt = 0.0;
        if constexpr (DW) {
          // Between the two barriers every warp but one would idle: the tile's derivative
          // (warp dw), the loss terms of the PREVIOUS tile (warp lw) and the running loss
          // sum over the tile before that (warp 0, which also issued the refill above) all
          // go there, so that after the second barrier the warps carry equal work.
          const int ip = (int)(i & 1);
          const int dw = 1 + rot, lw = 1 + (rot + 1 == NW - 1 ? 0 : rot + 1);
          if (wid == dw) {
            // two-class softmax, logistic form (mirror_logistic_row): s = lg
            const double lg = row_logit();
            const int lab = (int)tcur;
            const double q = hexp_nonpos(-fabs(lg));  // = hexp, branch-free
            const double den = 1.0 + q;
            const double p0 = (lg > 0.0 ? q : 1.0) / den;
            const double prw = lab == 0 ? p0 - 1.0 : p0;
            if (lane < NV) {
              *reinterpret_cast<double2*>(dsh + 2 * lane) = make_double2(prw, __dmul_rn(prw, 0x1.0p896));  // |prw| <= 1: exact
              *reinterpret_cast<double2*>(dsh + 2 * R + ip * 2 * R + 2 * lane) = make_double2(lab == 0 ? lg : -lg, den);
            }
          }
          if (wid == lw && i > 0 && lane < NV) {
            const double2 ad = *reinterpret_cast<const double2*>(dsh + 2 * R + (ip ^ 1) * 2 * R + 2 * lane);
            lts[(ip ^ 1) * R + lane] = (ad.x > 0.0 ? ad.x : 0.0) + hlog_1to2(ad.y);  // = hlog on [1, 2]
          }
          if (wid == 0 && i > 1) {
            const double* lp = lts + ip * R;  // tile i - 2: full, its terms written one tile ago
#pragma unroll
            for (int r = 0; r < R; ++r) la = la + lp[r];
          }
          rot = rot + 1 == NW - 1 ? 0 : rot + 1;
          __syncthreads();
        } else if constexpr (CC == 1) {
          const double lg = row_logit();
          pr = lg - tcur;
          lt = __dmul_rn(__dmul_rn(0.5, pr), pr);
        } else {
          // two-class softmax, logistic form (mirror_logistic_row): s = lg
          const double lg = row_logit();
          const int lab = (int)tcur;
          const double q = hexp_nonpos(-fabs(lg));  // = hexp, branch-free
          const double den = 1.0 + q;
          const double p0 = (lg > 0.0 ? q : 1.0) / den;
          pr = lab == 0 ? p0 - 1.0 : p0;
          if constexpr (SC && !MIXED) pr = __dmul_rn(pr, 0x1.0p896);  // |pr| <= 1: exact
          {
            const double a = lab == 0 ? lg : -lg;
            const double lterm = (a > 0.0 ? a : 0.0) + hlog_1to2(den);  // = hlog on [1, 2]
            if (lane < NV) lts[(jseq & 1) * R + lane] = lterm;
          }
          if (wid == 0 && i > 0) {
            const double* lp = lts + ((jseq - 1) & 1) * R;  // previous tile: full
#pragma unroll
            for (int r = 0; r < R; ++r) la = la + lp[r];
          }
        }
        double dlr[DW ? 1 : NV], dls[!DW && SC && MIXED ? NV : 1];
        if constexpr (!DW) {
#pragma unroll
          for (int v = 0; v < NV; ++v) dlr[v] = __shfl_sync(0xffffffffu, pr, v);
          if constexpr (SC && MIXED) {
#pragma unroll
            for (int v = 0; v < NV; ++v) dls[v] = __dmul_rn(dlr[v], 0x1.0p896);  // odd features: scaled domain
          }
        }
        if (CC == 1 && wid == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double t = __shfl_sync(0xffffffffu, lt, r);
            if (FULL || r < nr) la = la + t;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (FULL || r < nr) {
            if constexpr (RR) load_row(r, xr[0]);
            double dl_r, dl_s;  // row r's derivative, plain and in the 2^896-scaled domain (odd features)
            if constexpr (DW) {
              const double2 t2 = *reinterpret_cast<const double2*>(dsh + 2 * r);  // broadcast
              dl_r = t2.x;
              dl_s = t2.y;
            } else {
              dl_r = dlr[r];
              dl_s = dls[SC && MIXED ? r : 0];
            }
#pragma unroll
            for (int k = 0; k < NG; ++k)
#pragma unroll
              for (int q = 0; q < V; ++q)
                gacc[k][q] = fma((SC && MIXED && k1_scaled_feature(q)) ? dl_s : dl_r, xr[RR ? 0 : r][k][q],
                                 gacc[k][q]);
          }
        }
      };
      if (nr == R) body(BoolTag<true>{});
      else body(BoolTag<false>{});
    }
    if constexpr (DW) {  // drain: the last tile's loss terms, the sums over the last two tiles
      __syncthreads();
      const int lp1 = (int)((ntile - 1) & 1);
      if (ntile > 0) {
        if (wid == 1 && lane < NV) {
          const double2 ad = *reinterpret_cast<const double2*>(dsh + 2 * R + lp1 * 2 * R + 2 * lane);
          lts[lp1 * R + lane] = (ad.x > 0.0 ? ad.x : 0.0) + hlog_1to2(ad.y);
        }
        if (wid == 0 && ntile > 1) {
          const double* lp = lts + (lp1 ^ 1) * R;
#pragma unroll
          for (int r = 0; r < R; ++r) la = la + lp[r];
        }
      }
      __syncthreads();
      if (wid == 0 && ntile > 0) {
        const int nr_last = (int)(r1 - (r0 + (ntile - 1) * R));
        const double* lp = lts + lp1 * R;
        for (int r = 0; r < nr_last; ++r) la = la + lp[r];
      }
    } else if constexpr (CC == 2) {  // the split's last tile's loss terms
      __syncthreads();
      if (wid == 0 && ntile > 0) {
        const int nr_last = (int)(r1 - (r0 + (ntile - 1) * R));
        const double* lp = lts + ((jseq - 1) & 1) * R;
        for (int r = 0; r < nr_last; ++r) la = la + lp[r];
      }
    }

    double* out = p.partials + (size_t)ls * (D + 1);
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const int g = tid + k * T1;
      if (gval[k]) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const int j = g * V + q;
          if (j < d) {
            out[j] = gacc[k][q];
            if (CC == 2) out[(size_t)d + j] = -gacc[k][q];  // class 1 = -class 0, exactly
          }
        }
      }
    }
    if (tid == 0) out[D] = la;
  }
  };
  if (scaled) run(BoolTag<true>{});
  else run(BoolTag<false>{});
}

// ------------------------------------------------------------------ dispatch
namespace {

template <class Tx, int CC, int NW, int NG, int R, int STAGES, bool FULLG>
cudaError_t launch_stream_k(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  auto kern = k1_stream<Tx, CC, NW, NG, R, STAGES, FULLG>;
  const size_t smem = stream_smem_bytes(L.ld, (int)sizeof(Tx), NW, R, CC, STAGES);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem)) != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int grid = sms * per_sm;
  if (grid > L.nsplit_local) grid = L.nsplit_local;
  if (L.dry) return cudaSuccess;
  kern<<<grid, NW * 32, smem, st>>>(p, L.nsplit_local);
  return cudaGetLastError();
}

template <class Tx, int CC, int NW, int NG, int R, int STAGES>
cudaError_t launch_stream_f(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  constexpr int V = VecK<Tx>::V;
  const bool fullg = ((p.d + V - 1) / V) == NG * NW * 32;
  if (fullg) return launch_stream_k<Tx, CC, NW, NG, R, STAGES, true>(L, p, st);
  return launch_stream_k<Tx, CC, NW, NG, R, STAGES, false>(L, p, st);
}

// planned shapes (plan_for): key = NW*10000 + NG*1000 + R*10 + STAGES
template <class Tx, int CC>
cudaError_t launch_stream_cc(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  const int nw = L.threads / 32;
  switch (nw * 10000 + L.ng * 1000 + L.rows * 10 + L.stages) {
#define HALP_STREAM_CASE(NW, NG, R, ST) \
  case NW * 10000 + NG * 1000 + R * 10 + ST: return launch_stream_f<Tx, CC, NW, NG, R, ST>(L, p, st);
    HALP_STREAM_SHAPES(HALP_STREAM_CASE)
#undef HALP_STREAM_CASE
    default: return cudaErrorInvalidConfiguration;
  }
}

}  // namespace

// The instantiations are split by element type over three translation units
// (k_fullgrad_stream_{f64,f32,bf16}.cu define HALP_STREAM_TU = 0 / 1 / 2 and include this
// file) so that they compile in parallel; without the macro this file is the whole kernel.
cudaError_t launch_stream_f64(const FgLaunch& L, const FgParams& p, cudaStream_t st);
cudaError_t launch_stream_f32(const FgLaunch& L, const FgParams& p, cudaStream_t st);
cudaError_t launch_stream_bf16(const FgLaunch& L, const FgParams& p, cudaStream_t st);

#if !defined(HALP_STREAM_TU) || HALP_STREAM_TU == 0
cudaError_t launch_stream_f64(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if (p.C == 1) return launch_stream_cc<double, 1>(L, p, st);
  if (p.C == 2) return launch_stream_cc<double, 2>(L, p, st);
  return cudaErrorInvalidConfiguration;
}
#endif
#if !defined(HALP_STREAM_TU) || HALP_STREAM_TU == 2
cudaError_t launch_stream_bf16(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if (p.C == 1) return launch_stream_cc<__nv_bfloat16, 1>(L, p, st);
  if (p.C == 2) return launch_stream_cc<__nv_bfloat16, 2>(L, p, st);
  return cudaErrorInvalidConfiguration;
}
#endif
#if !defined(HALP_STREAM_TU) || HALP_STREAM_TU == 1
cudaError_t launch_stream_f32(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  if (p.C == 1) return launch_stream_cc<float, 1>(L, p, st);
  if (p.C == 2) return launch_stream_cc<float, 2>(L, p, st);
  return cudaErrorInvalidConfiguration;
}

size_t stream_smem_bytes(int ld, int elem, int warps, int R, int CC, int stages) {
  size_t b = (size_t)stages * R * ld * elem;
  b = (b + 15) / 16 * 16;
  (void)CC;
  b += (size_t)2 * warps * R * 8 + (size_t)2 * warps * R * 8 + (size_t)6 * R * 8 + (size_t)stages * 8;
  return b;
}

cudaError_t launch_fullgrad_stream(const FgLaunch& L, const FgParams& p, cudaStream_t st) {
  switch (L.dtype) {
    case 0: return launch_stream_f64(L, p, st);
    case 1: return launch_stream_f32(L, p, st);
    case 2: return launch_stream_bf16(L, p, st);
    default: return cudaErrorInvalidConfiguration;
  }
}
#endif

}  // namespace halp
