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
// contiguous coordinates [tau*M, tau*M + M).  w~, g~ and the codes of z live
// in registers for the whole epoch; the sampled row x_i is prefetched two
// steps ahead.
//
// Rounding stream: the reference's xorshift64* stream 1, reproduced exactly.
// Coordinate k of step t uses draw  D*(t+1) + k  of the epoch: each thread
// steps its M draws and jumps D draws per step with the GF(2) table of X^D
// held in shared memory -- inside the exchange wait, where it costs nothing
// (streaming precomputed uniforms from HBM measured ~0.4 us/step slower).
//
// Per step, ONE exchange: each warp reduces its partial logits with an
// xor-butterfly reduce-scatter and sends them (with its non-finite flag of the
// previous step) to every CTA of the cluster with st.async, completing on the
// receiver's mbarrier (no cluster barrier); a single CTA uses shared memory +
// __syncthreads.  Then EVERY warp combines the partials and evaluates the loss
// derivative itself (lane-parallel softmax: lane c = class c at wz, lane 16+c
// = at w~), so nothing is broadcast through a second barrier.
//
// Reduction order (mirrored by oracle MIRROR mode): thread partial =
// sequential fma over its coordinates; warp = xor butterfly 16..1; across
// warps, squared loss (C == 1): lane l sums warps l, l+32, ... sequentially,
// then a lane butterfly; softmax (C >= 2): sequential over the warps holding
// the class, in global warp order; the softmax denominator is a pairwise tree
// over 16 class slots (zero padded).
#include <algorithm>
#include <cstdio>

#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

constexpr int kMaxWarpsPerCluster = 128;

// developer build only (-DHALP_K3_PROF): per-phase clock64 split of one warp
#ifdef HALP_K3_PROF
#define K3_MARK(i)                         \
  do {                                     \
    if (prof_on) {                         \
      const long long c_ = clock64();      \
      prof_acc[i] += c_ - prof_last;       \
      prof_last = c_;                      \
    }                                      \
  } while (0)
#else
#define K3_MARK(i) \
  do {             \
  } while (0)
#endif

#ifndef HALP_K3_WAIT
#define HALP_K3_WAIT 0  // 0: relaxed cluster-scope wait + shared::cluster acquire fence; 1: default (acquire, CTA scope) wait
#endif
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
#if HALP_K3_WAIT == 1
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  // the payload arrived by st.async into OUR shared memory: an acquire restricted
  // to shared::cluster suffices (a plain .acquire.cluster wait also invalidates L1)
  asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
#endif
}
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
  return ra;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2f64(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}

__device__ __forceinline__ void st_async_v2s64(uint32_t raddr, long long a, long long b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(a), "l"(b), "r"(rbar)
               : "memory");
}

// exact warp sum of one int64 per lane whose absolute values sum to < 2^61 over
// the warp: three 21-bit limbs through REDUX.SUM (32-bit), recombined
__device__ __forceinline__ long long warp_sum_s64(long long v) {
  const int lo = __reduce_add_sync(0xffffffffu, (int)(v & 0x1FFFFF));
  const int mi = __reduce_add_sync(0xffffffffu, (int)((v >> 21) & 0x1FFFFF));
  const int hi = __reduce_add_sync(0xffffffffu, (int)(v >> 42));
  return (long long)hi * (1LL << 42) + (long long)mi * (1LL << 21) + (long long)lo;
}

// fire-and-forget prefetch of a line into L2 (no destination register, no scoreboard)
__device__ __forceinline__ void prefetch_l2(const void* g) { asm volatile("prefetch.global.L2 [%0];" ::"l"(g)); }

// the M raw elements x[fj[i]] of a row (one vector load when they are
// contiguous and aligned, else one load per coordinate)
template <class Tx, int M>
__device__ __forceinline__ void load_row_m(const Tx* row, const int (&fj)[M], bool vec, Tx (&o)[M]) {
  constexpr int B = M * (int)sizeof(Tx);
  if constexpr (B == 16) {
    if (vec) {
      const uint4 r = *reinterpret_cast<const uint4*>(row + fj[0]);
      const Tx* q = reinterpret_cast<const Tx*>(&r);
#pragma unroll
      for (int i = 0; i < M; ++i) o[i] = q[i];
      return;
    }
  } else if constexpr (B == 8) {
    if (vec) {
      const uint2 r = *reinterpret_cast<const uint2*>(row + fj[0]);
      const Tx* q = reinterpret_cast<const Tx*>(&r);
#pragma unroll
      for (int i = 0; i < M; ++i) o[i] = q[i];
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) o[i] = row[fj[i]];
}


// store M doubles (vectorised when all are valid; M*8-byte aligned by layout)
template <int M>
__device__ __forceinline__ void store_m(double* dst, const double (&v)[M], const bool (&valid)[M], bool allv) {
  if constexpr (M >= 2) {
    if (allv) {
#pragma unroll
      for (int i = 0; i < M; i += 2) *reinterpret_cast<double2*>(dst + i) = make_double2(v[i], v[i + 1]);
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i)
    if (valid[i]) dst[i] = v[i];
}

// KIND 0: squared loss (C == 1), one (wz, w~) pair per warp.
// KIND 1: softmax, every warp's 32*M coordinates touch at most two classes
//         (32*M <= d): two pairs per warp.
// KIND 2: softmax with small d: 2*C slots per warp.
template <int KIND>
struct K3Layout {
  static constexpr int NSLOT = KIND == 0 ? 2 : KIND == 1 ? 4 : 32;  // doubles per warp record
  static constexpr int FLAG = KIND == 2 ? 31 : -1;                  // explicit flag slot (KIND 2)
};
// KIND 0/1 carry the blowup flag in-band: a warp whose previous update was
// non-finite sends this signalling-NaN pattern in place of all its partials
// (arithmetic never produces it; NaN logits make receivers rescan for it).
constexpr long long kFlagBits = 0x7FF4A1B2C3D4E5F6LL;
// FX records (integer sums, |sum| < 2^60) carry it as values no sum can take:
// the sender's previous update was non-finite / one of its partials is not finite
constexpr long long kFxFlag = (long long)0x8000000000000001ULL, kFxNan = (long long)0x8000000000000002ULL;

// FAST (HALP, squared loss, plain exchange): every coordinate slot is a real coordinate
// (D = threads * M), no option-II snapshot, no code trace, the reciprocal quantizer applies --
// the launcher checks it; the per-step predicates and selects of those cases compile away.
// PF2 (FAST only): rows are also pulled into L2 one step before their register prefetch, for
// datasets that do not stay in L2 (C3: 0.924 -> 0.860 us/step; an L2-resident X is 4% slower
// with it, so the launcher decides by size).
template <class Tx, int M, bool CL, int KIND, bool BASE0, bool LV2, bool FX, bool FAST = false, bool PF2 = false>
__global__ void __launch_bounds__(256, 1) k3_inner(InParams p) {
  static_assert(!PF2 || FAST, "L2 prefetch: fast path only");
  static_assert(!FAST || (KIND == 0 && !BASE0 && !LV2 && !FX), "fast path: HALP squared loss, fp64 records");
  static_assert(!LV2 || (KIND == 0 && CL), "two-level exchange: squared loss on a cluster");
  static_assert(!FX || (KIND == 0 && !BASE0 && !LV2), "fixed-point exchange: HALP squared loss");
  constexpr int NSLOT = K3Layout<KIND>::NSLOT;
  constexpr int FLAG = K3Layout<KIND>::FLAG;
  constexpr bool SQ = KIND == 0;
  __shared__ uint64_t jt[2048];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(16) double gsc[2][8][32];  // softmax gathers: [parity][warp][lane]
  __shared__ __align__(16) double ctar[2][8][2];  // LV2: this CTA's warp records [parity][warp]
  extern __shared__ __align__(16) double xbuf_dyn[];  // [2][NGW][NSLOT]

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  const uint32_t rank = CL ? cluster_ctarank() : 0u;
  const int NC = CL ? (int)gridDim.x : 1;
  const int NGW = NC * NW;
  const int gw = (int)rank * NW + wid;
  const int NREC = LV2 ? NC : NGW;  // records per exchange (LV2: one per CTA)
  const int d = p.d, C = p.C, D = p.D, ld = p.ld;
  const int64_t k0 = ((int64_t)rank * blockDim.x + tid) * M;
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  const double delta = p.delta, alpha = p.alpha, l2 = p.l2, rcp = p.rcp;
  const int WC = 32 * M;  // coordinates per warp
  const int PAR_STRIDE = NGW * NSLOT;  // doubles between the two parity buffers
  auto XB = [&](int par_, int q_, int slot_) -> double& { return xbuf_dyn[par_ * PAR_STRIDE + q_ * NSLOT + slot_]; };
  const uint32_t bytes_step = KIND == 0 ? (uint32_t)NREC * 16u
                              : KIND == 1 ? (uint32_t)NGW * 32u
                                          : (uint32_t)NGW * (uint32_t)(2 * C + 1) * 8u;

  for (int i = tid; i < 2048; i += blockDim.x) jt[i] = p.jump_tab[i];
  if (CL && tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }

  // Remote targets of this lane's st.async messages, fixed for the epoch
  // (parity 1 = parity 0 + a constant offset in every CTA's window).
  //   KIND 0: lanes 0..15 send the pair to CTA lane.
  //   KIND 1: lanes with (lane & 8) == 0 send pair 2*(lane>>4) to CTAs
  //           (lane & 7) and (lane & 7) + 8.
  uint32_t ra0 = 0, ra1 = 0, rb0 = 0, rb1 = 0;
  bool s0ok = false, s1ok = false;
  const uint32_t xb_par_off = (uint32_t)(PAR_STRIDE * 8), mb_par_off = 8u;
  if (CL && KIND == 0) {
    const int r0 = lane & 15;
    s0ok = lane < 16 && r0 < NC;
    ra0 = mapa_u32(&XB(0, LV2 ? (int)rank : gw, 0), (uint32_t)(s0ok ? r0 : 0));
    rb0 = mapa_u32(&mbar[0], (uint32_t)(s0ok ? r0 : 0));
  } else if (CL && KIND == 1) {
    const int slot = 2 * (lane >> 4);
    const bool sender = !(lane & 8);
    const int r0 = lane & 7, r1 = (lane & 7) + 8;
    s0ok = sender && r0 < NC;
    s1ok = sender && r1 < NC;
    ra0 = mapa_u32(&XB(0, gw, slot), (uint32_t)(s0ok ? r0 : 0));
    ra1 = mapa_u32(&XB(0, gw, slot), (uint32_t)(s1ok ? r1 : 0));
    rb0 = mapa_u32(&mbar[0], (uint32_t)(s0ok ? r0 : 0));
    rb1 = mapa_u32(&mbar[0], (uint32_t)(s1ok ? r1 : 0));
  }

  // class of this warp's first coordinate (warp-uniform, KIND 1 split point)
  const int64_t wk0 = (int64_t)gw * WC;
  const int cw0 = (int)(wk0 < D ? wk0 / d : 0);

  // per-lane plan of the cross-warp logit sum (softmax): lane hc (+16 for w~)
  // reads the records of warps q_first..q_last, as offsets from its parity base
  const int hc = lane & 15;
  const int isw = (lane >> 4) & 1;
  int nq = 0, off_first = 0, off_rest = 0;
  if (!SQ && hc < C) {
    const int q_first = (int)(((int64_t)hc * d) / WC);
    const int q_last = (int)((((int64_t)hc + 1) * d - 1) / WC);
    int slot_first, slot_rest;
    if (KIND == 1) {
      const int c_of_first = (int)(((int64_t)q_first * WC) / d);
      slot_first = (c_of_first == hc ? 0 : 2) + isw;
      slot_rest = isw;
    } else {
      slot_first = slot_rest = 2 * hc + isw;
    }
    nq = q_last - q_first + 1;
    off_first = q_first * NSLOT + slot_first;
    off_rest = q_first * NSLOT + slot_rest;
  }

  double wt[M], gt[M], l2w[M], up[M], upp[M], Ua[M];  // up: u of this step, upp: of the previous one
  Tx xa[M], xb[M];
  double code[M], snap[M];  // z codes as exact doubles (|code| <= 2^(bits-1))
  const bool wide = p.hi > 0x1.0p53;
  int cls[M], fj[M];
  bool valid[M];
  bool allv = true;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    const int64_t k = k0 + i;
    valid[i] = FAST || k < D;
    allv = allv && valid[i];
    cls[i] = valid[i] ? (int)(k / d) : 0;
    fj[i] = valid[i] ? (int)(k % d) : 0;
    wt[i] = valid[i] ? p.w[k] : 0.0;
    gt[i] = valid[i] ? p.g[k] : 0.0;
    l2w[i] = __dmul_rn(l2, wt[i]);
    code[i] = (BASE0 && valid[i] && p.z0) ? p.z0[k] : 0.0;
    snap[i] = code[i];
    up[i] = 0.0;
    upp[i] = 0.0;
    Ua[i] = 0.0;
  }
  const int cA = cls[0];
  int cB = cA;
#pragma unroll
  for (int i = 0; i < M; ++i)
    if (valid[i]) cB = cls[i];
  const bool oneclass = __all_sync(0xffffffffu, cB == cA);
  // KIND 1: does this warp straddle two classes? (else a1 = b1 = 0 always)
  const bool wsplit = KIND == 1 && !__all_sync(0xffffffffu, !valid[0] || (cA == cw0 && cB == cw0));
  // vector row loads when the thread's coordinates are aligned and in one class
  const bool vecx = (d % M == 0) && (ld % M == 0);
  const int64_t T = p.T;
  // HALP: wz = w~ + z; LP-SVRG / SVRG / SGD / LP-SGD (BASE0 instantiations): the iterate is z itself
  constexpr bool base0 = BASE0;
  const bool fp_inner = BASE0 && (p.mode == 2 || p.mode == 3);  // SVRG, SGD: fp64 iterate
  const bool plain = BASE0 && (p.mode == 3 || p.mode == 4);     // SGD, LP-SGD: u = w - alpha*g
  uint64_t rs = jump_count(p.rstate0, (uint64_t)(k0 < D ? k0 : 0), p.pow_tab);

  // rows of steps 0 and 1 in flight (raw), the index of step 2 loaded
  int64_t row0 = p.idx[0];
  int64_t row1 = T > 1 ? p.idx[1] : row0;
  int64_t row2 = T > 2 ? p.idx[2] : row1;
  load_row_m<Tx, M>(X + row0 * ld, fj, vecx, xa);
  load_row_m<Tx, M>(X + row1 * ld, fj, vecx, xb);
  double yv = SQ ? p.y[row0] : 0.0, ynext = SQ ? p.y[row1] : 0.0;
  int lab = SQ ? 0 : p.labels[row0], labnext = SQ ? 0 : p.labels[row1];
  // one step further ahead the row (and its target) is only pulled into L2: the exchange's
  // acquire fence waits on all scoreboards, so the register prefetch above covers ~one exchange
  // (enough for an L2 hit, not for an HBM access); prefetch.global.L2 holds no scoreboard
  int64_t row3 = T > 3 ? p.idx[3] : row2;

  __syncthreads();
  if (CL) cluster_sync_all();

  int bad_prev = 0;
#ifdef HALP_K3_PROF
  const bool prof_on = rank == 0 && tid == 0;
  long long prof_acc[16] = {}, prof_last = clock64();
#endif
  for (int64_t t = 0; t <= T; ++t) {
    K3_MARK(7);
    if constexpr (FAST) {
      // the exchange after the last step only carries step T-1's blow-up flag: handled here,
      // so `last` is a compile-time false in the step below
      if (t == T) {
        const int parL = (int)(t & 1);
        if (CL && tid == 0) mbar_expect_tx(&mbar[parL], bytes_step);
        const double vL = __any_sync(0xffffffffu, bad_prev) ? __longlong_as_double(kFlagBits) : 0.0;
        if (CL) {
          if (s0ok) st_async_v2f64(ra0 + (parL ? xb_par_off : 0u), vL, vL, rb0 + (parL ? mb_par_off : 0u));
          mbar_wait_cluster(&mbar[parL], (uint32_t)((t >> 1) & 1));
        } else {
          if (lane == 0) *reinterpret_cast<double2*>(&XB(parL, gw, 0)) = make_double2(vL, vL);
          __syncthreads();
        }
        const double* xbL = xbuf_dyn + parL * PAR_STRIDE;
        int f = 0;
#pragma unroll
        for (int j = 0; j < kMaxWarpsPerCluster / 32; ++j) {
          const int q = lane + 32 * j;
          if (q < NREC) f |= __double_as_longlong(xbL[q * NSLOT]) == kFlagBits;
        }
        if (__any_sync(0xffffffffu, f)) {
          store_m<M>(p.u_out + k0, up, valid, allv);  // u of step T-1
          if (rank == 0 && tid == 0) *p.blow_step = (long long)(t - 1);
          if (CL) cluster_sync_all();
          return;
        }
        break;
      }
    }
    const bool last = FAST ? false : (t == T);
    const int par = (int)(t & 1);
    if (CL && tid == 0) mbar_expect_tx(&mbar[par], bytes_step);
    double xc[M];
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    if (!last) {
      if (!FAST && t == p.t_pick) {
#pragma unroll
        for (int i = 0; i < M; ++i) snap[i] = code[i];
      }
#pragma unroll
      for (int i = 0; i < M; ++i) {
        xc[i] = to_d<Tx>(xa[i]);
        xa[i] = xb[i];
      }
      if (t + 2 < T) load_row_m<Tx, M>(X + row2 * ld, fj, vecx, xb);  // raw prefetch, step t+2
      if constexpr (PF2) {
        if (t + 3 < T) {  // L2 prefetch, step t+3
          prefetch_l2(X + row3 * ld + fj[0]);
          if (SQ) prefetch_l2(p.y + row3);
        }
      }
      const int cS = KIND == 1 ? cw0 : cA;
      if (SQ || (KIND == 1 && !wsplit)) {  // single-class warp: one pair
#pragma unroll
        for (int i = 0; i < M; ++i) {
          if (!valid[i]) continue;
          const double zz = __dmul_rn(code[i], delta);
          const double wz = base0 ? zz : wt[i] + zz;
          a0 = fma(xc[i], wz, a0);
          b0 = fma(xc[i], wt[i], b0);
        }
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
          if (!valid[i]) continue;
          const double zz = __dmul_rn(code[i], delta);
          const double wz = base0 ? zz : wt[i] + zz;
          if (cls[i] == cS) {
            a0 = fma(xc[i], wz, a0);
            b0 = fma(xc[i], wt[i], b0);
          } else {
            a1 = fma(xc[i], wz, a1);
            b1 = fma(xc[i], wt[i], b1);
          }
        }
      }
    }
    K3_MARK(0);
    const bool flag = __any_sync(0xffffffffu, bad_prev);
    const double flagv = flag ? 1.0 : 0.0;
    const double fnan = __longlong_as_double(kFlagBits);
    if constexpr (FX) {
      // fixed point: every thread's partials rounded to integers at 2^S (S from a
      // bound on |x| |w~ + z| chosen per epoch so no sum can reach 2^60), the warp
      // sums by REDUX on 21-bit limbs, one integer record per warp to every CTA --
      // integer sums are exact, so the order of the combine is irrelevant
      const bool nanp = !(isfinite(a0) && isfinite(b0));
      const long long A = nanp ? 0 : __double2ll_rn(__dmul_rn(a0, p.fx_scale));
      const long long B = nanp ? 0 : __double2ll_rn(__dmul_rn(b0, p.fx_scale));
      long long SA = warp_sum_s64(A);
      const long long SB = warp_sum_s64(B);
      if (__any_sync(0xffffffffu, nanp)) SA = kFxNan;
      if (flag) SA = kFxFlag;
      if (CL) {
        const uint32_t xo = par ? xb_par_off : 0u, mo = par ? mb_par_off : 0u;
        if (s0ok) st_async_v2s64(ra0 + xo, SA, SB, rb0 + mo);
      } else {
        if (lane == 0) *reinterpret_cast<longlong2*>(&XB(par, gw, 0)) = make_longlong2(SA, SB);
      }
    } else if constexpr (KIND == 0) {
      // all-reduce butterfly of a0 on lanes 0..15 and of b0 on lanes 16..31
      const bool u16 = (lane & 16) != 0;
      double v = (u16 ? b0 : a0) + __shfl_xor_sync(0xffffffffu, u16 ? a0 : b0, 16);
      v = v + __shfl_xor_sync(0xffffffffu, v, 8);
      v = v + __shfl_xor_sync(0xffffffffu, v, 4);
      v = v + __shfl_xor_sync(0xffffffffu, v, 2);
      v = v + __shfl_xor_sync(0xffffffffu, v, 1);
      double vp = __shfl_xor_sync(0xffffffffu, v, 16);
      if (flag) v = vp = fnan;
      if constexpr (LV2) {
        // this CTA's warps summed in order by warp 0, one record per CTA to every CTA
        if (lane == 0) *reinterpret_cast<double2*>(&ctar[par][wid][0]) = make_double2(v, vp);
        asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
        if (wid == 0) {
          double2 r = *reinterpret_cast<const double2*>(&ctar[par][0][0]);
          bool fl2 = __double_as_longlong(r.x) == kFlagBits;
          for (int q = 1; q < NW; ++q) {
            const double2 rq = *reinterpret_cast<const double2*>(&ctar[par][q][0]);
            fl2 |= __double_as_longlong(rq.x) == kFlagBits;
            r.x = r.x + rq.x;
            r.y = r.y + rq.y;
          }
          if (fl2) r.x = r.y = fnan;
          const uint32_t xo = par ? xb_par_off : 0u, mo = par ? mb_par_off : 0u;
          if (s0ok) st_async_v2f64(ra0 + xo, r.x, r.y, rb0 + mo);
        }
      } else if (CL) {
        const uint32_t xo = par ? xb_par_off : 0u, mo = par ? mb_par_off : 0u;
        if (s0ok) st_async_v2f64(ra0 + xo, v, vp, rb0 + mo);
      } else {
        if (lane == 0) *reinterpret_cast<double2*>(&XB(par, gw, 0)) = make_double2(v, vp);
      }
    } else if constexpr (KIND == 1) {
      // warp reduce-scatter of (a0, b0, a1, b1): 8-lane group g ends with slot g
      const bool u16 = (lane & 16) != 0;
      const double s0 = (u16 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, u16 ? a0 : a1, 16);
      const double s1 = (u16 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, u16 ? b0 : b1, 16);
      const bool u8 = (lane & 8) != 0;
      double v = (u8 ? s1 : s0) + __shfl_xor_sync(0xffffffffu, u8 ? s0 : s1, 8);
      v = v + __shfl_xor_sync(0xffffffffu, v, 4);
      v = v + __shfl_xor_sync(0xffffffffu, v, 2);
      v = v + __shfl_xor_sync(0xffffffffu, v, 1);
      double vp = __shfl_xor_sync(0xffffffffu, v, 8);  // pair g with g^1
      if (flag) v = vp = fnan;
      if (CL) {
        const uint32_t xo = par ? xb_par_off : 0u, mo = par ? mb_par_off : 0u;
        if (s0ok) st_async_v2f64(ra0 + xo, v, vp, rb0 + mo);
        if (s1ok) st_async_v2f64(ra1 + xo, v, vp, rb1 + mo);
      } else {
        if ((lane & 15) == 0) *reinterpret_cast<double2*>(&XB(par, gw, (lane >> 4) << 1)) = make_double2(v, vp);
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
      const bool sender = lane < 2 * C || lane == FLAG;
      const double val = lane == FLAG ? flagv : sl[0];
      if (sender) {
        if (CL) {
          for (int r = 0; r < NC; ++r)
            st_async_f64(mapa_u32(&XB(par, gw, lane), (uint32_t)r), val, mapa_u32(&mbar[par], (uint32_t)r));
        } else {
          XB(par, gw, lane) = val;
        }
      }
    }
    K3_MARK(1);
    // ---- work independent of the exchange, done while it is in flight ----
    if (!last && !fp_inner) {
      uint64_t s = rs;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        s = xs_step(s);
        Ua[i] = uniform_of(s);
      }
      rs = jump_tab(rs, jt);
    }
    K3_MARK(2);
    if (CL) mbar_wait_cluster(&mbar[par], (uint32_t)((t >> 1) & 1));
    else __syncthreads();
    K3_MARK(3);

    const double* xbp = xbuf_dyn + par * PAR_STRIDE;
    double fxa = 0.0, fxb = 0.0;
    if constexpr (FX) {
      // every lane sums its records (integers), the warp by REDUX; flag values are counted apart
      long long pa = 0, pb = 0;
      int fb = 0;
#pragma unroll
      for (int j = 0; j < kMaxWarpsPerCluster / 32; ++j) {
        const int q = lane + 32 * j;
        if (q < NREC) {
          const longlong2 v = *reinterpret_cast<const longlong2*>(xbp + q * NSLOT);
          const bool isf = v.x == kFxFlag, isn = v.x == kFxNan;
          fb |= (isf ? 1 : 0) | (isn ? 2 : 0);
          pa += (isf || isn) ? 0 : v.x;
          pb += v.y;
        }
      }
      fb = (int)__reduce_or_sync(0xffffffffu, (unsigned)fb);
      if (fb & 1) {  // some warp's previous update was non-finite: blow-up of step t-1
        store_m<M>(p.u_out + k0, up, valid, allv);  // no update yet at step t: up holds u of step t-1
        if (rank == 0 && tid == 0) *p.blow_step = (long long)(t - 1);
        if (CL) cluster_sync_all();
        return;
      }
      if (last) break;
      const long long da = warp_sum_s64(pa), db = warp_sum_s64(pb);
      const bool nanstep = (fb & 2) != 0;  // a partial was not finite: the reference's dot is NaN
      fxa = nanstep ? __longlong_as_double(0x7FF8000000000000LL) : __dmul_rn(__ll2double_rn(da), p.fx_inv);
      fxb = nanstep ? __longlong_as_double(0x7FF8000000000000LL) : __dmul_rn(__ll2double_rn(db), p.fx_inv);
    }
    // blowup of step t-1?  Tested after this step's update (a blowup leaves
    // code[] dead; u of step t-1 is kept in upp[] and stored only then).  KIND 0/1: a lane
    // whose partial sums came out NaN raises `cand`, and the records are then
    // scanned for the flag pattern (a NaN of this step's own is not a flag).
    auto flagged = [&]() -> bool {
      int f = 0;
#pragma unroll
      for (int j = 0; j < kMaxWarpsPerCluster / 32; ++j) {
        const int q = lane + 32 * j;
        if (q < NREC) {
          if constexpr (KIND == 2) f |= xbp[q * NSLOT + FLAG] != 0.0;
          else f |= __double_as_longlong(xbp[q * NSLOT]) == kFlagBits;
        }
      }
      return __any_sync(0xffffffffu, f);
    };
    int fl = 0;
    if constexpr (KIND == 2) {
#pragma unroll
      for (int j = 0; j < kMaxWarpsPerCluster / 32; ++j) {
        const int q = lane + 32 * j;
        if (q < NGW) fl |= xbp[q * NSLOT + FLAG] != 0.0;
      }
    }
    if (last) {
      if (flagged()) {
        store_m<M>(p.u_out + k0, up, valid, allv);  // u of step T-1 (no update at t == T)
        if (rank == 0 && tid == 0) *p.blow_step = (long long)(t - 1);
        if (CL) cluster_sync_all();  // nobody leaves while remote stores may target it
        return;
      }
      break;
    }
    K3_MARK(4);
    const double yi = yv;
    const int li = lab;
    row0 = row1;
    row1 = row2;
    yv = ynext;
    lab = labnext;
    if constexpr (PF2) {
      row2 = row3;
      if (t + 4 < T) row3 = p.idx[t + 4];
    } else {
      if (t + 3 < T) row2 = p.idx[t + 3];
    }
    if (t + 2 < T) {
      if (SQ) ynext = p.y[row1];
      else labnext = p.labels[row1];
    }

    // loss derivative at wz (p1) and at w~ (p2) for this thread's classes
    double p1A, p2A, p1B, p2B;
    if constexpr (FX) {
      p1A = p1B = fxa - yi;
      p2A = p2B = fxb - yi;
    } else if constexpr (SQ) {
      double sa = 0.0, sb = 0.0;
#pragma unroll
      for (int j = 0; j < kMaxWarpsPerCluster / 32; ++j) {
        const int q = lane + 32 * j;
        if (q < NREC) {
          const double2 v = *reinterpret_cast<const double2*>(xbp + q * NSLOT);
          sa = sa + v.x;
          sb = sb + v.y;
        }
      }
      fl = isnan(sa) || isnan(sb);
      K3_MARK(8);
      // lanes >= NREC hold +0.0: butterfly levels that only add zeros are skipped
      if (NREC >= 32) {  // every lane holds records: the full butterfly, unrolled (no loop branches)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          sa = sa + __shfl_xor_sync(0xffffffffu, sa, o);
          sb = sb + __shfl_xor_sync(0xffffffffu, sb, o);
        }
      } else {
        for (int o = NREC > 1 ? (1 << (31 - __clz(NREC - 1))) : 0; o >= 1; o >>= 1) {
          sa = sa + __shfl_xor_sync(0xffffffffu, sa, o);
          sb = sb + __shfl_xor_sync(0xffffffffu, sb, o);
        }
      }
      if (NREC < 32) {
        sa = __shfl_sync(0xffffffffu, sa, 0);
        sb = __shfl_sync(0xffffffffu, sb, 0);
      }
      p1A = p1B = sa - yi;
      p2A = p2B = sb - yi;
    } else {
      // loads first, then the in-order chain (absent warps add +0.0: exact)
      constexpr int QH = 8;
      double pv[QH];
      pv[0] = nq > 0 ? xbp[off_first] : 0.0;
#pragma unroll
      for (int j = 1; j < QH; ++j) pv[j] = j < nq ? xbp[off_rest + j * NSLOT] : 0.0;
      double lg = pv[0];
#pragma unroll
      for (int j = 1; j < QH; ++j) lg = lg + pv[j];
      for (int j = QH; j < nq; ++j) lg = lg + xbp[off_rest + j * NSLOT];
      if (KIND == 1) fl = isnan(lg);
      K3_MARK(8);
      // every lane gathers its half's 16 logits (one shuffle round) and takes
      // the max in registers; softmax sum = pairwise tree over 16 (zeros pad)
      const bool act = hc < C;
      // gathers through a per-warp shared scratch (parity double-buffered):
      // one store + 8 broadcast 16-byte loads instead of 32 shuffles
      double* gs = &gsc[par][wid][0];
      const double2* gh = reinterpret_cast<const double2*>(gs + (lane & 16));
      double mv[16];
      gs[lane] = act ? lg : -INFINITY;
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 v2 = gh[c];
        mv[2 * c] = v2.x;
        mv[2 * c + 1] = v2.y;
      }
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
        for (int c = 0; c < h; ++c) mv[c] = fmax(mv[c], mv[c + h]);
      const double mx = mv[0];
      K3_MARK(9);
      const double e = act ? hexp(lg - mx) : 0.0;
      K3_MARK(10);
      __syncwarp();
      double ev[16];
      gs[lane] = e;
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 v2 = gh[c];
        ev[2 * c] = v2.x;
        ev[2 * c + 1] = v2.y;
      }
#pragma unroll
      for (int h = 1; h < 16; h <<= 1)
#pragma unroll
        for (int c = 0; c < 16; c += 2 * h) ev[c] = ev[c] + ev[c + h];
      const double s = ev[0];
      K3_MARK(11);
      // lanes without a class divide 1 by s: 0 / s would leave the division's
      // fast path (the whole warp would wait on the slow one)
      double pr = (act ? e : 1.0) / s;
      K3_MARK(12);
      if (hc == li) pr = pr - 1.0;
      p1A = __shfl_sync(0xffffffffu, pr, cA);
      p2A = __shfl_sync(0xffffffffu, pr, 16 + cA);
      if (oneclass) {
        p1B = p1A;
        p2B = p2A;
      } else {
        p1B = __shfl_sync(0xffffffffu, pr, cB);
        p2B = __shfl_sync(0xffffffffu, pr, 16 + cB);
      }
    }
    K3_MARK(5);

    // ---- element-wise update + stochastic rounding (branch-free) ----
    bool bad = false, slow_any = false;
    bool slow[M] = {};
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const bool inA = cls[i] == cA;
      const double pp1 = inA ? p1A : p1B, pp2 = inA ? p2A : p2B;
      const double z = __dmul_rn(code[i], delta);
      const double wz = base0 ? z : wt[i] + z;
      const double g1 = __dmul_rn(pp1, xc[i]) + __dmul_rn(l2, wz);
      const double g2 = __dmul_rn(pp2, xc[i]) + l2w[i];
      const double u = plain ? z - __dmul_rn(alpha, g1) : z - __dmul_rn(alpha, (g1 - g2) + gt[i]);
      upp[i] = up[i];
      up[i] = u;
      bad |= valid[i] && !isfinite(u);
      code[i] = fp_inner ? u : quantize_fast(u, delta, rcp, p.hi, p.lo, Ua[i], slow[i]);
      slow_any |= !fp_inner && valid[i] && slow[i];
    }
    if (fp_inner) bad = false;  // SVRG / SGD: no finiteness check inside the epoch (optimizers.cpp:244-246, 283-286)
    if (!fp_inner && (slow_any || (!FAST && (wide || rcp == 0.0)))) {  // IEEE-division path for the rare operands
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i] && (slow[i] || (!FAST && (wide || rcp == 0.0))))
          code[i] = (double)quantize_code(up[i], delta, p.hi, p.lo, p.maxc, p.minc, Ua[i]);
    }
    if (__any_sync(0xffffffffu, fl) && (KIND == 2 || flagged())) {
      // the failing update is step t-1's, still in registers (no per-step store)
      store_m<M>(p.u_out + k0, upp, valid, allv);
      if (rank == 0 && tid == 0) *p.blow_step = (long long)(t - 1);
      if (CL) cluster_sync_all();  // nobody leaves while remote stores may target it
      return;
    }
    bad_prev = bad ? 1 : 0;
    K3_MARK(6);
    if (!FAST && t < p.trace_steps) {
#pragma unroll
      for (int i = 0; i < M; ++i)
        if (valid[i]) p.trace[t * D + k0 + i] = __double2ll_rn(code[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (!valid[i]) continue;
    const double zc = (!FAST && p.t_pick >= 0) ? snap[i] : code[i];
    const double zr = __dmul_rn(zc, delta);
    p.w_out[k0 + i] = base0 ? zr : wt[i] + zr;
    p.codes_out[k0 + i] = fp_inner ? 0 : __double2ll_rn(code[i]);
    if (BASE0 && p.zc_out) p.zc_out[k0 + i] = zc;
  }
#ifdef HALP_K3_PROF
  if (prof_on)
    printf("K3PROF T=%lld dot %.0f | send %.0f | rng %.0f | wait %.0f | flag %.0f | deriv %.0f | update %.0f | tail %.0f\n",
           (long long)T, prof_acc[0] / (double)T, prof_acc[1] / (double)T, prof_acc[2] / (double)T,
           prof_acc[3] / (double)T, prof_acc[4] / (double)T, prof_acc[5] / (double)T, prof_acc[6] / (double)T,
           prof_acc[7] / (double)T);
  if (prof_on)
    printf("K3PROF deriv split: sum %.0f | max %.0f | exp %.0f | csum %.0f | div %.0f | rest %.0f\n", prof_acc[8] / (double)T,
           prof_acc[9] / (double)T, prof_acc[10] / (double)T, prof_acc[11] / (double)T, prof_acc[12] / (double)T,
           prof_acc[5] / (double)T);
#endif
  if (CL) cluster_sync_all();  // keep every CTA's shared memory alive until all remote stores landed
}

template <class Tx, int M, int KIND, bool BASE0>
static cudaError_t launch_in_b(const InLaunch& L, const InParams& p, cudaStream_t st) {
  if (L.ctas * L.threads / 32 > kMaxWarpsPerCluster) return cudaErrorInvalidConfiguration;
  const size_t smem = sizeof(double) * 2 * (size_t)(L.ctas * L.threads / 32) * K3Layout<KIND>::NSLOT;
  // the common HALP least-squares launch: no dead slots, no snapshot, no trace, reciprocal quantizer.
  // Measured on B200 (profiles/r02_s4_k3_experiments.txt): 6-8% faster on cluster plans and on one
  // CTA with M = 4, 11% slower on one CTA with M = 2 (C1's plan), which keeps the general kernel.
  const bool fast = KIND == 0 && !BASE0 && L.levels <= 1 && (int64_t)p.D == (int64_t)L.ctas * L.threads * M &&
                    p.t_pick < 0 && p.trace_steps == 0 && !(p.hi > 0x1.0p53) && p.rcp != 0.0 &&
                    (L.ctas > 1 || M >= 4);
  // a dataset well beyond the 126 MB L2: pull the sampled rows into L2 a step early
  const bool pf2 = L.pf2 < 0 ? (double)p.n * p.ld * sizeof(Tx) > 256e6 : L.pf2 != 0;
  if (L.ctas == 1) {
    auto kern = k3_inner<Tx, M, false, KIND, BASE0, false, false>;
    if constexpr (KIND == 0 && !BASE0) {
      if (L.levels == 3) kern = k3_inner<Tx, M, false, KIND, BASE0, false, true>;
      else if (fast) kern = k3_inner<Tx, M, false, KIND, BASE0, false, false, true>;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (L.dry) return cudaSuccess;
    kern<<<1, L.threads, smem, st>>>(p);
    return cudaGetLastError();
  }
  if (L.ctas > 16) return cudaErrorInvalidConfiguration;
  auto kern = k3_inner<Tx, M, true, KIND, BASE0, false, false>;
  if constexpr (KIND == 0) {
    if (L.levels == 2) kern = k3_inner<Tx, M, true, KIND, BASE0, true, false>;
    if constexpr (!BASE0) {
      if (L.levels == 3) kern = k3_inner<Tx, M, true, KIND, BASE0, false, true>;
      else if (fast && pf2) kern = k3_inner<Tx, M, true, KIND, BASE0, false, false, true, true>;
      else if (fast) kern = k3_inner<Tx, M, true, KIND, BASE0, false, false, true>;
    }
  }
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
  if (L.dry) return cudaSuccess;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

// HALP (mode 0) and the base-0 modes (LP-SVRG, SVRG) are separate instantiations
template <class Tx, int M, int KIND>
static cudaError_t launch_in_t(const InLaunch& L, const InParams& p, cudaStream_t st) {
  if (p.mode == 0) return launch_in_b<Tx, M, KIND, false>(L, p, st);
  return launch_in_b<Tx, M, KIND, true>(L, p, st);
}

template <class Tx, int M>
static cudaError_t launch_in_kind(const InLaunch& L, const InParams& p, cudaStream_t st) {
  if (p.loss == 0) return launch_in_t<Tx, M, 0>(L, p, st);
  if (32 * M <= p.d) return launch_in_t<Tx, M, 1>(L, p, st);
  return launch_in_t<Tx, M, 2>(L, p, st);
}

template <class Tx>
static cudaError_t launch_in_dt(const InLaunch& L, const InParams& p, cudaStream_t st) {
  switch (L.per) {
    case 1: return launch_in_kind<Tx, 1>(L, p, st);
    case 2: return launch_in_kind<Tx, 2>(L, p, st);
    case 4: return launch_in_kind<Tx, 4>(L, p, st);
    default: return launch_in_kind<Tx, 8>(L, p, st);
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

namespace halp {

// max |x| of a matrix (FX exchange bound), one block-reduced atomic max on the
// double's bit pattern (non-negative doubles order like their integer bits)
template <class Tx>
__global__ void k_absmax(const Tx* __restrict__ X, int64_t elems, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < elems; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = fabs(to_d<Tx>(X[i]));
    m = (v > m || v != v) ? v : m;  // NaN wins (its bits sort above +inf's)
  }
  for (int o = 16; o >= 1; o >>= 1) {
    const double q = __shfl_xor_sync(0xffffffffu, m, o);
    m = (q > m || q != q) ? q : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

cudaError_t launch_absmax(const void* X, int dtype, int64_t elems, double* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  int blocks = (int)std::min<int64_t>((elems + 255) / 256, 148 * 8);
  if (blocks < 1) blocks = 1;
  auto* o = reinterpret_cast<unsigned long long*>(out);
  if (dtype == 0) k_absmax<double><<<blocks, 256, 0, st>>>(reinterpret_cast<const double*>(X), elems, o);
  else if (dtype == 1) k_absmax<float><<<blocks, 256, 0, st>>>(reinterpret_cast<const float*>(X), elems, o);
  else k_absmax<__nv_bfloat16><<<blocks, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(X), elems, o);
  return cudaGetLastError();
}

}  // namespace halp
