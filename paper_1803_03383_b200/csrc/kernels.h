// kernels.h -- host-visible launch interface of the HALP CUDA kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

namespace halp {

constexpr int kMaxClasses = 15;  // softmax classes handled by the inner-loop reduction slots

// ---- K1 full-gradient pass ----
struct FgParams {
  const void* X;
  int64_t n;
  int d, ld, C, loss;
  const double* y;
  const int32_t* labels;
  const double* w;
  int S, split0, c0, write_loss;
  double* partials;  // [nsplit_local][D+1]
  int x_finite;      // 1: X checked finite at creation (bf16 integer conversion allowed)
};
struct FgLaunch {
  int dtype, ng, ct, threads, ld, nsplit_local;
  int fast, rows, stages;  // fast: 0 generic, 3 softmax C >= 3, 4 streaming C <= 2; rows per tile, ring depth
  int dry;                 // 1: set the kernel's attributes (loads it under lazy module loading), no launch
};
size_t fg_smem_bytes(int ld, int elem, int D, int C, int threads, int R, int stages);
cudaError_t launch_fullgrad(const FgLaunch& L, const FgParams& p, cudaStream_t st);
// any non-finite element in a bf16 matrix (n x ld) -> *flag = 1 (flag zeroed by the caller)
cudaError_t launch_nonfinite_bf16(const void* X, int64_t elems, int* flag, cudaStream_t st);
// softmax with 3..15 classes (FgLaunch.fast == 3), k_fullgrad_smx.cu
size_t smx_smem_bytes(int ld, int elem, int d, int C, int threads, int64_t split_rows);
cudaError_t launch_fullgrad_smx(const FgLaunch& L, const FgParams& p, cudaStream_t st);
// streaming kernel for C <= 2 (FgLaunch.fast == 4), k_fullgrad_stream.cu.
// Instantiated shapes (NW warps, NG groups/thread, R rows/tile, ring depth);
// plan_for only picks shapes from this list.
#ifdef HALP_STREAM_DEV_SHAPES  // developer builds: the C4 and C3 shapes only (fast SASS experiments)
#define HALP_STREAM_SHAPES(X) X(4, 1, 16, 2) X(8, 4, 2, 4) X(8, 4, 4, 3) X(8, 2, 2, 4) X(8, 2, 4, 4) X(8, 2, 8, 3) X(8, 1, 4, 4)
#else
#define HALP_STREAM_SHAPES(X) \
  X(1, 1, 4, 4) X(1, 1, 8, 4) X(2, 1, 4, 4) X(2, 1, 8, 4) X(4, 1, 4, 4) X(4, 1, 8, 4) X(8, 1, 2, 4) \
  X(8, 1, 4, 4) X(16, 1, 2, 4) X(16, 1, 4, 4) X(8, 2, 2, 4) X(16, 2, 1, 4) X(16, 2, 2, 4) X(8, 4, 1, 4) \
  X(8, 4, 2, 4) X(16, 4, 1, 4) X(16, 2, 2, 6) X(8, 2, 2, 6) X(8, 4, 2, 6) X(4, 1, 4, 6) \
  X(4, 1, 16, 2) X(2, 1, 16, 2) X(1, 1, 16, 2) X(8, 4, 4, 3) X(8, 2, 4, 4) X(8, 2, 8, 3)
#endif
size_t stream_smem_bytes(int ld, int elem, int warps, int R, int CC, int stages);
cudaError_t launch_fullgrad_stream(const FgLaunch& L, const FgParams& p, cudaStream_t st);
cudaError_t launch_split_tree(const double* partials, int nsplit, int D1, double* out, double* scratch,
                              cudaStream_t st);

struct FinParams {
  const double* rank_sums;  // [G][D+1]
  int G, D;
  const double* w;
  int64_t n;
  double l2, mu, delta_min;
  int bits;
  double* g_out;  // [D]
  double* stats;  // [gn, delta, loss]
};
cudaError_t launch_finalize(const FinParams& p, cudaStream_t st);

cudaError_t launch_samples(uint64_t state0, int64_t total, int opt2, uint64_t T, uint64_t n, const uint64_t* pow_tab,
                           int64_t* idx, int64_t* tpick, cudaStream_t st);

// ---- K3 persistent inner loop (one problem, one CTA cluster) ----
struct InParams {
  const void* X;
  int ld, d, C, D, loss;
  int64_t n;
  const double* y;
  const int32_t* labels;
  double l2, alpha, delta, hi, lo;
  long long maxc, minc;
  double rcp;          // RN(1/delta), 0 => use IEEE division
  const double* w;     // w~ [D]
  double* w_out;       // w~ after the epoch [D]
  const double* g;     // g~ [D]
  const int64_t* idx;  // sample indices [T]
  int64_t T, t_pick;
  uint64_t rstate0;    // rounding-stream state before the first draw of step 0
  const uint64_t* pow_tab;
  const uint64_t* jump_tab;  // X^D, 8x256
  long long* codes_out;      // [D] codes after the last step
  long long* trace;          // [trace_steps][D] or null
  int64_t trace_steps;
  long long* blow_step;      // -1 or failing step index (64-bit: user T may exceed 2^31)
  double* u_out;             // [D] update vector of the failing step
  // algorithm: 0 HALP (wz = w~ + z, z = Q(u)), 1 LP-SVRG (fixed scale: the
  // iterate itself is quantized, wz = z), 2 SVRG (fp64 iterate in z, delta = 1,
  // no rounding, no blow-up check), 3 SGD / 4 LP-SGD (as 2 / 1 with
  // u = z - alpha*g1, no variance reduction); w is the anchor of g2
  int mode;
  const double* z0;          // [D] initial z values (code * delta units: codes) or null = 0
  double* zc_out;            // [D] codes of the epoch's result (snapshot under option II) or null
  // fixed-point exchange (InLaunch::levels == 3, HALP squared loss on a cluster):
  // thread partials rounded to integers at 2^fx_s, summed exactly as int64
  double fx_scale, fx_inv;   // 2^S, 2^-S
};
struct InLaunch {
  int dtype, ctas, threads, per, nslot_pow2;
  int dry;     // 1: load + configure the kernel only (see FgLaunch::dry)
  int levels;  // 1: warp records exchanged across the cluster; 2: combined per CTA first;
               // 3: fixed-point integer records (k_inner.cu FX)
  int pf2;     // fast path L2 prefetch of the sampled rows: -1 by dataset size, 0 off, 1 on (HALP_K3_PF2)
};
cudaError_t launch_inner(const InLaunch& L, const InParams& p, cudaStream_t st);
// max |x| over an n x ld matrix of the stored dtype -> *out (one double)
cudaError_t launch_absmax(const void* X, int dtype, int64_t elems, double* out, cudaStream_t st);

// ---- LM-HALP (k_lm.cu): K7 epoch stats over the quantized rows, K8 integer inner loop ----
constexpr int kLmMaxD = 4096;  // d*C over one 256-thread CTA, <= 16 coordinates per thread
struct LmStatsParams {
  const void* q;  // [n][d] codes (int8 for bits <= 8, int16 for bits <= 16)
  int64_t n;
  int d, C, loss;
  double delta_x;  // data scale
  const double* y;
  const int32_t* labels;
  const double* w;  // w~ [D]
  int S, split0;
  double* partials;  // [nsplit_local][D+1]
  double* phi;       // [n][C] logits at w~
};
cudaError_t launch_lm_stats(const LmStatsParams& p, int nblocks, int code_bytes, cudaStream_t st);
struct LmInnerParams {
  const void* q;
  int d, C, loss, bits;
  const double* phi;
  const double* y;
  const int32_t* labels;
  double alpha, daux, dm, sc;  // sc = delta_x * delta_m (dot_lp's scale)
  const long long* h;          // [D] codes of Q_i(alpha g~) at delta_inner
  const double* w;             // w~ [D]
  double* w_out;               // w~ + to_real(z) after the epoch
  const int64_t* idx;          // [T] sample indices
  int64_t T;
  uint64_t rstate0;            // rounding stream before the first draw of step 0
  const uint64_t* pow_tab;
  const uint64_t* jump_tab;    // X^(C(d+1))
  long long* trace;            // [trace_steps][D] z codes or null
  int64_t trace_steps;
  int* bad;                    // 1 if a beta was non-finite (quantize: input must be finite)
};
cudaError_t launch_lm_inner(const LmInnerParams& p, int code_bytes, cudaStream_t st);

// ---- K6 synthetic data ----
struct GenParams {
  int kind;
  int64_t n;
  int d, C, dtype;
  double noise_sd, x_scale, density;
  uint64_t seed;
  void* X;
  double* y;
  int32_t* labels;
};
cudaError_t launch_datagen(const GenParams& p, cudaStream_t st);

// ---- K5 batched independent problems ----
struct BatchParams {
  const void* X;        // [nprob][n][ld]
  int ld, d, dtype;
  int64_t n;
  int nprob;
  int64_t x_rows_per_prob;  // n (own data per problem) or 0 (one dataset shared by every problem)
  const double* y;      // [nprob][n] or [n]
  double l2;
  const double* alpha;  // per problem
  const double* mu;
  const double* delta_min;
  const double* div_limit;
  const double* metric_every;
  const int* bits;
  const int* epochs;
  const int* option;
  const int64_t* T;
  const uint64_t* seed;  // [nprob][2]: initial states of streams 0 and 1 (rng.hpp:29-32)
  const double* init;    // [nprob][d] or null
  const uint64_t* pow_tab;
  const uint64_t* jump_tab;  // X^d
  int splits, max_rows;
  double* rows;          // [nprob][max_rows][5]: pass, seconds, loss, grad_norm, delta
  uint64_t* rhash;       // [nprob][max_rows]
  int* rows_n;
  int* status;           // 0 ok, 1 converged, 2 diverged, 3 invalid delta
  int64_t* steps;
  double* w_out;         // [nprob][d] final iterate (the failing update on blow-up)
};
cudaError_t launch_batch(const BatchParams& p, int threads, cudaStream_t st);
// K5 plan: 1 = one warp per problem (k5_batch_w1, M = D/32 per lane), 2 / 4 =
// two / four warps (k5_batch, M = D/64 or D/128 per thread); HALP_K5_WARPS
// overrides.  Measured on B200 (tools/gpu_r2_lm.sh, gpu_r2_e2e.sh, gpu_r2_k3opt.sh):
// the 663-run 1000 x 64 grid 20.5-22.0 ms (1 warp) vs 27.0 (2) vs 35.9 (4); C5's
// 512 x (4096 x 128) 135 ms (1) vs 82.0 (2) vs 84.6 (4)
inline int batch_warps_per_problem(int d) {
  const char* e = std::getenv("HALP_K5_WARPS");
  if (e && (std::atoi(e) == 1 || std::atoi(e) == 2 || std::atoi(e) == 4)) return std::atoi(e);
  return d <= 64 ? 1 : d <= 128 ? 2 : 4;
}

}  // namespace halp
