/*
 * halp.h -- C ABI of the B200-native HALP solver (libhalp_b200.so).
 *
 * Drop-in boundary for the reference's solver entry point
 *     lpopt::RunRecord lpopt::run_halp(const Objective&, const OptimizerConfig&)
 *                                           proj/include/lpopt/optimizers.hpp:87
 * reached through lpopt::run(...) when cfg.algorithm == Algorithm::Halp
 *                                           proj/src/optimizers.cpp:629-639
 * with the problem plugin lpopt::Objective (Squared / Softmax losses, l2)
 *                                           proj/include/lpopt/objectives.hpp:14,59-91
 * and its hot-path members
 *     Objective::full_gradient              proj/src/objectives.cpp:258-311
 *     Objective::loss                       proj/src/objectives.cpp:193-223
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns
 * a halp_status; the message of the last failure on the calling thread is
 * available from halp_last_error().  The C++ header halp_lpopt.hpp wraps
 * this ABI in the reference's own types and exceptions.
 *
 * There is no CPU fallback: on a machine without a B200 (sm_100) every
 * compute entry point fails with HALP_CUDA_ERROR.
 */
#ifndef HALP_B200_H
#define HALP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HALP_ABI_VERSION 4

typedef enum {
  HALP_OK = 0,
  HALP_INVALID_INPUT = 1, /* lpopt::InvalidInputError (errors.hpp:13-15) */
  HALP_DIVERGED = 2,      /* lpopt::DivergenceError; the record holds the partial run (optimizers.hpp:71-75) */
  HALP_CUDA_ERROR = 3,
  HALP_NCCL_ERROR = 4,
  HALP_CAPACITY = 5,      /* caller-provided rows buffer too small */
  HALP_UNSUPPORTED = 6    /* shape outside what the kernels implement */
} halp_status;

typedef enum { HALP_F64 = 0, HALP_F32 = 1, HALP_BF16 = 2 } halp_dtype;
typedef enum { HALP_SQUARED = 0, HALP_SOFTMAX = 1 } halp_loss; /* LossFamily, objectives.hpp:14 */
typedef enum { HALP_MEM_HOST = 0, HALP_MEM_DEVICE = 1 } halp_mem;
typedef enum { HALP_STATUS_OK = 0, HALP_STATUS_CONVERGED = 1, HALP_STATUS_DIVERGED = 2 } halp_run_status;

/* Problem = lpopt::Objective + its Dataset (objectives.hpp:23-33,59-91).
 * X is row-major n x d (the reference stores fp64 column-major; any dtype
 * here is upcast exactly to fp64 inside the kernels).  mem says whether X,
 * y and labels are host or device (cuda:device) pointers; host data is
 * copied once at creation.  Device inputs (HALP_MEM_DEVICE) must be ready
 * when halp_problem_create is called: the library reads them on its own
 * non-blocking stream without waiting on the producer's stream (the Python
 * mirror synchronizes torch's current stream first).  Multi-GPU (world_size > 1): every rank passes
 * the same full problem and a shared 128-byte ncclUniqueId; the
 * full-gradient pass is row-sharded across ranks with one NCCL all-gather
 * per epoch, the sequential inner loop is replicated. */
typedef struct {
  const void*    X;
  int32_t        dtype;        /* halp_dtype */
  int32_t        mem;          /* halp_mem */
  int64_t        n;
  int32_t        d;
  int32_t        loss;         /* halp_loss */
  int32_t        num_classes;  /* softmax classes (>= 2); ignored for squared */
  const double*  y;            /* squared: n targets */
  const int32_t* labels;       /* softmax: n labels in [0, num_classes) */
  double         l2;
  int32_t        device;
  int32_t        world_size;   /* 1 => single GPU */
  int32_t        rank;
  const void*    nccl_id;      /* 128 bytes (ncclUniqueId) when world_size > 1 or collective == 1 */
  int32_t        collective;   /* 0: NCCL iff world_size > 1; 1: always run the NCCL route (all-gather
                                  of the rank sums + rank-tree finalize), also at world_size 1;
                                  2: no NCCL, the caller moves the rank sums (test hook:
                                  halp_rank_partial / halp_finalize_gathered only); ABI >= 4 */
  /* lpopt::QuantizedExamples (objectives.hpp): the dataset's LM-HALP codes,
   * int64 [n][d] in HOST memory (also when mem == HALP_MEM_DEVICE) at one
   * scale (halp_quantize_dataset), or NULL; ABI >= 4 */
  const int64_t* qcodes;
  int32_t        qbits;
  double         qdelta;
} halp_problem_desc;

typedef struct halp_problem halp_problem;

/* lpopt::OptimizerConfig (optimizers.hpp:31-47): the fields of the
 * algorithms this library runs (Halp; Svrg and LpSvrg on the same kernels) */
typedef struct {
  double        alpha;
  int32_t       epochs;
  int64_t       inner_steps;          /* 0 => full_grad_period * n */
  int32_t       bits;
  double        mu;
  int32_t       option;               /* 0 = EpochOption::LastIterate (I), 1 = SampledIterate (II) */
  int32_t       full_grad_period;
  uint64_t      seed;
  double        metric_every_passes;
  double        delta_min;
  double        divergence_limit;
  const double* init;                 /* host, d*num_outputs doubles, NULL => zeros */
  double        delta;                /* fixed scale of LpSvrg (OptimizerConfig::delta); ABI >= 3 */
  int32_t       algorithm;            /* HALP_ALGO_*: lpopt::Algorithm numbering; ABI >= 3 */
} halp_config;

/* lpopt::Algorithm values halp_run accepts (optimizers.hpp:13-15) */
enum { HALP_ALGO_SGD = 0, HALP_ALGO_SVRG = 1, HALP_ALGO_LP_SGD = 2, HALP_ALGO_LP_SVRG = 3, HALP_ALGO_HALP = 4,
       HALP_ALGO_LM_HALP = 5 /* needs qcodes; bits <= 16, d*C <= 4096, one GPU */ };

/* lpopt::MetricRow (optimizers.hpp:49-58), HALP subset */
typedef struct {
  double   pass;
  double   seconds;
  double   loss;
  double   grad_norm;
  double   delta;
  uint64_t iterate_hash;
  double   delta_inner;  /* LM-HALP inner-update scale (0 otherwise); ABI >= 4 */
  double   delta_aux;    /* LM-HALP auxiliary scalar scale */
} halp_row;

/* lpopt::RunRecord (optimizers.hpp:60-67).  Caller-owned buffers. */
typedef struct {
  halp_row* rows;
  int32_t   rows_cap;
  int32_t   rows_n;
  double*   final_iterate;            /* host, d*num_outputs doubles */
  int32_t   status;                   /* halp_run_status */
  int64_t   steps_taken;
  uint64_t  inner_fp_vector_ops;      /* 8*T per epoch, like the reference's instr counters */
  uint64_t  inner_lp_vector_ops;      /* 0 for HALP */
} halp_record;

/* Device timings of the last halp_run / halp_full_gradient (CUDA events on
 * the solver stream), milliseconds summed over the run. */
typedef struct {
  double  fullgrad_ms;     /* K1 full-gradient + loss pass (incl. split reduce) */
  double  finalize_ms;     /* collective + centering (norm, delta) */
  double  inner_ms;        /* K3 persistent inner loop */
  double  sample_ms;       /* K4 sample-index generation */
  int64_t fullgrad_launches;
  int64_t inner_launches;
  int64_t kernel_launches; /* every kernel this library launched */
  int64_t inner_steps;     /* inner steps executed */
  int64_t h2d_bytes;       /* host->device bytes moved by the call (inputs, iterate upload) */
  int64_t d2h_bytes;       /* device->host bytes (stats, iterates for the row hashes, result) */
} halp_timing;

/* Reduction plan of the problem's kernels (consumed by the oracle's MIRROR
 * mode in the tests to reproduce the device's floating-point order). */
typedef struct {
  int32_t fg_threads, fg_vec, fg_splits;
  int32_t in_ctas, in_threads, in_per;
  int32_t fg_rows_per_stage, fg_stages;
  int64_t fg_split_begin, fg_split_end; /* this rank's splits */
  int32_t in_levels;                    /* K3 cross-warp combine: 1 warp records (fp64), 2 CTA records then cluster, 3 fixed-point integer records (HALP_IN_LEVELS overrides the default 1) */
} halp_plan;

const char* halp_last_error(void);
int32_t     halp_abi_version(void);

int  halp_problem_create(const halp_problem_desc* desc, halp_problem** out);
void halp_problem_destroy(halp_problem* p);
int  halp_problem_plan(const halp_problem* p, halp_plan* out);

/* lpopt::run_halp.  On HALP_DIVERGED the record holds the partial run
 * with status HALP_STATUS_DIVERGED (what DivergenceError::partial carries). */
int halp_run(halp_problem* p, const halp_config* cfg, halp_record* rec);

/* lpopt::Objective::full_gradient + loss in one device pass (host w, g). */
int halp_full_gradient(halp_problem* p, const double* w, double* g, double* loss);

/* Test hook: dump the z codes of the first `steps` inner steps of each
 * halp_run into codes[epoch][step][D] (host, int64), up to cap entries. */
int halp_set_trace(halp_problem* p, int64_t* codes, int64_t cap);

int halp_last_timing(const halp_problem* p, halp_timing* out);

/* The two halves of the sharded full gradient with the exchange done by the
 * caller (problems created with collective == 2; test hook for the rank
 * plumbing on one GPU): this rank's subtree root [D+1] (K1 over its splits
 * + split tree) at host w, and the finalize over world_size gathered roots
 * [world][D+1] -> g (D), loss. */
int halp_rank_partial(halp_problem* p, const double* w, double* root);
int halp_finalize_gathered(halp_problem* p, const double* w, const double* gathered, double* g, double* loss);

/* Kernel-only timing helper for bench.py: runs `reps` full-gradient passes
 * at the device-resident iterate and returns the average device time per
 * pass (ms): K1 + split tree, plus the NCCL all-gather and the finalize
 * when the problem uses the collective (so multi-GPU GB/s include it). */
int halp_bench_full_gradient(halp_problem* p, int reps, double* ms_per_pass);

/* ---- batched independent problems (one persistent CTA per problem) ---- */
typedef struct {
  const void*   X;           /* [nprob][n][d] row-major, or [n][d] when shared */
  int32_t       dtype;
  int32_t       mem;
  int64_t       n;
  int32_t       d;
  int32_t       nprob;
  const double* y;           /* [nprob][n], or [n] when shared */
  double        l2;
  int32_t       device;
  int32_t       shared;      /* 1: every problem solves the SAME dataset (grid searches,
                                harness.cpp:379-447) with its own config; ABI >= 2 */
} halp_batch_desc;

typedef struct halp_batch halp_batch;
int  halp_batch_create(const halp_batch_desc* desc, halp_batch** out);
void halp_batch_destroy(halp_batch* b);
/* cfgs[nprob], recs[nprob]; every problem is an independent lpopt::run_halp
 * (squared loss, d <= 256).  A diverged problem gets status DIVERGED and its
 * partial record; the call itself returns HALP_OK.  device_ms = kernel time. */
int  halp_batch_run(halp_batch* b, const halp_config* cfgs, halp_record* recs, double* device_ms);
/* the batch kernel's reduction plan (for the oracle's MIRROR mode) */
int  halp_batch_plan(const halp_batch* b, halp_plan* out);

/* ---- synthetic data on the device (configs C2..C5 of BASELINE.json) ---- */
typedef struct {
  int32_t  kind;        /* 0 gaussian regression, 1 sparse-uniform softmax, 2 bf16 logistic (labels) */
  int64_t  n;
  int32_t  d;
  int32_t  num_classes;
  int32_t  dtype;
  double   noise_sd;
  double   x_scale;     /* std of x (kind 0/2) */
  double   density;     /* kind 1: fraction of nonzero entries */
  uint64_t seed;
} halp_datagen_desc;
/* X_dev [n][d] (dtype), y_dev [n] doubles (kind 0) or labels_dev [n] (kind 1/2) */
int halp_datagen(const halp_datagen_desc* desc, int32_t device, void* X_dev, double* y_dev, int32_t* labels_dev);

/* CPU-callable host logic (no GPU needed): the row/split shard plan of
 * rank `rank` of `world` for a problem of n rows and d*C = D coordinates. */
int halp_shard_plan(int64_t n, int32_t d, int32_t C, int32_t dtype, int32_t world, int32_t rank,
                    int64_t* split_begin, int64_t* split_end, int64_t* splits_total,
                    int64_t* row_begin, int64_t* row_end);

/* CPU-callable: the kernel plan the library would choose for a problem of
 * this shape (what halp_problem_plan reports after creation). */
int halp_plan_for(int64_t n, int32_t d, int32_t C, int32_t dtype, int32_t world, int32_t rank, halp_plan* out);

/* ---- the reference's own dataset generators (host, CPU-callable) ----
 * make_regression (objectives.cpp:27-45): X [n][d] row-major fp64, y [n] */
int halp_make_regression(int64_t n, int32_t d, double noise_sd, uint64_t seed, double* X, double* y);
/* make_classification (objectives.cpp:46-76): X [n][d], labels [n] */
int halp_make_classification(int64_t n, int32_t d, int32_t num_classes, double separation, uint64_t seed,
                             double* X, int32_t* labels);
/* quantize_dataset (objectives.cpp:110-133): codes [n][d] int64, *delta = data scale */
int halp_quantize_dataset(const double* X, int64_t n, int32_t d, int32_t bits, uint64_t seed, int64_t* codes,
                          double* delta);
/* `count` successive QuantRng(seed, stream).next_normal() draws (rng.hpp:57-62) */
int halp_normals(uint64_t seed, uint64_t stream, int64_t count, double* out);

/* xorshift64* stream state after `count` draws of (seed, stream) computed
 * by GF(2) jump-ahead (host), for tests of the counter-indexed RNG. */
uint64_t halp_rng_state_after(uint64_t seed, uint64_t stream, uint64_t count);

#ifdef __cplusplus
}
#endif
#endif /* HALP_B200_H */
