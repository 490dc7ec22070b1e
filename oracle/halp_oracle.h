/*
 * halp_oracle.h -- CPU restatement of the reference HALP hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 product path (paper_1803_03383_b200/csrc).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product never links, imports or calls it.
 *
 * It restates, from the reference C++ library `lpopt`
 * (/root/reference/proj, which cannot be built here: Eigen3 and vendor/
 * are absent):
 *   - QuantRng xorshift64* with splitmix seeding   include/lpopt/rng.hpp:12-64
 *   - quantize_code / quantize_vector / to_real     src/fixed_point.cpp:30-50,99-123
 *   - make_regression                               src/objectives.cpp:17-45
 *   - Objective loss / component_gradient_into /
 *     full_gradient (Squared, Softmax)              src/objectives.cpp:162-311
 *   - theory::halp_scale                            src/theory.cpp:33-35,93-102
 *   - run_halp + Recorder + validate_config +
 *     resolve_inner_steps + hash_vector             src/optimizers.cpp:36-167,209-227,387-459
 *
 * Two reduction-order modes:
 *   REF    -- sequential dots and block-ordered sums in the reference's
 *             structure (1024-row blocks, block partials summed in order).
 *             Pinned against the reference's golden traces
 *             proj/out/regression_floor/halp-{8,16}_seed{1..5}.csv and its
 *             RNG / quantizer known-answer tests (tests/golden/).
 *   MIRROR -- the exact floating-point operation order of the B200 kernels
 *             (described by oq_plan), so
 *             the GPU result can be checked bit for bit.
 * Element-wise arithmetic (the inner update, the quantizer, to_real) is the
 * reference's in both modes; it is never FMA-contracted (the reference is
 * built without -march, so without FMA: proj/CMakeLists.txt:27).
 */
#ifndef HALP_ORACLE_H
#define HALP_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror of include/halp.h) ---- */
enum { OQ_OK = 0, OQ_INVALID_INPUT = 1, OQ_DIVERGED = 2, OQ_CAPACITY = 5 };

/* ---- RNG: rng.hpp:27-64 ---- */
typedef struct { uint64_t state; } oq_rng;
void     oq_rng_init(oq_rng* r, uint64_t seed, uint64_t stream);
uint64_t oq_next_u64(oq_rng* r);
double   oq_next_uniform(oq_rng* r);
uint64_t oq_next_index(oq_rng* r, uint64_t n);
double   oq_next_normal(oq_rng* r);
/* fill out[0..count) with successive next_u64 outputs */
void     oq_fill_u64(uint64_t seed, uint64_t stream, uint64_t skip, uint64_t* out, int64_t count);

/* ---- quantizer: fixed_point.cpp:30-50 ---- */
/* returns the code; *err = 1 on non-finite x (reference throws InvalidInputError) */
int64_t oq_quantize_code(double x, double delta, int bits, double u, int* err);
/* theory.cpp:93-102 (returns -1 on invalid input) */
double  oq_halp_scale(double grad_norm, double mu, int bits);

/* ---- data ---- */
enum { OQ_F64 = 0, OQ_F32 = 1, OQ_BF16 = 2 };
enum { OQ_SQUARED = 0, OQ_SOFTMAX = 1 };
/* objectives.cpp:27-45; X row-major n x d fp64, y length n */
int oq_make_regression(int64_t n, int d, double noise_sd, uint64_t seed, double* X, double* y);

typedef struct {
  const void*    X;        /* row-major n x d, dtype below */
  int            dtype;    /* OQ_F64 / OQ_F32 / OQ_BF16 */
  int64_t        n;
  int            d;
  int            C;        /* 1 for squared, num_classes for softmax */
  int            loss;     /* OQ_SQUARED / OQ_SOFTMAX */
  const double*  y;        /* squared targets (n) */
  const int32_t* labels;   /* softmax labels (n) */
  double         l2;
} oq_objective;

/* Reduction plan of the B200 kernels (MIRROR mode).  NULL => REF mode.
 * Full-gradient pass (K1 fullgrad kernel):
 *   fg_threads   threads per row-dot (multiple of 32)
 *   fg_vec       features per vector load (group width)
 *   fg_splits    number of row splits (power of two); split s covers
 *                rows [s*n/S, (s+1)*n/S) (integer floor); splits are
 *                combined by a pairwise tree.
 * Inner loop (K3 cluster kernel):
 *   in_ctas      CTAs cooperating on one step (cluster size)
 *   in_threads   threads per CTA doing coordinate work (multiple of 32)
 *   in_per       coordinates per thread (contiguous flat index)
 *   in_levels    1: row dots combined across the cluster's warps directly;
 *                2: per CTA first (its warps in order), then across CTAs  */
typedef struct {
  int fg_threads, fg_vec, fg_splits;
  int in_ctas, in_threads, in_per;
  int in_levels;
} oq_plan;

int oq_loss(const oq_objective* o, const double* w, const oq_plan* plan, double* out);
int oq_full_gradient(const oq_objective* o, const double* w, int num_threads,
                     const oq_plan* plan, double* g);
/* fused pass used by MIRROR mode: gradient and loss from one sweep */
int oq_component_gradient(const oq_objective* o, int64_t i, const double* w,
                          const oq_plan* plan, double* out);

/* ---- run_halp: optimizers.cpp:387-459 ---- */
typedef struct {
  double   alpha;
  int32_t  epochs;
  int64_t  inner_steps;          /* 0 => full_grad_period * n */
  int32_t  bits;
  double   mu;
  int32_t  option;               /* 0 = LastIterate (I), 1 = SampledIterate (II) */
  int32_t  full_grad_period;
  uint64_t seed;
  double   metric_every_passes;
  double   delta_min;
  double   divergence_limit;
  const double* init;            /* NULL => zeros */
  double   delta;                /* fixed scale of LP-SVRG (OptimizerConfig::delta) */
  int32_t  algorithm;            /* lpopt::Algorithm: 0 Sgd, 1 Svrg, 2 LpSgd, 3 LpSvrg, 4 Halp */
} oq_config;

enum { OQ_ALGO_SGD = 0, OQ_ALGO_SVRG = 1, OQ_ALGO_LP_SGD = 2, OQ_ALGO_LP_SVRG = 3, OQ_ALGO_HALP = 4, OQ_ALGO_LM_HALP = 5 };

typedef struct {
  double   pass, seconds, loss, grad_norm, delta;
  uint64_t iterate_hash;
  double   delta_inner, delta_aux;   /* LM-HALP scales (optimizers.hpp:56-57), 0 otherwise */
} oq_row;

enum { OQ_STATUS_OK = 0, OQ_STATUS_CONVERGED = 1, OQ_STATUS_DIVERGED = 2 };

typedef struct {
  oq_row*  rows;        /* caller-allocated */
  int32_t  rows_cap;
  int32_t  rows_n;
  double*  final_iterate; /* caller-allocated, length d*C */
  int32_t  status;
  int64_t  steps_taken;
  uint64_t inner_fp_vector_ops;
  /* optional trace hook: if non-NULL, codes of every inner step are
   * written as int64 [epoch][t][D] up to trace_cap entries */
  int64_t* trace_codes;
  int64_t  trace_cap;
  /* optional: full-gradient timing (seconds, summed) for reporting */
  double   fullgrad_seconds;
  double   inner_seconds;
  int      fullgrad_threads;   /* threads for full_gradient (reference default 1) */
  /* optional: one 64-bit hash of the codes after every inner step,
   * [epoch][t] up to step_hash_cap entries (oq_code_hash).  Comparing the
   * REF-order and MIRROR-order runs' hashes counts the steps whose rounding
   * decisions depend on the reduction order. */
  uint64_t* step_hash;
  int64_t   step_hash_cap;
  uint64_t  inner_lp_vector_ops;  /* LM-HALP's integer vector ops (instr counters) */
} oq_record;

int      oq_run_halp(const oq_objective* o, const oq_config* cfg, const oq_plan* plan, oq_record* rec);
/* run_svrg / run_lp_svrg (optimizers.cpp:258-296, 336-385) and the run()
 * dispatch (optimizers.cpp:629-639) over the algorithms the B200 builds */
int      oq_run(const oq_objective* o, const oq_config* cfg, const oq_plan* plan, oq_record* rec);
int64_t  oq_resolve_inner_steps(const oq_config* cfg, int64_t n);
uint64_t oq_hash_vector(const double* v, int64_t len);
/* FNV-1a over the int64 code bytes of one inner step (test hook) */
uint64_t oq_code_hash(const int64_t* codes, int64_t len);
const char* oq_last_error(void);

/* ---- LM-HALP: quantize_dataset (objectives.cpp:110-133, data_scale :112-122)
 * and run_lm_halp (optimizers.cpp:461-627), non-bypass path ----
 * codes [n][d] int64 out, *delta = the data scale (LPRepr delta) */
int oq_quantize_dataset(const double* X, int64_t n, int d, int bits, uint64_t seed, int64_t* codes, double* delta);
typedef struct {
  const int64_t* codes;  /* [n][d] */
  double         delta;
  int            bits;
} oq_quantized;
/* MIRROR plan: only fg_splits is used (the device's split count); the LM
 * stats pass uses 128-thread row dots.  Trace: z codes [epoch][t][D]. */
int oq_run_lm_halp(const oq_objective* o, const oq_quantized* q, const oq_config* cfg, const oq_plan* plan,
                   oq_record* rec);

/* MIRROR-mode pieces of the multi-GPU full gradient: one rank's split
 * subtree root [D+1] and the finalize over G gathered rank sums */
int oq_split_subtree(const oq_objective* o, const double* w, const oq_plan* plan, int64_t s0, int64_t s1,
                     double* out);
int oq_finalize(const oq_objective* o, const double* w, const double* rank_sums, int G, double* g, double* loss);

/* ---- K6 synthetic data, host restatement (oracle/datagen.c) ---- */
typedef struct {
  int32_t  kind;        /* 0 gaussian regression, 1 sparse-uniform softmax, 2 logistic labels */
  int64_t  n;
  int32_t  d;
  int32_t  num_classes;
  int32_t  dtype;       /* OQ_F64 / OQ_F32 / OQ_BF16 (raw uint16 bits) */
  double   noise_sd;
  double   x_scale;
  double   density;
  uint64_t seed;
} oq_datagen_desc;
/* rows [row0, row0 + nrows) of the dataset K6 generates for `g` (same bytes),
 * written to X [nrows][d] and y / labels [nrows]; nthreads host threads */
int oq_datagen(const oq_datagen_desc* g, int64_t row0, int64_t nrows, int nthreads, void* X, double* y,
               int32_t* labels);

/* exponent S of K3's fixed-point exchange (plan in_levels 3) for an epoch */
int oq_fx_exponent(double xmax, const double* w, int64_t D, double delta, int bits);

/* mirror-mode exp/log (identical operation sequence to the device code) */
double oq_mexp(double x);
/* REF-mode Eigen packet width (1, 2 or 4); default pinned by golden traces */
void oq_set_ref_lanes(int lanes);
double oq_mlog(double x);
/* Markstein reciprocal-division check (mismatches vs IEEE x/delta in n cases) */
int64_t oq_div_check(int64_t n, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
