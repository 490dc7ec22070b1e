// halp_capi.cpp -- host driver of the B200 HALP solver behind the C ABI
// (include/halp.h).  It owns the device problem, chooses the kernel plan,
// runs the epoch loop of lpopt::run_halp (proj/src/optimizers.cpp:387-459)
// with the reference's Recorder semantics (:104-167), and talks NCCL for the
// row-sharded full gradient.  Everything numeric happens in the CUDA
// kernels (k_fullgrad.cu, k_inner.cu, k_batch.cu, k_datagen.cu); the host
// only orders launches, computes RNG jump states and formats MetricRows.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/halp.h"
#include "kernels.h"
#include "rng_jump.hpp"

using namespace halp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(expr)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return fail(HALP_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
  } while (0)

int64_t env_int(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoll(v) : dflt;
}

int elem_size(int dtype) { return dtype == HALP_F64 ? 8 : dtype == HALP_F32 ? 4 : 2; }

int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}
int64_t prev_pow2(int64_t v) {
  int64_t p = 1;
  while (p * 2 <= v) p <<= 1;
  return p;
}

// ---- NCCL through dlopen (the soname torch already loaded, if any) ----
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    return commInitRank && allGather && commDestroy && errStr;
  }
  static Nccl& get() {
    static Nccl n;
    return n;
  }
};

struct ShardPlan {
  int64_t S = 1, split_begin = 0, split_end = 1, row_begin = 0, row_end = 0;
  int64_t local_splits() const { return split_end - split_begin; }
};

// Split grid of the full-gradient pass: S splits (the leaves of the pairwise
// reduction tree, one (D+1) partial each), a power of two <= 4096 within an
// eighth of X's bytes; ranks own aligned, equal blocks of splits.
ShardPlan make_shard_plan(int64_t n, int d, int C, int dtype, int world, int rank) {
  ShardPlan sp;
  const int64_t D1 = (int64_t)d * C + 1;
  const double xbytes = (double)n * d * elem_size(dtype);
  const double budget = std::max(xbytes / 8.0, 2.0 * (1 << 20));
  int64_t S = 1;
  const int64_t smax = std::max<int64_t>(1, env_int("HALP_FG_MAX_SPLITS", 4096));  // experiment knob
  while (S * 2 <= smax && S * 2 <= std::max<int64_t>(1, n / 2) && (double)(S * 2) * D1 * 8.0 <= budget) S *= 2;
  if (S < world) S = next_pow2(world);
  sp.S = S;
  sp.split_begin = S / world * rank;
  sp.split_end = S / world * (rank + 1);
  sp.row_begin = (int64_t)((unsigned __int128)n * sp.split_begin / sp.S);
  sp.row_end = (int64_t)((unsigned __int128)n * sp.split_end / sp.S);
  return sp;
}

struct Events {
  cudaEvent_t a = nullptr, b = nullptr;
  ~Events() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

uint64_t fnv1a(const double* v, int64_t len) {  // optimizers.cpp:218-227
  uint64_t h = 1469598103934665603ULL;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(v);
  const size_t nb = sizeof(double) * (size_t)len;
  for (size_t i = 0; i < nb; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

// Blocking copy ordered on `st`.  Every device buffer of a problem / batch is
// produced and consumed on its own non-blocking stream, so copies must be
// issued there too: a legacy-stream cudaMemcpy is not ordered against it
// (and a pageable H2D cudaMemcpy may return before its DMA has landed).
cudaError_t copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

// ---- device memory: the device's stream-ordered pool, never trimmed ----
// Problems are created and destroyed per solve (run_prepared, sweeps, the e2e
// path); keeping freed blocks in the pool makes that O(1) instead of a
// cudaMalloc/cudaFree (and page-table work) per solve.
std::mutex& host_state_mutex() {  // guards the per-device host-side caches below
  static std::mutex m;
  return m;
}

int pool_setup(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64) return HALP_INVALID_INPUT;
  std::lock_guard<std::mutex> lock(host_state_mutex());
  if (done[device]) return HALP_OK;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return HALP_CUDA_ERROR;
  uint64_t keep = UINT64_MAX;
  if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess) return HALP_CUDA_ERROR;
  done[device] = true;
  return HALP_OK;
}
template <class T>
cudaError_t dalloc(T** ptr, size_t bytes, cudaStream_t st) {
  return cudaMallocAsync(reinterpret_cast<void**>(ptr), std::max<size_t>(bytes, 16), st);
}

// RNG jump tables, uploaded once per device and kept resident: the 64
// power tables X^(2^b) (1 MiB) and, per epoch length D, the X^D table (16 KiB)
struct RngTables {
  const uint64_t* pow_tab = nullptr;
  std::vector<std::pair<int64_t, const uint64_t*>> jump;  // (D, table)
};
int rng_tables(int device, int64_t D, const uint64_t** pow_tab, const uint64_t** jump_tab, cudaStream_t st) {
  static RngTables per_dev[64];
  if (device < 0 || device >= 64) return fail(HALP_INVALID_INPUT, "device index out of range");
  std::lock_guard<std::mutex> lock(host_state_mutex());
  RngTables& t = per_dev[device];
  const auto& jt = JumpTables::get();
  if (!t.pow_tab) {
    uint64_t* d = nullptr;
    CU(cudaMalloc(&d, sizeof(uint64_t) * jt.flat.size()));
    CU(copy_sync(d, jt.flat.data(), sizeof(uint64_t) * jt.flat.size(), cudaMemcpyHostToDevice, st));
    t.pow_tab = d;
  }
  *pow_tab = t.pow_tab;
  for (const auto& e : t.jump)
    if (e.first == D) {
      *jump_tab = e.second;
      return HALP_OK;
    }
  std::vector<uint64_t> tab(2048);
  mat_tables(jt.power((uint64_t)D), tab.data());
  uint64_t* d = nullptr;
  CU(cudaMalloc(&d, sizeof(uint64_t) * 2048));
  CU(copy_sync(d, tab.data(), sizeof(uint64_t) * 2048, cudaMemcpyHostToDevice, st));
  t.jump.emplace_back(D, d);
  *jump_tab = d;
  return HALP_OK;
}

}  // namespace

struct halp_problem {
  int device = 0, dtype = 0, loss = 0;
  int64_t n = 0;
  int d = 0, C = 1, D = 1, ld = 0;
  double l2 = 0.0;
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  // device data
  void* X = nullptr;
  bool own_X = false;
  double* y = nullptr;
  int32_t* labels = nullptr;
  // plans
  ShardPlan sp;
  FgLaunch fg{};
  InLaunch in{};
  int fg_passes = 1;
  // workspace
  double *zb0 = nullptr, *zb1 = nullptr;  // K3 z0 / zc_out ping-pong (SVRG, LP-SVRG)
  double *w = nullptr, *w2 = nullptr, *g = nullptr, *partials = nullptr, *rank_sum = nullptr, *gathered = nullptr,
         *stats = nullptr, *u_out = nullptr, *tree_scratch = nullptr;
  int64_t* idx = nullptr;
  int64_t idx_cap = 0;
  long long* codes = nullptr;
  long long* blow = nullptr;
  const uint64_t *pow_tab = nullptr, *jump_tab = nullptr;  // resident per device (rng_tables)
  long long* trace_dev = nullptr;
  int64_t trace_dev_steps = 0;
  int64_t* trace_host = nullptr;
  int64_t trace_cap = 0;
  halp_timing timing{};
  int64_t create_h2d = 0;  // bytes uploaded by halp_problem_create
  int x_finite = 0;        // bf16 X checked finite (K1 integer-conversion path)
  bool host_exchange = false;  // collective == 2: the caller moves the rank sums (test hook)
  // LM-HALP: the quantized dataset (int8 / int16 codes), logits at w~ per row, h codes, error flag
  void* q = nullptr;
  int qbits = 0, qbytes = 0;
  double qdelta = 0.0;
  double* phi = nullptr;
  long long* hdev = nullptr;
  int* lm_bad = nullptr;
  // pinned bounce buffer for the small per-epoch copies (stats, iterates): a
  // pageable copy would queue behind another problem's multi-GB upload on the
  // copy engine and stall this solve (e2e streaming of consecutive problems)
  double* pin = nullptr;
  size_t pin_bytes = 0;
  double xmax = -1.0;  // max |x| (fixed-point exchange bound), computed on first use
  Events ev_fg, ev_fin, ev_in, ev_smp;

  ~halp_problem() {
    cudaSetDevice(device);
    // stream-ordered frees back into the device pool (no device-wide sync)
    for (void* ptr : {(void*)w, (void*)w2, (void*)g, (void*)partials, (void*)rank_sum, (void*)gathered, (void*)stats,
                      (void*)u_out, (void*)idx, (void*)codes, (void*)blow, (void*)trace_dev, (void*)y,
                      (void*)labels, (void*)tree_scratch, (void*)zb0, (void*)zb1, q, (void*)phi, (void*)hdev,
                      (void*)lm_bad})
      if (ptr) cudaFreeAsync(ptr, stream);
    if (own_X && X) cudaFreeAsync(X, stream);
    if (pin) cudaFreeHost(pin);
    if (comm) Nccl::get().commDestroy(comm);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// small copies through the problem's pinned buffer (see halp_problem::pin)
cudaError_t p_d2h(halp_problem* p, void* dst, const void* src, size_t bytes) {
  if (!p->pin || bytes > p->pin_bytes) return copy_sync(dst, src, bytes, cudaMemcpyDeviceToHost, p->stream);
  cudaError_t e = copy_sync(p->pin, src, bytes, cudaMemcpyDeviceToHost, p->stream);
  if (e == cudaSuccess) std::memcpy(dst, p->pin, bytes);
  return e;
}
cudaError_t p_h2d(halp_problem* p, void* dst, const void* src, size_t bytes) {
  if (!p->pin || bytes > p->pin_bytes) return copy_sync(dst, src, bytes, cudaMemcpyHostToDevice, p->stream);
  std::memcpy(p->pin, src, bytes);
  return copy_sync(dst, p->pin, bytes, cudaMemcpyHostToDevice, p->stream);
}

constexpr int kDefaultInLevels = 1;  // measured on B200: see DESIGN.md 8

struct KernelPlan {
  FgLaunch fg{};
  InLaunch in{};
  int fg_passes = 1;
};

// K1 streaming-kernel plan for C <= 2 (k_fullgrad_stream.cu): thread count
// covering the 16-byte feature groups, rows per tile by the register budget,
// only shapes instantiated in HALP_STREAM_SHAPES.  Returns false if none fits.
bool stream_shape_ok(int nw, int ng, int r, int st) {
#define HALP_STREAM_OK(NW, NG, R, ST) \
  if (nw == NW && ng == NG && r == R && st == ST) return true;
  HALP_STREAM_SHAPES(HALP_STREAM_OK)
#undef HALP_STREAM_OK
  return false;
}

bool plan_stream(int d, int C, int dtype, FgLaunch* out) {
  const int es = elem_size(dtype);
  const int V = 16 / es;
  const int ld = (int)(((int64_t)d * es + 15) / 16 * 16 / es);
  const int ngroups = (d + V - 1) / V;
  int NG = (int)env_int("HALP_FG_NG", 0);
  if (NG <= 0) {
    NG = 1;  // measured on B200 (tools/fg_sweep.py): 256-thread CTAs beat 512 at C3
    while (ngroups > 256 * NG) NG *= 2;
  }
  if (NG > 4) return false;
  int T1 = 32;
  while (T1 < 512 && T1 * NG < ngroups) T1 *= 2;
  if (T1 * NG < ngroups) return false;
  const int row_bytes = ld * es;
  int stages = (int)env_int("HALP_FG_STAGES", 4);
  int R = (int)env_int("HALP_FG_ROWS", 0);
  if (R <= 0) {
    R = 8;
    const int reg_cap = std::min(255, 65536 / T1);
    // one effective column for both losses (two classes: the logistic form)
    auto regs = [&](int r) { return 2 * (r * NG * V + 2 * NG * V + r) + 48; };
    // tiles up to 32 KB in a 4-deep ring; 64 KB tiles in a 3-deep ring where that shape is
    // instantiated (C3's 16 KB rows: 4-row tiles halve the per-tile barrier / reduce cost,
    // measured on B200 12.35 -> 10.55 ms per pass, tools/fg_sweep.py, profiles/r02_s5_k1_c3_rows4.txt)
    const bool free_stages = env_int("HALP_FG_STAGES", 0) == 0;
    auto tile_ok = [&](int r) {
      if ((int64_t)r * row_bytes <= 32 * 1024 && stream_shape_ok(T1 / 32, NG, r, stages)) return true;
      return free_stages && (int64_t)r * row_bytes <= 64 * 1024 && stream_shape_ok(T1 / 32, NG, r, 3);
    };
    while (R > 1 && (R * NG * V > 64 || regs(R) > reg_cap || !tile_ok(R))) R /= 2;
    if (free_stages && (int64_t)R * row_bytes > 32 * 1024) stages = 3;
    // bf16 two-class rows (C4): 16-row tiles with x re-read from shared memory
    // for the gradient phase, double-buffered (measured on B200, tools/fg_sweep.py:
    // 51% vs 48% of HBM for 8-row register tiles; the gradient is bit-identical)
    if (C == 2 && es == 2 && NG == 1 && env_int("HALP_FG_STAGES", 0) == 0 && stream_shape_ok(T1 / 32, NG, 16, 2) &&
        (int64_t)16 * row_bytes <= 48 * 1024) {
      R = 16;
      stages = 2;
    }
  }
  if (!stream_shape_ok(T1 / 32, NG, R, stages)) return false;
  if (stream_smem_bytes(ld, es, T1 / 32, R, C, stages) > 220 * 1024) return false;
  *out = FgLaunch{dtype, NG, C, T1, ld, 0, 4, R, stages};
  return true;
}

ShardPlan shard_plan_for(int64_t n, int d, int C, int dtype, int world, int rank) {
  return make_shard_plan(n, d, C, dtype, world, rank);
}

// kernel plan as a pure function of the problem shape (CPU-callable)
int plan_for(int64_t n, int d, int C, int dtype, KernelPlan* kp) {
  (void)n;
  const int es = elem_size(dtype);
  const int V = 16 / es;
  const int ld = (int)(((int64_t)d * es + 15) / 16 * 16 / es);
  const int ngroups = (d + V - 1) / V;
  int T1 = (int)std::min<int64_t>(256, (ngroups + 31) / 32 * 32);
  int NG = (int)next_pow2((ngroups + T1 - 1) / T1);
  if (NG > 8) return fail(HALP_UNSUPPORTED, "full_gradient: d too large for the register-resident column tiles");
  int CT = 8;
  while (CT > 1 && (NG * V * CT > 64 || CT >= 2 * C)) CT /= 2;
  if (CT > C) CT = (int)next_pow2(C);
  kp->fg = FgLaunch{dtype, NG, CT, T1, ld, 0, 0, 2, 4};
  kp->fg_passes = (C + CT - 1) / CT;
  // persistent streaming kernel (C <= 2; HALP_FG_GENERIC=1 forces the generic kernel for least squares)
  if (C <= 2 && env_int("HALP_FG_GENERIC", 0) == 0) {
    FgLaunch fl;
    if (plan_stream(d, C, dtype, &fl)) {
      kp->fg = fl;
      kp->fg_passes = 1;
    } else if (C == 2) {
      // the two-class logistic form (MIRROR order) exists only in the streaming kernel
      return fail(HALP_UNSUPPORTED, "full_gradient: two-class rows wider than the streaming kernel's register tiles");
    }
  } else if (C == 2) {
    return fail(HALP_UNSUPPORTED, "full_gradient: two-class objectives need the streaming kernel");
  } else {
    const size_t smem = fg_smem_bytes(ld, es, d * C, C, T1, 2, 4);
    // softmax with 3..15 classes: one-pass kernel with a 32-slot reduce-scatter
    const int64_t S_ = make_shard_plan(n, d, C, dtype, 1, 0).S;
    const int Ts = (int)((ngroups + 31) / 32 * 32);
    if (C >= 3 && ngroups <= 256 && V * C <= 64 && !(es == 2 && C < 8) && env_int("HALP_FG_GENERIC", 0) == 0 &&
        smx_smem_bytes(ld, es, d, C, Ts, (n + S_ - 1) / S_ + 1) <= 220 * 1024) {
      kp->fg = FgLaunch{dtype, 1, C, Ts, ld, 0, 3, 32 / C, 4};
      kp->fg_passes = 1;
    } else if (smem > 220 * 1024) {
      return fail(HALP_UNSUPPORTED, "full_gradient: row tile + iterate exceed shared memory");
    }
  }
  // inner loop: M coordinates per thread, up to 16 CTAs per cluster
  const int64_t D = (int64_t)d * C;
  // Measured on B200 (tools/sweep_inner.py): one CTA (__syncthreads exchange)
  // wins while <= 128 threads cover D; beyond, 128-thread CTAs up to a 16-CTA
  // cluster with the fewest coordinates per thread; 256-thread CTAs last.
  int M = (int)env_int("HALP_IN_M", 0);
  int NC = (int)env_int("HALP_IN_NC", 0);
  int64_t threads = 0;
  if (M <= 0) {
    if (D <= 512) {
      M = 1;
      while (M < 4 && (D + M - 1) / M > 128) M *= 2;
      if (NC <= 0) NC = 1;
    } else {
      M = 2;
      while (M < 8 && (D + M - 1) / M > 16 * 128) M *= 2;
    }
  }
  while (M > 1 && M > d) M /= 2;
  threads = (D + M - 1) / M;
  if (NC <= 0) NC = (int)((threads + 127) / 128);
  if (NC > 16) NC = (int)((threads + 255) / 256);
  while (NC > 16 && M < 8) {
    M *= 2;
    threads = (D + M - 1) / M;
    NC = (int)((threads + 255) / 256);
  }
  if (NC > 16) return fail(HALP_UNSUPPORTED, "inner loop: d*C too large for one 16-CTA cluster");
  int T3 = (int)(((threads + NC - 1) / NC + 31) / 32 * 32);
  if (T3 > 256) return fail(HALP_UNSUPPORTED, "inner loop: bad cluster plan");
  const int nslots = 2 * C + 1;
  kp->in = InLaunch{dtype, NC, T3, M, (int)std::max<int64_t>(4, next_pow2(nslots))};
  // squared loss on a cluster: the CTA's warps pre-reduced in shared memory, one
  // record per CTA in the DSMEM exchange (k_inner.cu LV2; HALP_IN_LEVELS overrides)
  {
    const int lv = (int)env_int("HALP_IN_LEVELS", 0);
    const bool can = C == 1 && NC > 1 && T3 >= 64;
    const bool can_fx = C == 1;
    kp->in.levels = lv == 3 && can_fx ? 3 : can && lv == 2 ? 2 : lv == 1 ? 1 : (can_fx && kDefaultInLevels == 3) ? 3 : 1;
    kp->in.pf2 = (int)env_int("HALP_K3_PF2", -1);
  }
  return HALP_OK;
}

int choose_plans(halp_problem* p) {
  KernelPlan kp;
  int rc = plan_for(p->n, p->d, p->C, p->dtype, &kp);
  if (rc) return rc;
  p->fg = kp.fg;
  p->in = kp.in;
  p->fg_passes = kp.fg_passes;
  return HALP_OK;
}

int ensure_workspace(halp_problem* p) {
  const int64_t D1 = p->D + 1;
  const int64_t nloc = p->sp.local_splits();
  if (!p->w) {
    cudaStream_t st = p->stream;
    CU(dalloc(&p->w, sizeof(double) * p->D, st));
    CU(dalloc(&p->w2, sizeof(double) * p->D, st));
    CU(dalloc(&p->g, sizeof(double) * p->D, st));
    CU(dalloc(&p->u_out, sizeof(double) * p->D, st));
    CU(dalloc(&p->partials, sizeof(double) * D1 * nloc, st));
    CU(dalloc(&p->tree_scratch, sizeof(double) * D1 * std::max<int64_t>(1, nloc / 64), st));
    CU(dalloc(&p->rank_sum, sizeof(double) * D1, st));
    CU(dalloc(&p->gathered, sizeof(double) * D1 * p->world, st));
    CU(dalloc(&p->stats, sizeof(double) * 4, st));
    CU(dalloc(&p->codes, sizeof(long long) * p->D, st));
    CU(dalloc(&p->blow, sizeof(long long), st));
    CU(dalloc(&p->zb0, sizeof(double) * p->D, st));
    CU(dalloc(&p->zb1, sizeof(double) * p->D, st));
    p->pin_bytes = sizeof(double) * (size_t)std::max<int64_t>(p->D + 8, 64);
    CU(cudaMallocHost(reinterpret_cast<void**>(&p->pin), p->pin_bytes));
    int rc = rng_tables(p->device, p->D, &p->pow_tab, &p->jump_tab, p->stream);
    if (rc) return rc;
    CU(cudaEventCreate(&p->ev_fg.a));
    CU(cudaEventCreate(&p->ev_fg.b));
    CU(cudaEventCreate(&p->ev_fin.a));
    CU(cudaEventCreate(&p->ev_fin.b));
    CU(cudaEventCreate(&p->ev_in.a));
    CU(cudaEventCreate(&p->ev_in.b));
    CU(cudaEventCreate(&p->ev_smp.a));
    CU(cudaEventCreate(&p->ev_smp.b));
  }
  return HALP_OK;
}

FgParams fg_params(const halp_problem* p, int pass) {
  return FgParams{p->X, p->n, p->d, p->ld, p->C, p->loss, p->y, p->labels, p->w,
                  (int)p->sp.S, (int)p->sp.split_begin, pass * p->fg.ct, pass == 0, p->partials, p->x_finite};
}

// the exchange step of the row-sharded full gradient: every rank's subtree
// root (D+1 doubles) all-gathered over NCCL, then the same rank tree on
// every rank (k_finalize) -> identical g, |g|, delta, loss on all ranks
int gather_finalize(halp_problem* p, double mu, int bits, double delta_min) {
  const int64_t D1 = p->D + 1;
  if (p->comm) {
    ncclResult_t r = Nccl::get().allGather(p->rank_sum, p->gathered, (size_t)D1, ncclFloat64, p->comm, p->stream);
    if (r != ncclSuccess) return fail(HALP_NCCL_ERROR, std::string("ncclAllGather: ") + Nccl::get().errStr(r));
  }
  FinParams fin{p->gathered, p->world, p->D, p->w, p->n, p->l2, mu, delta_min, bits, p->g, p->stats};
  CU(launch_finalize(fin, p->stream));
  ++p->timing.kernel_launches;
  return HALP_OK;
}

// K1 + split tree (+ all-gather) + finalize at p->w; stats -> host
int full_pass(halp_problem* p, double* gn, double* delta, double* loss, double mu, int bits, double delta_min) {
  const int64_t D1 = p->D + 1;
  const int nloc = (int)p->sp.local_splits();
  CU(cudaEventRecord(p->ev_fg.a, p->stream));
  for (int pass = 0; pass < p->fg_passes; ++pass) {
    FgParams fp = fg_params(p, pass);
    FgLaunch L = p->fg;
    L.nsplit_local = nloc;
    CU(launch_fullgrad(L, fp, p->stream));
    ++p->timing.kernel_launches;
  }
  CU(launch_split_tree(p->partials, nloc, (int)D1, p->comm ? p->rank_sum : p->gathered, p->tree_scratch,
                        p->stream));
  ++p->timing.kernel_launches;
  CU(cudaEventRecord(p->ev_fg.b, p->stream));
  CU(cudaEventRecord(p->ev_fin.a, p->stream));
  int rc = gather_finalize(p, mu, bits, delta_min);
  if (rc) return rc;
  CU(cudaEventRecord(p->ev_fin.b, p->stream));
  double st[4];
  CU(p_d2h(p, st, p->stats, sizeof(double) * 3));
  p->timing.d2h_bytes += sizeof(double) * 3;
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, p->ev_fg.a, p->ev_fg.b));
  p->timing.fullgrad_ms += ms;
  p->timing.fullgrad_launches += p->fg_passes;
  CU(cudaEventElapsedTime(&ms, p->ev_fin.a, p->ev_fin.b));
  p->timing.finalize_ms += ms;
  *gn = st[0];
  *delta = st[1];
  *loss = st[2];
  return HALP_OK;
}

// Recorder (optimizers.cpp:104-167)
struct Recorder {
  const halp_config* cfg;
  halp_record* rec;
  double t0, next_pass = 0.0;
  int D;
  int boundary(double pass, const double* w, double loss, double gn, double delta, bool forced, double delta_inner = 0.0,
               double delta_aux = 0.0) {
    const bool bad =
        !(std::isfinite(loss) && std::isfinite(gn)) || loss > cfg->divergence_limit || gn > cfg->divergence_limit;
    const bool due = forced || cfg->metric_every_passes <= 0.0 || pass + 1e-9 >= next_pass;
    if (due || bad) {
      if (rec->rows_n >= rec->rows_cap) return fail(HALP_CAPACITY, "halp_run: rows capacity exceeded");
      halp_row& r = rec->rows[rec->rows_n++];
      r.pass = pass;
      r.seconds = now_s() - t0;
      r.loss = loss;
      r.grad_norm = gn;
      r.delta = delta;
      r.iterate_hash = fnv1a(w, D);
      r.delta_inner = delta_inner;
      r.delta_aux = delta_aux;
      if (cfg->metric_every_passes > 0.0) next_pass = pass + cfg->metric_every_passes;
    }
    if (bad) {
      rec->status = HALP_STATUS_DIVERGED;
      if (rec->final_iterate) std::memcpy(rec->final_iterate, w, sizeof(double) * D);
      rec->steps_taken = 0;  // DivergenceError's partial record (optimizers.cpp:457 never ran)
      char m[128];
      std::snprintf(m, sizeof m, "run diverged near pass %f", pass);
      return fail(HALP_DIVERGED, m);
    }
    return HALP_OK;
  }
};

// optimizers.cpp:36-97 (HALP checks)
// fixed_point.cpp:30-50 quantize_code (host: LP-SVRG's one-time quantization
// of the initial iterate; the device quantizer is quantize_fast in K3)
int64_t host_quantize_code(double x, double delta, int bits, double u) {
  const int64_t maxc = bits == 64 ? INT64_MAX : (int64_t)((1ULL << (bits - 1)) - 1);
  const int64_t minc = bits == 64 ? INT64_MIN : -(int64_t)(1ULL << (bits - 1));
  const double t = x / delta;
  if (t >= (double)maxc) return maxc;
  if (t <= (double)minc) return minc;
  const double snapped = std::nearbyint(t);
  if (snapped * delta == x) return (int64_t)snapped;
  const double fl = std::floor(t);
  const double frac = t - fl;
  int64_t code = (int64_t)fl;
  if (frac > 0.0 && u < frac) ++code;
  return code;
}

int validate(const halp_problem* p, const halp_config* c) {
  if (!(std::isfinite(c->alpha) && c->alpha >= 0.0)) return fail(HALP_INVALID_INPUT, "optimizer: alpha must be finite and >= 0");
  if (c->epochs < 0) return fail(HALP_INVALID_INPUT, "optimizer: epochs must be >= 0");
  if (c->inner_steps < 0) return fail(HALP_INVALID_INPUT, "optimizer: inner_steps must be >= 0");
  if (c->full_grad_period < 1) return fail(HALP_INVALID_INPUT, "optimizer: full_grad_period must be >= 1");
  if (!(std::isfinite(c->metric_every_passes) && c->metric_every_passes >= 0.0))
    return fail(HALP_INVALID_INPUT, "optimizer: metric_every_passes must be finite and >= 0");
  if (!(std::isfinite(c->divergence_limit) && c->divergence_limit > 0.0))
    return fail(HALP_INVALID_INPUT, "optimizer: divergence_limit must be positive");
  if (!(std::isfinite(c->delta_min) && c->delta_min > 0.0)) return fail(HALP_INVALID_INPUT, "optimizer: delta_min must be positive");
  if (c->algorithm < HALP_ALGO_SGD || c->algorithm > HALP_ALGO_LM_HALP)
    return fail(HALP_INVALID_INPUT, "unknown algorithm enum value");
  if (c->algorithm == HALP_ALGO_LP_SVRG || c->algorithm == HALP_ALGO_LP_SGD) {  // uses_fixed_scale
    if (c->bits < 2 || c->bits > 64) return fail(HALP_INVALID_INPUT, "optimizer: bits must be in [2, 64]");
    if (!(std::isfinite(c->delta) && c->delta > 0.0))
      return fail(HALP_INVALID_INPUT, "optimizer: delta must be positive for fixed-scale runs");
  }
  if (c->algorithm == HALP_ALGO_HALP || c->algorithm == HALP_ALGO_LM_HALP) {  // uses_bit_centering
    if (c->bits < 2 || c->bits > 64) return fail(HALP_INVALID_INPUT, "optimizer: bits must be in [2, 64]");
    if (!(std::isfinite(c->mu) && c->mu > 0.0))
      return fail(HALP_INVALID_INPUT, "optimizer: mu must be positive for bit-centered runs");
  }
  if (c->option != 0 && c->option != 1) return fail(HALP_INVALID_INPUT, "optimizer: option must be 0 (I) or 1 (II)");
  if (c->algorithm == HALP_ALGO_LM_HALP && p) {  // optimizers.cpp:77-96
    if (c->bits > 32) return fail(HALP_INVALID_INPUT, "lm_halp: bits must be <= 32 (inner arithmetic is 2b wide)");
    if (c->option != 0) return fail(HALP_INVALID_INPUT, "lm_halp: only the last-iterate epoch update is defined");
    if (!p->qbits) return fail(HALP_INVALID_INPUT, "lm_halp: dataset has no quantized examples");
    if (p->qbits != c->bits) return fail(HALP_INVALID_INPUT, "lm_halp: dataset quantized at a different width");
    if (c->bits > 16) return fail(HALP_UNSUPPORTED, "lm_halp: the B200 inner loop supports bits <= 16");
    if (p->D > kLmMaxD) return fail(HALP_UNSUPPORTED, "lm_halp: d * classes above 4096");
    if (p->world > 1 || p->comm) return fail(HALP_UNSUPPORTED, "lm_halp: single-GPU problems only");
  }
  return HALP_OK;
}

// Scale exponent of the fixed-point exchange (k_inner.cu FX; oracle oq_fx_exponent):
// every |x_j (w~_j + z_j)| <= xmax (|w~_j| + delta 2^(b-1)), so all partial and
// total sums stay below B = xmax (|w~|_1 + D delta 2^(b-1)); S = 59 - ilogb(B) keeps
// B 2^S < 2^60 (3 bits of headroom below int64's 2^63)
int fx_exponent(double xmax, const double* w, int64_t D, double delta, int bits) {
  double l1 = 0.0;
  for (int64_t j = 0; j < D; ++j) l1 += std::fabs(w[j]);
  const double B = xmax * (l1 + (double)D * delta * std::ldexp(1.0, bits - 1));
  if (!(B > 0.0) || !std::isfinite(B)) return 0;
  const int S = 59 - std::ilogb(B);
  return S < -1000 ? -1000 : S > 1000 ? 1000 : S;
}

// LM-HALP scale chain (optimizers.cpp:509-521; theory.cpp:93-102)
int lm_scales(double gn, const halp_config* c, double delta_d, double* dm, double* di, double* daux, bool check) {
  *dm = *di = *daux = 0.0;
  if (std::isfinite(gn) && gn > 0.0) {
    const double span = std::ldexp(1.0, c->bits - 1) - 1.0;
    const double s = std::max(gn / (c->mu * span), c->delta_min);
    const double di0 = std::ldexp(s, -c->bits);
    *daux = di0 / delta_d;
    if (check && !(std::isfinite(*daux) && *daux > 0.0))
      return fail(HALP_INVALID_INPUT, "lm_halp: auxiliary scale left the double range");
    *di = *daux * delta_d;
    *dm = std::ldexp(*di, c->bits);
  }
  return HALP_OK;
}

}  // namespace

extern "C" {

const char* halp_last_error(void) { return g_err.c_str(); }
int32_t halp_abi_version(void) { return HALP_ABI_VERSION; }

int halp_shard_plan(int64_t n, int32_t d, int32_t C, int32_t dtype, int32_t world, int32_t rank, int64_t* split_begin,
                    int64_t* split_end, int64_t* splits_total, int64_t* row_begin, int64_t* row_end) {
  if (n < 1 || d < 1 || C < 1 || world < 1 || rank < 0 || rank >= world || (world & (world - 1)))
    return fail(HALP_INVALID_INPUT, "halp_shard_plan: bad arguments (world must be a power of two)");
  ShardPlan sp = shard_plan_for(n, d, C, dtype, world, rank);
  *split_begin = sp.split_begin;
  *split_end = sp.split_end;
  *splits_total = sp.S;
  *row_begin = sp.row_begin;
  *row_end = sp.row_end;
  return HALP_OK;
}

int halp_plan_for(int64_t n, int32_t d, int32_t C, int32_t dtype, int32_t world, int32_t rank, halp_plan* out) {
  if (!out || n < 1 || d < 1 || C < 1 || dtype < 0 || dtype > 2 || world < 1 || rank < 0 || rank >= world ||
      (world & (world - 1)))
    return fail(HALP_INVALID_INPUT, "halp_plan_for: bad arguments");
  KernelPlan kp;
  int rc = plan_for(n, d, C, dtype, &kp);
  if (rc) return rc;
  const ShardPlan sp = shard_plan_for(n, d, C, dtype, world, rank);
  out->fg_threads = kp.fg.threads;
  out->fg_vec = 16 / elem_size(dtype);
  out->fg_splits = (int32_t)sp.S;
  out->in_ctas = kp.in.ctas;
  out->in_threads = kp.in.threads;
  out->in_per = kp.in.per;
  out->in_levels = kp.in.levels > 1 ? kp.in.levels : 1;
  out->fg_rows_per_stage = kp.fg.fast ? kp.fg.rows : 2;
  out->fg_stages = kp.fg.fast ? kp.fg.stages : 4;
  out->fg_split_begin = sp.split_begin;
  out->fg_split_end = sp.split_end;
  return HALP_OK;
}

uint64_t halp_rng_state_after(uint64_t seed, uint64_t stream, uint64_t count) {
  return JumpTables::get().jump(rng_seed_state(seed, stream), count);
}

int halp_problem_create(const halp_problem_desc* desc, halp_problem** out) {
  if (!desc || !out) return fail(HALP_INVALID_INPUT, "halp_problem_create: null argument");
  *out = nullptr;
  // Objective ctor checks (objectives.cpp:135-160)
  if (!(std::isfinite(desc->l2) && desc->l2 >= 0.0)) return fail(HALP_INVALID_INPUT, "Objective: l2 must be finite and >= 0");
  if (desc->n < 1 || desc->d < 1 || !desc->X) return fail(HALP_INVALID_INPUT, "Objective: dataset is empty");
  if (desc->dtype < 0 || desc->dtype > 2) return fail(HALP_INVALID_INPUT, "Objective: bad dtype");
  int C = 1;
  if (desc->loss == HALP_SQUARED) {
    if (!desc->y) return fail(HALP_INVALID_INPUT, "Objective: squared loss needs one target per row");
  } else if (desc->loss == HALP_SOFTMAX) {
    if (desc->num_classes < 2 || !desc->labels) return fail(HALP_INVALID_INPUT, "Objective: softmax loss needs labels and classes");
    C = desc->num_classes;
  } else {
    return fail(HALP_INVALID_INPUT, "Objective: unknown loss family");
  }
  if (C > kMaxClasses) return fail(HALP_UNSUPPORTED, "Objective: more than 15 softmax classes");
  const int world = std::max(1, desc->world_size);
  if (world & (world - 1)) return fail(HALP_INVALID_INPUT, "world_size must be a power of two");
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0)
    return fail(HALP_CUDA_ERROR, std::string("no CUDA device (no CPU fallback): ") + cudaGetErrorString(ce));
  if (desc->device < 0 || desc->device >= ndev) return fail(HALP_INVALID_INPUT, "device index out of range");
  CU(cudaSetDevice(desc->device));
  int major = 0;
  CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, desc->device));
  if (major != 10) return fail(HALP_CUDA_ERROR, "libhalp_b200 is built for sm_100a (B200) only");
  if (pool_setup(desc->device)) return fail(HALP_CUDA_ERROR, "cannot configure the device memory pool");

  auto* p = new halp_problem();
  p->device = desc->device;
  p->dtype = desc->dtype;
  p->loss = desc->loss;
  p->n = desc->n;
  p->d = desc->d;
  p->C = C;
  p->D = desc->d * C;
  p->l2 = desc->l2;
  p->world = world;
  p->rank = desc->rank;
  auto bail = [&](int rc) {
    delete p;
    return rc;
  };
  if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(HALP_CUDA_ERROR, "cudaStreamCreate failed"));
  const int es = elem_size(p->dtype);
  // rows padded to 16 bytes so every row tile is one bulk copy
  p->ld = (int)(((int64_t)p->d * es + 15) / 16 * 16 / es);
  const bool dev_in = desc->mem == HALP_MEM_DEVICE;
  const bool aligned = ((uintptr_t)desc->X % 16) == 0;
  if (dev_in && p->ld == p->d && aligned) {
    p->X = const_cast<void*>(desc->X);
    p->own_X = false;
  } else {
    const size_t bytes = (size_t)p->n * p->ld * es;
    if (dalloc(&p->X, bytes, p->stream) != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "cudaMallocAsync(X) failed"));
    p->own_X = true;
    // padding columns must be zero: kernels process whole 16-byte groups
    if (p->ld != p->d && cudaMemsetAsync(p->X, 0, bytes, p->stream) != cudaSuccess)
      return bail(fail(HALP_CUDA_ERROR, "cudaMemset(X) failed"));
    // async on the problem's stream (a DMA straight from pinned host memory); a
    // plain 1-D copy when the rows need no padding
    const cudaMemcpyKind kind = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // In 256 MiB pieces with at most 1 GiB queued: the copy engine serves the
    // queued copies in order, so another problem's small per-epoch copies (a
    // solve running while this one uploads) wait for one GiB, not for all of X.
    cudaError_t ce2 = cudaSuccess;
    if (p->ld == p->d) {
      // groups of 4 chunks; the host waits for group g-1 after queueing group g,
      // so 1-2 GiB stay queued (no bubble) and never all of X
      constexpr size_t kChunk = (size_t)256 << 20;
      cudaEvent_t ev[2] = {nullptr, nullptr};
      if (!dev_in) {
        ce2 = cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
        if (ce2 == cudaSuccess) ce2 = cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
      }
      int queued = 0, group = 0;
      for (size_t off = 0; off < bytes && ce2 == cudaSuccess; off += kChunk) {
        ce2 = cudaMemcpyAsync(static_cast<char*>(p->X) + off, static_cast<const char*>(desc->X) + off,
                              std::min(kChunk, bytes - off), kind, p->stream);
        if (ce2 == cudaSuccess && !dev_in && ++queued == 4) {
          queued = 0;
          ce2 = cudaEventRecord(ev[group & 1], p->stream);
          if (ce2 == cudaSuccess && group > 0) ce2 = cudaEventSynchronize(ev[(group - 1) & 1]);
          ++group;
        }
      }
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    } else {
      ce2 = cudaMemcpy2DAsync(p->X, (size_t)p->ld * es, desc->X, (size_t)p->d * es, (size_t)p->d * es, (size_t)p->n,
                              kind, p->stream);
    }
    if (ce2 != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "copy of X to the device failed"));
    if (!dev_in) p->create_h2d += (int64_t)p->n * p->d * es;
  }
  if (p->loss == HALP_SQUARED) {
    if (dalloc(&p->y, sizeof(double) * p->n, p->stream) != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "cudaMallocAsync(y)"));
    if (cudaMemcpyAsync(p->y, desc->y, sizeof(double) * p->n, dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                        p->stream) != cudaSuccess)
      return bail(fail(HALP_CUDA_ERROR, "copy of y failed"));
    if (!dev_in) p->create_h2d += (int64_t)p->n * 8;
  } else {
    // Objective ctor: every label in [0, C) (objectives.cpp:150-153); host labels are checked in place
    std::vector<int32_t> lab;
    const int32_t* lh = static_cast<const int32_t*>(desc->labels);
    if (dev_in) {
      lab.resize(p->n);
      if (copy_sync(lab.data(), desc->labels, sizeof(int32_t) * p->n, cudaMemcpyDeviceToHost, p->stream) != cudaSuccess)
        return bail(fail(HALP_CUDA_ERROR, "copy of labels failed"));
      lh = lab.data();
    }
    for (int64_t i = 0; i < p->n; ++i)
      if (lh[i] < 0 || lh[i] >= C) return bail(fail(HALP_INVALID_INPUT, "Objective: label outside [0, num_classes)"));
    if (dalloc(&p->labels, sizeof(int32_t) * p->n, p->stream) != cudaSuccess)
      return bail(fail(HALP_CUDA_ERROR, "cudaMallocAsync(labels)"));
    if (cudaMemcpyAsync(p->labels, desc->labels, sizeof(int32_t) * p->n,
                        dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, p->stream) != cudaSuccess)
      return bail(fail(HALP_CUDA_ERROR, "copy of labels failed"));
    if (!dev_in) p->create_h2d += (int64_t)p->n * 4;
  }
  if (desc->qcodes) {
    // QuantizedExamples: one LPRepr, codes within its width (LPVector ctor, fixed_point.cpp:83-93)
    if (desc->qbits < 2 || desc->qbits > 64 || !(std::isfinite(desc->qdelta) && desc->qdelta > 0.0))
      return bail(fail(HALP_INVALID_INPUT, "LPRepr: delta must be positive and finite"));
    p->qbits = desc->qbits;
    p->qdelta = desc->qdelta;
    if (desc->qbits <= 16) {  // wider codes: kept as metadata only (halp_run reports UNSUPPORTED)
      const size_t cnt = (size_t)p->n * p->d;
      const int64_t* src = desc->qcodes;  // host memory whatever desc->mem says (halp_quantize_dataset output)
      const int64_t lo = -(1LL << (desc->qbits - 1)), hi = (1LL << (desc->qbits - 1)) - 1;
      p->qbytes = desc->qbits <= 8 ? 1 : 2;
      std::vector<char> packed(cnt * p->qbytes);
      for (size_t k = 0; k < cnt; ++k) {
        if (src[k] < lo || src[k] > hi) return bail(fail(HALP_INVALID_INPUT, "LPVector: code outside representable range"));
        if (p->qbytes == 1) reinterpret_cast<int8_t*>(packed.data())[k] = (int8_t)src[k];
        else reinterpret_cast<int16_t*>(packed.data())[k] = (int16_t)src[k];
      }
      if (dalloc(&p->q, packed.size(), p->stream) != cudaSuccess ||
          copy_sync(p->q, packed.data(), packed.size(), cudaMemcpyHostToDevice, p->stream) != cudaSuccess)
        return bail(fail(HALP_CUDA_ERROR, "upload of the quantized codes failed"));
      if (dalloc(&p->phi, sizeof(double) * (size_t)p->n * C, p->stream) != cudaSuccess ||
          dalloc(&p->hdev, sizeof(long long) * (size_t)p->d * C, p->stream) != cudaSuccess ||
          dalloc(&p->lm_bad, sizeof(int), p->stream) != cudaSuccess)
        return bail(fail(HALP_CUDA_ERROR, "cudaMallocAsync(LM buffers)"));
    }
  }
  p->sp = shard_plan_for(p->n, p->d, C, p->dtype, world, p->rank);
  int rc = choose_plans(p);
  if (rc) return bail(rc);
  if (desc->collective < 0 || desc->collective > 2)
    return bail(fail(HALP_INVALID_INPUT, "halp_problem_create: collective must be 0, 1 or 2"));
  if (desc->rank < 0 || desc->rank >= world) return bail(fail(HALP_INVALID_INPUT, "rank outside [0, world_size)"));
  p->host_exchange = desc->collective == 2;
  if (!p->host_exchange && (world > 1 || desc->collective == 1)) {
    if (!desc->nccl_id) return bail(fail(HALP_INVALID_INPUT, "the NCCL route needs an ncclUniqueId"));
    if (!Nccl::get().load()) return bail(fail(HALP_NCCL_ERROR, "cannot load libnccl.so.2"));
    ncclUniqueId id;
    std::memcpy(&id, desc->nccl_id, sizeof id);
    ncclResult_t r = Nccl::get().commInitRank(&p->comm, world, id, p->rank);
    if (r != ncclSuccess) return bail(fail(HALP_NCCL_ERROR, std::string("ncclCommInitRank: ") + Nccl::get().errStr(r)));
  }
  rc = ensure_workspace(p);
  if (rc) return bail(rc);
  // load and configure the planned K1 / K3 kernels now (lazy module loading
  // would otherwise put a first-launch delay of several ms inside a solve's
  // first epoch and inside its event-timed kernels)
  {
    FgLaunch L = p->fg;
    L.nsplit_local = (int)p->sp.local_splits();
    L.dry = 1;
    FgParams fp = fg_params(p, 0);
    const cudaError_t e1 = launch_fullgrad(L, fp, p->stream);
    if (e1 != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, std::string("K1 preparation failed: ") + cudaGetErrorString(e1)));
    InLaunch IL = p->in;
    IL.dry = 1;
    InParams ip{};
    ip.loss = p->loss;
    ip.d = p->d;
    ip.C = p->C;
    ip.D = (int)p->D;
    for (int mode = 0; mode < 2; ++mode) {
      ip.mode = mode;
      const cudaError_t e3 = launch_inner(IL, ip, p->stream);
      if (e3 != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, std::string("K3 preparation failed: ") + cudaGetErrorString(e3)));
    }
  }
  // bf16 two-class sweeps may convert X with integer ops (k1_stream); that
  // needs every element finite, checked once here on the device
  if (p->dtype == HALP_BF16 && C == 2 && env_int("HALP_FG_F2F", 0) == 0) {
    int* flag = nullptr;
    int bad = 1;
    if (dalloc(&flag, sizeof(int), p->stream) != cudaSuccess || cudaMemsetAsync(flag, 0, sizeof(int), p->stream) ||
        launch_nonfinite_bf16(p->X, p->n * (int64_t)p->ld, flag, p->stream) ||
        cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, p->stream) ||
        cudaStreamSynchronize(p->stream) || cudaFreeAsync(flag, p->stream))
      return bail(fail(HALP_CUDA_ERROR, "finiteness check of X failed"));
    p->x_finite = bad ? 0 : 1;
  }
  // the caller may release its host buffers when create returns
  if (cudaStreamSynchronize(p->stream) != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "upload of the dataset failed"));
  p->timing.h2d_bytes = p->create_h2d;
  *out = p;
  return HALP_OK;
}

void halp_problem_destroy(halp_problem* p) { delete p; }

int halp_problem_plan(const halp_problem* p, halp_plan* out) {
  if (!p || !out) return fail(HALP_INVALID_INPUT, "halp_problem_plan: null argument");
  out->fg_threads = p->fg.threads;
  out->fg_vec = 16 / elem_size(p->dtype);
  out->fg_splits = (int32_t)p->sp.S;
  out->in_ctas = p->in.ctas;
  out->in_threads = p->in.threads;
  out->in_per = p->in.per;
  out->in_levels = p->in.levels > 1 ? p->in.levels : 1;
  out->fg_rows_per_stage = p->fg.fast ? p->fg.rows : 2;
  out->fg_stages = p->fg.fast ? p->fg.stages : 4;
  out->fg_split_begin = p->sp.split_begin;
  out->fg_split_end = p->sp.split_end;
  return HALP_OK;
}

int halp_set_trace(halp_problem* p, int64_t* codes, int64_t cap) {
  if (!p) return fail(HALP_INVALID_INPUT, "halp_set_trace: null problem");
  p->trace_host = codes;
  p->trace_cap = codes ? cap : 0;
  return HALP_OK;
}

int halp_last_timing(const halp_problem* p, halp_timing* out) {
  if (!p || !out) return fail(HALP_INVALID_INPUT, "halp_last_timing: null argument");
  *out = p->timing;
  return HALP_OK;
}

int halp_rank_partial(halp_problem* p, const double* w, double* root) {
  if (!p || !w || !root) return fail(HALP_INVALID_INPUT, "halp_rank_partial: null argument");
  CU(cudaSetDevice(p->device));
  const int64_t D1 = p->D + 1;
  const int nloc = (int)p->sp.local_splits();
  CU(p_h2d(p, p->w, w, sizeof(double) * p->D));
  for (int pass = 0; pass < p->fg_passes; ++pass) {
    FgParams fp = fg_params(p, pass);
    FgLaunch L = p->fg;
    L.nsplit_local = nloc;
    CU(launch_fullgrad(L, fp, p->stream));
  }
  CU(launch_split_tree(p->partials, nloc, (int)D1, p->rank_sum, p->tree_scratch, p->stream));
  CU(copy_sync(root, p->rank_sum, sizeof(double) * D1, cudaMemcpyDeviceToHost, p->stream));
  return HALP_OK;
}

int halp_finalize_gathered(halp_problem* p, const double* w, const double* gathered, double* g, double* loss) {
  if (!p || !w || !gathered) return fail(HALP_INVALID_INPUT, "halp_finalize_gathered: null argument");
  CU(cudaSetDevice(p->device));
  const int64_t D1 = p->D + 1;
  CU(p_h2d(p, p->w, w, sizeof(double) * p->D));
  CU(copy_sync(p->gathered, gathered, sizeof(double) * D1 * p->world, cudaMemcpyHostToDevice, p->stream));
  FinParams fin{p->gathered, p->world, p->D, p->w, p->n, p->l2, 1.0, 1e-300, 8, p->g, p->stats};
  CU(launch_finalize(fin, p->stream));
  double st[3];
  CU(p_d2h(p, st, p->stats, sizeof st));
  if (g) CU(p_d2h(p, g, p->g, sizeof(double) * p->D));
  if (loss) *loss = st[2];
  return HALP_OK;
}

int halp_full_gradient(halp_problem* p, const double* w, double* g, double* loss) {
  if (!p || !w) return fail(HALP_INVALID_INPUT, "halp_full_gradient: null argument");
  if (p->host_exchange) return fail(HALP_INVALID_INPUT, "host-exchange problem: use halp_rank_partial / halp_finalize_gathered");
  CU(cudaSetDevice(p->device));
  p->timing = halp_timing{};
  CU(p_h2d(p, p->w, w, sizeof(double) * p->D));
  double gn, delta, l;
  int rc = full_pass(p, &gn, &delta, &l, 1.0, 8, 1e-300);
  if (rc) return rc;
  if (g) CU(p_d2h(p, g, p->g, sizeof(double) * p->D));
  if (loss) *loss = l;
  return HALP_OK;
}

int halp_bench_full_gradient(halp_problem* p, int reps, double* ms_per_pass) {
  if (!p || reps < 1 || p->host_exchange) return fail(HALP_INVALID_INPUT, "halp_bench_full_gradient: bad arguments");
  CU(cudaSetDevice(p->device));
  const int64_t D1 = p->D + 1;
  const int nloc = (int)p->sp.local_splits();
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  CU(cudaEventRecord(a, p->stream));
  for (int r = 0; r < reps; ++r) {
    for (int pass = 0; pass < p->fg_passes; ++pass) {
      FgParams fp = fg_params(p, pass);
      FgLaunch L = p->fg;
      L.nsplit_local = nloc;
      CU(launch_fullgrad(L, fp, p->stream));
    }
    CU(launch_split_tree(p->partials, nloc, (int)D1, p->comm ? p->rank_sum : p->gathered, p->tree_scratch,
                         p->stream));
    if (p->comm) {  // the exchange step is part of a sharded pass
      int rc = gather_finalize(p, 1.0, 8, 1e-300);
      if (rc) return rc;
    }
  }
  CU(cudaEventRecord(b, p->stream));
  CU(cudaEventSynchronize(b));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms_per_pass = ms / reps;
  return HALP_OK;
}

// lpopt::run_lm_halp (optimizers.cpp:461-627, the integer inner loop): per
// epoch K7 (k_lm_stats) + split tree + k_finalize -> g, |g|, loss and the
// logits phi at w~; the scale chain and the h codes on the host; K4 sample
// indices; K8 (k3_lm) the T integer steps.
static int run_lm(halp_problem* p, const halp_config* cfg, halp_record* rec) {
  const int64_t n = p->n, D = p->D;
  const int d = p->d, C = p->C, b = cfg->bits;
  const int64_t T = cfg->inner_steps > 0 ? cfg->inner_steps : (int64_t)cfg->full_grad_period * n;
  if (T < 1) return fail(HALP_INVALID_INPUT, "optimizer: epoch length must be >= 1");
  p->timing = halp_timing{};
  if (p->idx_cap < T) {
    if (p->idx) cudaFreeAsync(p->idx, p->stream);
    CU(dalloc(&p->idx, sizeof(int64_t) * T, p->stream));
    p->idx_cap = T;
  }
  const uint64_t* jtab = nullptr;
  const uint64_t* ptab = nullptr;
  {
    int rc = rng_tables(p->device, (int64_t)C * (d + 1), &ptab, &jtab, p->stream);
    if (rc) return rc;
  }
  const auto& jt = JumpTables::get();
  const uint64_t s_sample = rng_seed_state(cfg->seed, 0);
  const uint64_t s_round = rng_seed_state(cfg->seed, 1);
  std::vector<double> wh(D, 0.0), gh(D);
  if (cfg->init) std::memcpy(wh.data(), cfg->init, sizeof(double) * D);
  CU(p_h2d(p, p->w, wh.data(), sizeof(double) * D));
  p->timing.h2d_bytes += sizeof(double) * D;
  int64_t tr_steps = p->trace_cap > 0 ? std::min<int64_t>(T, p->trace_cap / D) : 0, traced = 0;
  if (tr_steps > p->trace_dev_steps) {
    if (p->trace_dev) cudaFreeAsync(p->trace_dev, p->stream);
    CU(dalloc(&p->trace_dev, sizeof(long long) * tr_steps * D, p->stream));
    p->trace_dev_steps = tr_steps;
  }
  rec->rows_n = 0;
  rec->status = HALP_STATUS_OK;
  rec->steps_taken = 0;
  rec->inner_fp_vector_ops = 0;
  rec->inner_lp_vector_ops = 0;
  Recorder r{cfg, rec, now_s(), 0.0, (int)D};
  const int64_t D1 = D + 1;
  const int nloc = (int)p->sp.local_splits();
  // K7 + tree + finalize at p->w -> g (device), stats -> host
  auto stats = [&](double* gn, double* loss) -> int {
    CU(cudaEventRecord(p->ev_fg.a, p->stream));
    LmStatsParams sp{p->q, n, d, C, p->loss, p->qdelta, p->y, p->labels, p->w, (int)p->sp.S, (int)p->sp.split_begin,
                     p->partials, p->phi};
    CU(launch_lm_stats(sp, nloc, p->qbytes, p->stream));
    CU(launch_split_tree(p->partials, nloc, (int)D1, p->gathered, p->tree_scratch, p->stream));
    CU(cudaEventRecord(p->ev_fg.b, p->stream));
    FinParams fin{p->gathered, 1, (int)D, p->w, n, p->l2, 1.0, 1e-300, 8, p->g, p->stats};
    CU(launch_finalize(fin, p->stream));
    p->timing.kernel_launches += 3;
    p->timing.fullgrad_launches += 1;
    double st[3];
    CU(p_d2h(p, st, p->stats, sizeof st));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, p->ev_fg.a, p->ev_fg.b));
    p->timing.fullgrad_ms += ms;
    *gn = st[0];
    *loss = st[2];
    return HALP_OK;
  };
  const uint64_t per_step = (uint64_t)C * (uint64_t)(d + 1);
  const uint64_t per_epoch = 2 * (uint64_t)D + (uint64_t)T * per_step;
  const long long maxb = (1LL << (b - 1)) - 1, minb = -(1LL << (b - 1));
  int64_t steps = 0;
  bool converged = false;
  for (int k = 0; k < cfg->epochs && !converged; ++k) {
    double gn, loss, dm, di, daux;
    int rc = stats(&gn, &loss);
    if (rc) return rc;
    CU(p_d2h(p, wh.data(), p->w, sizeof(double) * D));
    rc = lm_scales(gn, cfg, p->qdelta, &dm, &di, &daux, true);
    if (rc) return rc;
    rc = r.boundary((double)steps / (double)n, wh.data(), loss, gn, dm, k == 0 || gn == 0.0, di, daux);
    if (rc) return rc;
    if (gn == 0.0) {
      rec->status = HALP_STATUS_CONVERGED;
      converged = true;
      break;
    }
    // h = Q_inner(alpha g~) (widen_range keeps the codes); its D draws follow Q_m(0)'s D
    CU(p_d2h(p, gh.data(), p->g, sizeof(double) * D));
    std::vector<long long> hh(D);
    uint64_t st = jt.jump(s_round, (uint64_t)k * per_epoch + (uint64_t)D);
    for (int64_t q = 0; q < D; ++q) {
      st = xs_step_host(st);
      const double u = (double)((st * 0x2545F4914F6CDD1DULL) >> 11) * 0x1.0p-53;
      const double a = cfg->alpha * gh[q];
      if (!std::isfinite(a)) return fail(HALP_INVALID_INPUT, "quantize: input must be finite");
      hh[q] = (long long)host_quantize_code(a, di, b, u);
      (void)maxb;
      (void)minb;
    }
    CU(p_h2d(p, p->hdev, hh.data(), sizeof(long long) * D));
    const uint64_t sbase = jt.jump(s_sample, (uint64_t)k * (uint64_t)T);
    CU(cudaEventRecord(p->ev_smp.a, p->stream));
    CU(launch_samples(sbase, T, 0, (uint64_t)T, (uint64_t)n, p->pow_tab, p->idx, nullptr, p->stream));
    CU(cudaEventRecord(p->ev_smp.b, p->stream));
    CU(cudaMemsetAsync(p->lm_bad, 0, sizeof(int), p->stream));
    LmInnerParams ip{p->q, d, C, p->loss, b, p->phi, p->y, p->labels, cfg->alpha, daux, dm, p->qdelta * dm,
                     p->hdev, p->w, p->w2, p->idx, T, jt.jump(s_round, (uint64_t)k * per_epoch + 2 * (uint64_t)D),
                     ptab, jtab, tr_steps > 0 ? p->trace_dev : nullptr, tr_steps, p->lm_bad};
    CU(cudaEventRecord(p->ev_in.a, p->stream));
    CU(launch_lm_inner(ip, p->qbytes, p->stream));
    CU(cudaEventRecord(p->ev_in.b, p->stream));
    p->timing.kernel_launches += 2;
    p->timing.inner_launches += 1;
    int bad = 0;
    CU(p_d2h(p, &bad, p->lm_bad, sizeof(int)));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, p->ev_in.a, p->ev_in.b));
    p->timing.inner_ms += ms;
    CU(cudaEventElapsedTime(&ms, p->ev_smp.a, p->ev_smp.b));
    p->timing.sample_ms += ms;
    if (bad) return fail(HALP_INVALID_INPUT, "quantize: input must be finite");
    if (tr_steps > 0 && p->trace_host && traced < p->trace_cap) {
      const int64_t cnt = std::min<int64_t>(tr_steps * D, p->trace_cap - traced);
      std::vector<long long> tmp(cnt);
      CU(copy_sync(tmp.data(), p->trace_dev, sizeof(long long) * cnt, cudaMemcpyDeviceToHost, p->stream));
      for (int64_t q = 0; q < cnt; ++q) p->trace_host[traced + q] = tmp[q];
      traced += cnt;
    }
    p->timing.inner_steps += T;
    std::swap(p->w, p->w2);
    rec->inner_lp_vector_ops += (uint64_t)(6 * C) * (uint64_t)T;
    steps += T;
  }
  if (!converged) {
    double gn, loss, dm, di, daux;
    int rc = stats(&gn, &loss);
    if (rc) return rc;
    CU(p_d2h(p, wh.data(), p->w, sizeof(double) * D));
    lm_scales(gn, cfg, p->qdelta, &dm, &di, &daux, false);
    rc = r.boundary((double)steps / (double)n, wh.data(), loss, gn, dm, true, di, daux);
    if (rc) return rc;
    if (gn == 0.0) rec->status = HALP_STATUS_CONVERGED;
  } else {
    CU(p_d2h(p, wh.data(), p->w, sizeof(double) * D));
  }
  if (rec->final_iterate) std::memcpy(rec->final_iterate, wh.data(), sizeof(double) * D);
  rec->steps_taken = steps;
  return HALP_OK;
}

int halp_run(halp_problem* p, const halp_config* cfg, halp_record* rec) {
  // lpopt::run_halp (optimizers.cpp:387-459), run_svrg (:258-296) and
  // run_lp_svrg (:336-385): one epoch loop, K1 + K2 at the boundary, K4 + K3
  // inside; the three differ in the K3 mode and in how z / the scale start.
  if (!p || !cfg || !rec) return fail(HALP_INVALID_INPUT, "halp_run: null argument");
  if (p->host_exchange) return fail(HALP_INVALID_INPUT, "host-exchange problem: use halp_rank_partial / halp_finalize_gathered");
  int rc = validate(p, cfg);
  if (rc) return rc;
  CU(cudaSetDevice(p->device));
  if (cfg->algorithm == HALP_ALGO_LM_HALP) return run_lm(p, cfg, rec);
  const int algo = cfg->algorithm;
  const bool halp = algo == HALP_ALGO_HALP;
  const bool lp = algo == HALP_ALGO_LP_SVRG || algo == HALP_ALGO_LP_SGD;  // fixed-scale quantized iterate
  const bool sgd = algo == HALP_ALGO_SGD || algo == HALP_ALGO_LP_SGD;    // no variance reduction, no option II
  const int mode = halp ? 0 : algo == HALP_ALGO_LP_SVRG ? 1 : algo == HALP_ALGO_SVRG ? 2 : algo == HALP_ALGO_SGD ? 3 : 4;
  const int64_t n = p->n, D = p->D;
  const int64_t T = cfg->inner_steps > 0 ? cfg->inner_steps : (int64_t)cfg->full_grad_period * n;
  if (T < 1) return fail(HALP_INVALID_INPUT, "optimizer: epoch length must be >= 1");
  const int opt2 = cfg->option == 1 && !sgd;
  p->timing = halp_timing{};
  if (p->idx_cap < T) {
    if (p->idx) cudaFreeAsync(p->idx, p->stream);
    CU(dalloc(&p->idx, sizeof(int64_t) * T, p->stream));
    p->idx_cap = T;
  }
  const auto& jt = JumpTables::get();
  const uint64_t s_sample = rng_seed_state(cfg->seed, 0);  // kSampleStream
  const uint64_t s_round = rng_seed_state(cfg->seed, 1);   // kRoundStream
  std::vector<double> wh(D, 0.0);
  if (cfg->init) std::memcpy(wh.data(), cfg->init, sizeof(double) * D);
  // z at the start of the first epoch: HALP resets it per epoch (Q(0));
  // LP-SVRG / LP-SGD quantize the initial iterate once (D rounding draws); SVRG / SGD hold w itself
  std::vector<double> z0(D, 0.0);
  if (lp) {
    uint64_t st = s_round;
    for (int64_t q = 0; q < D; ++q) {
      st = xs_step_host(st);
      const double u = (double)((st * 0x2545F4914F6CDD1DULL) >> 11) * 0x1.0p-53;
      if (!std::isfinite(wh[q])) return fail(HALP_INVALID_INPUT, "quantize: input must be finite");
      z0[q] = (double)host_quantize_code(wh[q], cfg->delta, cfg->bits, u);
    }
    for (int64_t q = 0; q < D; ++q) wh[q] = z0[q] * cfg->delta;  // to_real
  } else if (!halp) {
    z0 = wh;
  }
  CU(p_h2d(p, p->w, wh.data(), sizeof(double) * D));
  p->timing.h2d_bytes += sizeof(double) * D;
  double* zin = p->zb0;
  double* zout = p->zb1;
  if (!halp) {
    CU(p_h2d(p, zin, z0.data(), sizeof(double) * D));
    p->timing.h2d_bytes += sizeof(double) * D;
  }

  // trace buffer (test hook)
  int64_t traced = 0;
  int64_t tr_steps = p->trace_cap > 0 ? std::min<int64_t>(T, p->trace_cap / D) : 0;
  if (tr_steps > p->trace_dev_steps) {
    if (p->trace_dev) cudaFreeAsync(p->trace_dev, p->stream);
    CU(dalloc(&p->trace_dev, sizeof(long long) * tr_steps * D, p->stream));
    p->trace_dev_steps = tr_steps;
  }

  rec->rows_n = 0;
  rec->status = HALP_STATUS_OK;
  rec->steps_taken = 0;
  rec->inner_fp_vector_ops = 0;
  rec->inner_lp_vector_ops = 0;
  Recorder r{cfg, rec, now_s(), 0.0, (int)D};
  const int bits = halp || lp ? cfg->bits : 64;
  const double hi = bits == 64 ? (double)INT64_MAX : (double)((1LL << (bits - 1)) - 1);
  const double lo = bits == 64 ? (double)INT64_MIN : (double)(-(1LL << (bits - 1)));
  const long long maxc = bits == 64 ? INT64_MAX : (1LL << (bits - 1)) - 1;
  const long long minc = bits == 64 ? INT64_MIN : -(1LL << (bits - 1));
  // instr counters per inner step: two component gradients (2 each) + the
  // update (+ quantize_vector, to_real; HALP counts both its updates)
  const uint64_t ops_per_step = halp ? 8 : sgd ? (lp ? 5 : 3) : (lp ? 7 : 5);
  const double mu = halp ? cfg->mu : 1.0;
  int64_t steps = 0;
  bool converged = false;
  for (int k = 0; k < cfg->epochs && !converged; ++k) {
    double gn, delta, loss;
    rc = full_pass(p, &gn, &delta, &loss, mu, bits, cfg->delta_min);
    if (rc) return rc;
    CU(p_d2h(p, wh.data(), p->w, sizeof(double) * D));
    p->timing.d2h_bytes += sizeof(double) * D;
    const double row_delta = halp ? delta : lp ? cfg->delta : 0.0;
    rc = r.boundary((double)steps / (double)n, wh.data(), loss, gn, row_delta, k == 0 || (halp && gn == 0.0));
    if (rc) return rc;
    if (halp && gn == 0.0) {
      rec->status = HALP_STATUS_CONVERGED;
      converged = true;
      break;
    }
    if (halp && !(std::isfinite(delta) && delta > 0.0))
      return fail(HALP_INVALID_INPUT, "LPRepr: delta must be positive and finite");
    const double kdelta = halp ? delta : lp ? cfg->delta : 1.0;
    // sample stream: epoch k starts after k*(T+opt2) draws; option II draws t_pick first
    const uint64_t sbase = jt.jump(s_sample, (uint64_t)k * (uint64_t)(T + opt2));
    int64_t t_pick = -1;
    uint64_t s0 = sbase;
    if (opt2) {
      s0 = xs_step_host(sbase);
      t_pick = (int64_t)(((unsigned __int128)(s0 * 0x2545F4914F6CDD1DULL) * (unsigned __int128)T) >> 64);
    }
    CU(cudaEventRecord(p->ev_smp.a, p->stream));
    CU(launch_samples(s0, T, 0, (uint64_t)T, (uint64_t)n, p->pow_tab, p->idx, nullptr, p->stream));
    ++p->timing.kernel_launches;
    CU(cudaEventRecord(p->ev_smp.b, p->stream));
    // rounding stream at step 0 of epoch k: HALP k*D*(T+1) + D (Q(0) per epoch);
    // LP-SVRG D + k*D*T (the initial quantization once); SVRG draws none
    const uint64_t rdraws = halp ? (uint64_t)k * (uint64_t)D * (uint64_t)(T + 1) + (uint64_t)D
                                 : (uint64_t)D + (uint64_t)k * (uint64_t)D * (uint64_t)T;
    const uint64_t r0 = jt.jump(s_round, rdraws);
    CU(cudaMemsetAsync(p->blow, 0xFF, sizeof(long long), p->stream));
    const double rcp = 1.0 / kdelta;
    // fixed-point exchange (levels 3, HALP): S such that D max|x| (|w~|_1/D + delta 2^(b-1)) 2^S < 2^60
    double fx_scale = 1.0, fx_inv = 1.0;
    if (halp && p->in.levels == 3) {
      if (p->xmax < 0.0) {
        double* dm = nullptr;
        CU(dalloc(&dm, sizeof(double), p->stream));
        CU(launch_absmax(p->X, p->dtype, p->n * (int64_t)p->ld, dm, p->stream));
        CU(p_d2h(p, &p->xmax, dm, sizeof(double)));
        CU(cudaFreeAsync(dm, p->stream));
      }
      const int S = fx_exponent(p->xmax, wh.data(), D, kdelta, bits);
      fx_scale = std::ldexp(1.0, S);
      fx_inv = std::ldexp(1.0, -S);
    }
    InParams ip{p->X, p->ld, p->d, p->C, (int)D, p->loss, n, p->y, p->labels, p->l2, cfg->alpha, kdelta, hi, lo, maxc,
                minc, std::isfinite(rcp) && rcp != 0.0 && env_int("HALP_IEEE_DIV", 0) == 0 ? rcp : 0.0, p->w, p->w2,
                p->g, p->idx, T, t_pick, r0, p->pow_tab, p->jump_tab, p->codes, tr_steps > 0 ? p->trace_dev : nullptr,
                tr_steps, p->blow, p->u_out, mode, halp ? nullptr : zin, halp ? nullptr : zout, fx_scale, fx_inv};
    CU(cudaEventRecord(p->ev_in.a, p->stream));
    CU(launch_inner(p->in, ip, p->stream));
    ++p->timing.kernel_launches;
    ++p->timing.inner_launches;
    CU(cudaEventRecord(p->ev_in.b, p->stream));
    long long blow = -1;
    CU(p_d2h(p, &blow, p->blow, sizeof(long long)));
    p->timing.d2h_bytes += sizeof(long long);
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, p->ev_in.a, p->ev_in.b));
    p->timing.inner_ms += ms;
    CU(cudaEventElapsedTime(&ms, p->ev_smp.a, p->ev_smp.b));
    p->timing.sample_ms += ms;
    if (tr_steps > 0 && p->trace_host && traced < p->trace_cap) {
      const int64_t ns = std::min<int64_t>(tr_steps, (blow >= 0 ? blow : T));
      const int64_t cnt = std::min<int64_t>(ns * D, p->trace_cap - traced);
      std::vector<long long> tmp(cnt);
      CU(copy_sync(tmp.data(), p->trace_dev, sizeof(long long) * cnt, cudaMemcpyDeviceToHost, p->stream));
      for (int64_t q = 0; q < cnt; ++q) p->trace_host[traced + q] = tmp[q];
      traced += cnt;
    }
    if (blow >= 0) {
      // Recorder::blowup (optimizers.cpp:156-160; HALP :432-434, LP-SVRG :370-372)
      p->timing.inner_steps += blow + 1;
      std::vector<double> u(D);
      CU(p_d2h(p, u.data(), p->u_out, sizeof(double) * D));
      return r.boundary((double)(steps + blow + 1) / (double)n, u.data(), INFINITY, INFINITY, kdelta, true);
    }
    p->timing.inner_steps += T;
    std::swap(p->w, p->w2);  // w~ += z (HALP) / w~ = the epoch's (snapshot) iterate
    std::swap(zin, zout);    // next epoch starts from this epoch's (snapshot) codes
    rec->inner_fp_vector_ops += ops_per_step * (uint64_t)T;
    steps += T;
  }
  if (!converged) {
    double gn, delta, loss;
    rc = full_pass(p, &gn, &delta, &loss, mu, bits, cfg->delta_min);
    if (rc) return rc;
    CU(p_d2h(p, wh.data(), p->w, sizeof(double) * D));
    p->timing.d2h_bytes += sizeof(double) * D;
    rc = r.boundary((double)steps / (double)n, wh.data(), loss, gn, halp ? delta : lp ? cfg->delta : 0.0, true);
    if (rc) return rc;
    if (halp && gn == 0.0) rec->status = HALP_STATUS_CONVERGED;
  } else {
    CU(p_d2h(p, wh.data(), p->w, sizeof(double) * D));
  }
  if (rec->final_iterate) std::memcpy(rec->final_iterate, wh.data(), sizeof(double) * D);
  rec->steps_taken = steps;
  return HALP_OK;
}

}  // extern "C"

extern "C" int halp_datagen(const halp_datagen_desc* desc, int32_t device, void* X_dev, double* y_dev,
                            int32_t* labels_dev) {
  if (!desc || !X_dev) return fail(HALP_INVALID_INPUT, "halp_datagen: null argument");
  if (desc->kind < 0 || desc->kind > 2 || desc->n < 1 || desc->d < 1)
    return fail(HALP_INVALID_INPUT, "halp_datagen: bad kind or shape");
  if (desc->kind == 0 && !y_dev) return fail(HALP_INVALID_INPUT, "halp_datagen: regression needs y");
  if (desc->kind != 0 && !labels_dev) return fail(HALP_INVALID_INPUT, "halp_datagen: classification needs labels");
  if (desc->kind == 1 && (desc->num_classes < 2 || desc->num_classes > kMaxClasses))
    return fail(HALP_INVALID_INPUT, "halp_datagen: num_classes out of range");
  CU(cudaSetDevice(device));
  GenParams gp{desc->kind, desc->n, desc->d, desc->num_classes, desc->dtype, desc->noise_sd, desc->x_scale,
               desc->density, desc->seed, X_dev, y_dev, labels_dev};
  CU(launch_datagen(gp, 0));
  CU(cudaDeviceSynchronize());
  return HALP_OK;
}

struct halp_batch {
  int device = 0, dtype = 0, d = 0, ld = 0, nprob = 0, splits = 4;
  bool shared = false;
  int64_t n = 0;
  double l2 = 0.0;
  void* X = nullptr;
  double* y = nullptr;
  const uint64_t *pow_tab = nullptr, *jump_tab = nullptr;  // resident per device (rng_tables)
  cudaStream_t stream = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  void* arena = nullptr;  // per-run parameters + outputs (one pooled block, reused across runs)
  size_t arena_bytes = 0;
  ~halp_batch() {
    cudaSetDevice(device);
    for (void* q : {(void*)X, (void*)y, arena})
      if (q) cudaFreeAsync(q, stream);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (stream) cudaStreamDestroy(stream);
  }
};

extern "C" int halp_batch_create(const halp_batch_desc* desc, halp_batch** out) {
  if (!desc || !out) return fail(HALP_INVALID_INPUT, "halp_batch_create: null argument");
  *out = nullptr;
  if (desc->nprob < 1 || desc->n < 1 || desc->d < 1 || !desc->X || !desc->y)
    return fail(HALP_INVALID_INPUT, "halp_batch_create: empty problems");
  if (!(std::isfinite(desc->l2) && desc->l2 >= 0.0)) return fail(HALP_INVALID_INPUT, "Objective: l2 must be finite and >= 0");
  if (desc->d > 256) return fail(HALP_UNSUPPORTED, "halp_batch: d > 256 (use halp_run per problem)");
  if (desc->dtype < 0 || desc->dtype > 2) return fail(HALP_INVALID_INPUT, "halp_batch_create: bad dtype");
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0) return fail(HALP_CUDA_ERROR, "no CUDA device (no CPU fallback)");
  if (desc->device < 0 || desc->device >= ndev) return fail(HALP_INVALID_INPUT, "device index out of range");
  CU(cudaSetDevice(desc->device));
  if (pool_setup(desc->device)) return fail(HALP_CUDA_ERROR, "cannot configure the device memory pool");
  auto* b = new halp_batch();
  b->device = desc->device;
  b->dtype = desc->dtype;
  b->d = desc->d;
  b->n = desc->n;
  b->nprob = desc->nprob;
  b->l2 = desc->l2;
  auto bail = [&](int rc) {
    delete b;
    return rc;
  };
  const int es = elem_size(b->dtype);
  b->ld = (int)(((int64_t)b->d * es + 15) / 16 * 16 / es);
  b->splits = (int)std::max<int64_t>(4, make_shard_plan(b->n, b->d, 1, b->dtype, 1, 0).S);
  const bool dev_in = desc->mem == HALP_MEM_DEVICE;
  b->shared = desc->shared != 0;
  const size_t rows_total = (size_t)(b->shared ? 1 : b->nprob) * b->n;
  if (cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(HALP_CUDA_ERROR, "cudaStreamCreate failed"));
  if (cudaEventCreate(&b->e0) != cudaSuccess || cudaEventCreate(&b->e1) != cudaSuccess)
    return bail(fail(HALP_CUDA_ERROR, "cudaEventCreate failed"));
  cudaStream_t st = b->stream;
  // everything on the batch's own stream (stream-ordered pool, async copies), one sync at the end
  if (dalloc(&b->X, rows_total * b->ld * es, st) != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "cudaMallocAsync(X)"));
  if (b->ld != b->d && cudaMemsetAsync(b->X, 0, rows_total * b->ld * es, st) != cudaSuccess)
    return bail(fail(HALP_CUDA_ERROR, "cudaMemset(X)"));
  if (cudaMemcpy2DAsync(b->X, (size_t)b->ld * es, desc->X, (size_t)b->d * es, (size_t)b->d * es, rows_total,
                        dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st) != cudaSuccess)
    return bail(fail(HALP_CUDA_ERROR, "copy of X failed"));
  if (dalloc(&b->y, sizeof(double) * rows_total, st) != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "cudaMallocAsync(y)"));
  if (cudaMemcpyAsync(b->y, desc->y, sizeof(double) * rows_total,
                      dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st) != cudaSuccess)
    return bail(fail(HALP_CUDA_ERROR, "copy of y failed"));
  int rc = rng_tables(b->device, b->d, &b->pow_tab, &b->jump_tab, st);
  if (rc) return bail(rc);
  // the caller may release its buffers when create returns
  if (cudaStreamSynchronize(st) != cudaSuccess) return bail(fail(HALP_CUDA_ERROR, "upload of the batch failed"));
  *out = b;
  return HALP_OK;
}

extern "C" void halp_batch_destroy(halp_batch* b) { delete b; }

extern "C" int halp_batch_plan(const halp_batch* b, halp_plan* out) {
  if (!b || !out) return fail(HALP_INVALID_INPUT, "halp_batch_plan: null argument");
  *out = halp_plan{};
  out->fg_threads = 32;
  out->fg_vec = 16 / elem_size(b->dtype);
  out->fg_splits = b->splits;
  out->in_ctas = 1;
  if (batch_warps_per_problem(b->d) == 1) {  // k5_batch_w1: one warp, M = D/32 per lane
    out->in_threads = 32;
    const int M = (b->d + 31) / 32;
    out->in_per = M <= 1 ? 1 : M <= 2 ? 2 : M <= 4 ? 4 : 8;
  } else if (batch_warps_per_problem(b->d) == 2) {  // k5_batch<.., 2>: M = D/64 per thread
    out->in_threads = 64;
    const int M = (b->d + 63) / 64;
    out->in_per = M <= 1 ? 1 : M <= 2 ? 2 : 4;
  } else {  // k5_batch: 4 warps per problem, M = D/128 coordinates per thread
    out->in_threads = 128;
    out->in_per = b->d <= 128 ? 1 : 2;
  }
  out->in_levels = 1;
  out->fg_split_begin = 0;
  out->fg_split_end = b->splits;
  return HALP_OK;
}

extern "C" int halp_batch_run(halp_batch* b, const halp_config* cfgs, halp_record* recs, double* device_ms) {
  if (!b || !cfgs || !recs) return fail(HALP_INVALID_INPUT, "halp_batch_run: null argument");
  CU(cudaSetDevice(b->device));
  const int P = b->nprob, D = b->d;
  std::vector<double> alpha(P), mu(P), dmin(P), divl(P), mev(P);
  std::vector<int> bits(P), epochs(P), option(P);
  std::vector<int64_t> T(P);
  std::vector<uint64_t> seeds(2 * (size_t)P);
  std::vector<double> init((size_t)P * D, 0.0);
  bool any_init = false;
  int max_rows = 2;
  for (int q = 0; q < P; ++q) {
    const halp_config& c = cfgs[q];
    if (c.algorithm != HALP_ALGO_HALP) return fail(HALP_UNSUPPORTED, "halp_batch_run: Algorithm::Halp only");
    int rc = validate(nullptr, &c);
    if (rc) {
      g_err = "problem " + std::to_string(q) + ": " + g_err;
      return rc;
    }
    T[q] = c.inner_steps > 0 ? c.inner_steps : (int64_t)c.full_grad_period * b->n;
    alpha[q] = c.alpha;
    mu[q] = c.mu;
    dmin[q] = c.delta_min;
    divl[q] = c.divergence_limit;
    mev[q] = c.metric_every_passes;
    bits[q] = c.bits;
    epochs[q] = c.epochs;
    option[q] = c.option;
    seeds[2 * q] = rng_seed_state(c.seed, 0);
    seeds[2 * q + 1] = rng_seed_state(c.seed, 1);
    if (c.init) {
      any_init = true;
      std::memcpy(&init[(size_t)q * D], c.init, sizeof(double) * D);
    }
    max_rows = std::max(max_rows, std::max(c.epochs, 0) + 2);
  }
  // one pooled device arena for the per-problem parameters and the outputs
  // (kept by the batch and reused by the next run of the same or smaller size)
  struct Part {
    const void* src;
    size_t bytes;
    size_t off;
  };
  std::vector<Part> parts;
  size_t total = 0;
  auto part = [&](const void* src, size_t bytes) -> size_t {
    const size_t off = total;
    parts.push_back(Part{src, bytes, off});
    total += (std::max<size_t>(bytes, 8) + 255) / 256 * 256;
    return off;
  };
  const size_t o_alpha = part(alpha.data(), 8 * P), o_mu = part(mu.data(), 8 * P), o_dmin = part(dmin.data(), 8 * P),
               o_divl = part(divl.data(), 8 * P), o_mev = part(mev.data(), 8 * P), o_bits = part(bits.data(), 4 * P),
               o_ep = part(epochs.data(), 4 * P), o_opt = part(option.data(), 4 * P), o_T = part(T.data(), 8 * P),
               o_seed = part(seeds.data(), 16 * (size_t)P),
               o_init = part(any_init ? init.data() : nullptr, any_init ? 8 * (size_t)P * D : 0);
  const size_t in_bytes = total;
  const size_t o_rows = part(nullptr, 8 * 5 * (size_t)P * max_rows), o_rh = part(nullptr, 8 * (size_t)P * max_rows),
               o_rn = part(nullptr, 4 * (size_t)P), o_st = part(nullptr, 4 * (size_t)P), o_stp = part(nullptr, 8 * (size_t)P),
               o_w = part(nullptr, 8 * (size_t)P * D);
  if (total > b->arena_bytes) {
    if (b->arena) CU(cudaFreeAsync(b->arena, b->stream));
    b->arena = nullptr;
    CU(dalloc(&b->arena, total, b->stream));
    b->arena_bytes = total;
  }
  char* A = static_cast<char*>(b->arena);
  {  // the inputs as one pinned-free staging copy
    std::vector<char> stage(in_bytes);
    for (const Part& q : parts)
      if (q.src && q.off < in_bytes) std::memcpy(stage.data() + q.off, q.src, q.bytes);
    CU(copy_sync(A, stage.data(), in_bytes, cudaMemcpyHostToDevice, b->stream));
  }
  BatchParams bp{};
  bp.X = b->X;
  bp.ld = b->ld;
  bp.d = D;
  bp.dtype = b->dtype;
  bp.n = b->n;
  bp.nprob = P;
  bp.x_rows_per_prob = b->shared ? 0 : b->n;
  bp.y = b->y;
  bp.l2 = b->l2;
  bp.alpha = (const double*)(A + o_alpha);
  bp.mu = (const double*)(A + o_mu);
  bp.delta_min = (const double*)(A + o_dmin);
  bp.div_limit = (const double*)(A + o_divl);
  bp.metric_every = (const double*)(A + o_mev);
  bp.bits = (const int*)(A + o_bits);
  bp.epochs = (const int*)(A + o_ep);
  bp.option = (const int*)(A + o_opt);
  bp.T = (const int64_t*)(A + o_T);
  bp.seed = (const uint64_t*)(A + o_seed);
  bp.init = any_init ? (const double*)(A + o_init) : nullptr;
  bp.pow_tab = b->pow_tab;
  bp.jump_tab = b->jump_tab;
  bp.splits = b->splits;
  bp.max_rows = max_rows;
  bp.rows = (double*)(A + o_rows);
  bp.rhash = (uint64_t*)(A + o_rh);
  bp.rows_n = (int*)(A + o_rn);
  bp.status = (int*)(A + o_st);
  bp.steps = (int64_t*)(A + o_stp);
  bp.w_out = (double*)(A + o_w);
  CU(cudaEventRecord(b->e0, b->stream));
  CU(launch_batch(bp, 128, b->stream));
  CU(cudaEventRecord(b->e1, b->stream));
  std::vector<double> rows(5 * (size_t)P * max_rows), wout((size_t)P * D);
  std::vector<uint64_t> rh((size_t)P * max_rows);
  std::vector<int> rn(P), st(P);
  std::vector<int64_t> stp(P);
  {  // the outputs: one copy of the arena's output region
    std::vector<char> res(total - in_bytes);
    CU(copy_sync(res.data(), A + in_bytes, res.size(), cudaMemcpyDeviceToHost, b->stream));
    auto R = [&](size_t off) { return res.data() + (off - in_bytes); };
    std::memcpy(rows.data(), R(o_rows), rows.size() * 8);
    std::memcpy(rh.data(), R(o_rh), rh.size() * 8);
    std::memcpy(rn.data(), R(o_rn), 4 * (size_t)P);
    std::memcpy(st.data(), R(o_st), 4 * (size_t)P);
    std::memcpy(stp.data(), R(o_stp), 8 * (size_t)P);
    std::memcpy(wout.data(), R(o_w), wout.size() * 8);
  }
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, b->e0, b->e1));
  if (device_ms) *device_ms = ms;
  int invalid = -1;
  for (int q = 0; q < P; ++q) {
    halp_record& r = recs[q];
    r.rows_n = std::min(rn[q], r.rows_cap);
    for (int k = 0; k < r.rows_n; ++k) {
      const double* src = &rows[((size_t)q * max_rows + k) * 5];
      r.rows[k] = halp_row{src[0], src[1], src[2], src[3], src[4], rh[(size_t)q * max_rows + k]};
    }
    r.status = st[q] == 1 ? HALP_STATUS_CONVERGED : st[q] >= 2 ? HALP_STATUS_DIVERGED : HALP_STATUS_OK;
    r.steps_taken = stp[q];
    r.inner_fp_vector_ops = 0;
    r.inner_lp_vector_ops = 0;
    if (st[q] <= 1) {
      const int64_t ep = T[q] > 0 ? stp[q] / T[q] : 0;
      r.inner_fp_vector_ops = (uint64_t)(8 * T[q] * ep);
    }
    if (r.final_iterate) std::memcpy(r.final_iterate, &wout[(size_t)q * D], sizeof(double) * D);
    if (st[q] == 3 && invalid < 0) invalid = q;
  }
  if (invalid >= 0)
    return fail(HALP_INVALID_INPUT, "problem " + std::to_string(invalid) + ": LPRepr: delta must be positive and finite");
  return HALP_OK;
}
