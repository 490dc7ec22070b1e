// halp_lpopt.hpp -- header-only C++ mirror of the reference's HALP solver
// interface over the C ABI (halp.h), for C++ callers of lpopt::run_halp.
//
// Same names, fields, defaults and error behaviour as
//   proj/include/lpopt/objectives.hpp:14,23-33,59-91   (LossFamily, Dataset, Objective)
//   proj/include/lpopt/optimizers.hpp:13-91            (Algorithm, EpochOption, OptimizerConfig,
//                                                        MetricRow, RunRecord, DivergenceError,
//                                                        run_halp, run)
//   proj/include/lpopt/errors.hpp:8-36                 (Error, InvalidInputError)
// but Eigen-free: vectors are std::vector<double> (parameter layout d x C
// column-major, like the reference) and X is row-major n x d.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "halp.h"

namespace lpopt_b200 {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidInputError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};
struct UnsupportedError : Error {
  using Error::Error;
};

enum class LossFamily { Squared, Softmax };
enum class Algorithm { Sgd, Svrg, LpSgd, LpSvrg, Halp, LmHalp };
enum class EpochOption { LastIterate, SampledIterate };

// lpopt::QuantizedExamples (objectives.hpp): LM-HALP's integer rows, one scale
struct QuantizedExamples {
  std::vector<std::int64_t> codes;  // row-major n x d
  double delta = 0.0;
  int bits = 0;
  std::uint64_t seed = 0;
};

struct Dataset {
  std::vector<double> X;      // row-major n x d (the reference holds it column-major)
  long n = 0;
  int d = 0;
  std::vector<double> targets;
  std::vector<int> labels;
  int num_classes = 0;
  bool has_quantized = false;  // std::optional<QuantizedExamples> quantized in the reference
  QuantizedExamples quantized;
};

struct MetricRow {
  double pass = 0.0, seconds = 0.0, loss = 0.0, grad_norm = 0.0, delta = 0.0;
  std::uint64_t iterate_hash = 0;
  double delta_inner = 0.0, delta_aux = 0.0;
};

struct RunRecord {
  std::vector<MetricRow> rows;
  std::vector<double> final_iterate;
  std::string status = "ok";
  std::uint64_t inner_fp_vector_ops = 0;
  std::uint64_t inner_lp_vector_ops = 0;
  long steps_taken = 0;
};

struct DivergenceError : Error {
  RunRecord partial;
  DivergenceError(const std::string& msg, RunRecord rec) : Error(msg), partial(std::move(rec)) {}
};

struct OptimizerConfig {
  Algorithm algorithm = Algorithm::Svrg;
  double alpha = 1e-3;
  int epochs = 1;
  long inner_steps = 0;
  int bits = 8;
  double delta = 0.0;
  double mu = 0.0;
  EpochOption option = EpochOption::LastIterate;
  int full_grad_period = 2;
  std::uint64_t seed = 0;
  double metric_every_passes = 0.0;
  double delta_min = 1e-300;
  double divergence_limit = 1e12;
  bool lm_bypass_aux_quant = false;
  std::vector<double> init;
};

namespace detail {
[[noreturn]] inline void raise(int rc) {
  const std::string m = halp_last_error();
  if (rc == HALP_INVALID_INPUT) throw InvalidInputError(m);
  if (rc == HALP_UNSUPPORTED) throw UnsupportedError(m);
  if (rc == HALP_CUDA_ERROR || rc == HALP_NCCL_ERROR) throw CudaError(m);
  throw Error(m);
}
}  // namespace detail

// lpopt::Objective backed by a device problem (one GPU; see halp.h for NCCL sharding).
class Objective {
 public:
  Objective(Dataset ds, LossFamily loss, double l2, int device = 0) : ds_(std::move(ds)), loss_(loss), l2_(l2) {
    halp_problem_desc desc{};
    desc.X = ds_.X.data();
    desc.dtype = HALP_F64;
    desc.mem = HALP_MEM_HOST;
    desc.n = ds_.n;
    desc.d = ds_.d;
    desc.loss = loss == LossFamily::Squared ? HALP_SQUARED : HALP_SOFTMAX;
    desc.num_classes = ds_.num_classes;
    if (loss == LossFamily::Squared) {
      if ((long)ds_.targets.size() != ds_.n) throw InvalidInputError("Objective: squared loss needs one target per row");
      desc.y = ds_.targets.data();
    } else {
      if ((long)ds_.labels.size() != ds_.n || ds_.num_classes < 2)
        throw InvalidInputError("Objective: softmax loss needs labels and classes");
      labels32_.assign(ds_.labels.begin(), ds_.labels.end());
      desc.labels = labels32_.data();
    }
    desc.l2 = l2;
    desc.device = device;
    desc.world_size = 1;
    if (ds_.has_quantized) {
      if ((long)ds_.quantized.codes.size() != ds_.n * (long)ds_.d)
        throw InvalidInputError("lm_halp: quantized rows do not match the dataset shape");
      desc.qcodes = ds_.quantized.codes.data();
      desc.qbits = ds_.quantized.bits;
      desc.qdelta = ds_.quantized.delta;
    }
    const int rc = halp_problem_create(&desc, &h_);
    if (rc) detail::raise(rc);
    outputs_ = loss == LossFamily::Squared ? 1 : ds_.num_classes;
  }
  Objective(const Objective&) = delete;
  Objective& operator=(const Objective&) = delete;
  ~Objective() {
    if (h_) halp_problem_destroy(h_);
  }

  long num_components() const { return ds_.n; }
  int feature_dim() const { return ds_.d; }
  int num_outputs() const { return outputs_; }
  int dim() const { return ds_.d * outputs_; }
  LossFamily loss_family() const { return loss_; }
  double l2() const { return l2_; }
  const Dataset& dataset() const { return ds_; }
  halp_problem* handle() const { return h_; }

  // objectives.cpp:258-311 / :193-223, one fused device pass
  std::vector<double> full_gradient(const std::vector<double>& w, int num_threads = 1) const {
    if (num_threads < 1) throw InvalidInputError("full_gradient: num_threads must be >= 1");
    if ((int)w.size() != dim()) throw InvalidInputError("full_gradient: parameter length mismatch");
    std::vector<double> g(dim());
    double l = 0.0;
    const int rc = halp_full_gradient(h_, w.data(), g.data(), &l);
    if (rc) detail::raise(rc);
    return g;
  }
  double loss(const std::vector<double>& w) const {
    if ((int)w.size() != dim()) throw InvalidInputError("loss: parameter length mismatch");
    std::vector<double> g(dim());
    double l = 0.0;
    const int rc = halp_full_gradient(h_, w.data(), g.data(), &l);
    if (rc) detail::raise(rc);
    return l;
  }

 private:
  Dataset ds_;
  LossFamily loss_;
  double l2_;
  int outputs_ = 1;
  std::vector<int32_t> labels32_;
  halp_problem* h_ = nullptr;
};

namespace detail {
// one of the device algorithms (HALP_ALGO_*) through halp_run
inline RunRecord run_algo(const Objective& obj, const OptimizerConfig& cfg, int algo) {
  if (!cfg.init.empty() && (int)cfg.init.size() != obj.dim())
    throw InvalidInputError("optimizer: init length does not match objective");
  halp_config c{};
  c.algorithm = algo;
  c.delta = cfg.delta;
  c.alpha = cfg.alpha;
  c.epochs = cfg.epochs;
  c.inner_steps = cfg.inner_steps;
  c.bits = cfg.bits;
  c.mu = cfg.mu;
  c.option = cfg.option == EpochOption::SampledIterate ? 1 : 0;
  c.full_grad_period = cfg.full_grad_period;
  c.seed = cfg.seed;
  c.metric_every_passes = cfg.metric_every_passes;
  c.delta_min = cfg.delta_min;
  c.divergence_limit = cfg.divergence_limit;
  c.init = cfg.init.empty() ? nullptr : cfg.init.data();
  const int cap = (cfg.epochs > 0 ? cfg.epochs : 0) + 2;
  std::vector<halp_row> rows(cap);
  RunRecord out;
  out.final_iterate.assign(obj.dim(), 0.0);
  halp_record rec{rows.data(), cap, 0, out.final_iterate.data(), 0, 0, 0, 0};
  const int rc = halp_run(obj.handle(), &c, &rec);
  auto fill = [&]() {
    for (int i = 0; i < rec.rows_n; ++i) {
      MetricRow r;
      r.pass = rows[i].pass;
      r.seconds = rows[i].seconds;
      r.loss = rows[i].loss;
      r.grad_norm = rows[i].grad_norm;
      r.delta = rows[i].delta;
      r.iterate_hash = rows[i].iterate_hash;
      r.delta_inner = rows[i].delta_inner;
      r.delta_aux = rows[i].delta_aux;
      out.rows.push_back(r);
    }
    out.status = rec.status == HALP_STATUS_CONVERGED ? "converged" : rec.status == HALP_STATUS_DIVERGED ? "diverged" : "ok";
    out.steps_taken = rec.steps_taken;
    out.inner_fp_vector_ops = rec.inner_fp_vector_ops;
    out.inner_lp_vector_ops = rec.inner_lp_vector_ops;
  };
  if (rc == HALP_DIVERGED) {
    fill();
    throw DivergenceError(halp_last_error(), std::move(out));
  }
  if (rc) detail::raise(rc);
  fill();
  return out;
}
}  // namespace detail

// lpopt::run_halp (optimizers.cpp:387-459)
inline RunRecord run_halp(const Objective& obj, const OptimizerConfig& cfg) {
  return detail::run_algo(obj, cfg, HALP_ALGO_HALP);
}
// lpopt::run_svrg (optimizers.cpp:258-296)
inline RunRecord run_svrg(const Objective& obj, const OptimizerConfig& cfg) {
  return detail::run_algo(obj, cfg, HALP_ALGO_SVRG);
}
// lpopt::run_lp_svrg (optimizers.cpp:336-385)
inline RunRecord run_lp_svrg(const Objective& obj, const OptimizerConfig& cfg) {
  return detail::run_algo(obj, cfg, HALP_ALGO_LP_SVRG);
}

// lpopt::run_sgd (optimizers.cpp:229-256)
inline RunRecord run_sgd(const Objective& obj, const OptimizerConfig& cfg) {
  return detail::run_algo(obj, cfg, HALP_ALGO_SGD);
}
// lpopt::run_lp_sgd (optimizers.cpp:297-334)
inline RunRecord run_lp_sgd(const Objective& obj, const OptimizerConfig& cfg) {
  return detail::run_algo(obj, cfg, HALP_ALGO_LP_SGD);
}

// lpopt::run_lm_halp (optimizers.cpp:461-627): the integer inner loop over
// obj.dataset().quantized (bits <= 16 and d * classes <= 4096 on the B200)
inline RunRecord run_lm_halp(const Objective& obj, const OptimizerConfig& cfg) {
  if (cfg.lm_bypass_aux_quant) throw UnsupportedError("lm_halp: the bypass test hook is not on the B200 path");
  return detail::run_algo(obj, cfg, HALP_ALGO_LM_HALP);
}

// objectives.cpp:110-133 quantize_dataset: attaches the codes to ds
inline void quantize_dataset(Dataset& ds, int bits, std::uint64_t seed) {
  QuantizedExamples q;
  q.codes.resize((size_t)ds.n * ds.d);
  q.bits = bits;
  q.seed = seed;
  if (halp_quantize_dataset(ds.X.data(), ds.n, ds.d, bits, seed, q.codes.data(), &q.delta))
    throw InvalidInputError("data_scale: bits must be in [2, 64] and the matrix finite");
  ds.quantized = std::move(q);
  ds.has_quantized = true;
}

// lpopt::run (optimizers.cpp:629-639)
inline RunRecord run(const Objective& obj, const OptimizerConfig& cfg) {
  switch (cfg.algorithm) {
    case Algorithm::Halp: return run_halp(obj, cfg);
    case Algorithm::Svrg: return run_svrg(obj, cfg);
    case Algorithm::LpSvrg: return run_lp_svrg(obj, cfg);
    case Algorithm::Sgd: return run_sgd(obj, cfg);
    case Algorithm::LpSgd: return run_lp_sgd(obj, cfg);
    case Algorithm::LmHalp: return run_lm_halp(obj, cfg);
  }
  throw InvalidInputError("unknown algorithm enum value");
}

// harness.cpp:296-312 (LM-HALP on a dataset without codes of the run's width
// quantizes a copy with data_seed first)
inline RunRecord run_prepared(const Objective& obj, const OptimizerConfig& cfg, std::uint64_t data_seed = 0) {
  try {
    if (cfg.algorithm == Algorithm::LmHalp &&
        (!obj.dataset().has_quantized || obj.dataset().quantized.bits != cfg.bits)) {
      Dataset ds = obj.dataset();
      quantize_dataset(ds, cfg.bits, data_seed);
      const Objective prepared(std::move(ds), obj.loss_family(), obj.l2());
      return run(prepared, cfg);
    }
    return run(obj, cfg);
  } catch (const DivergenceError& e) {
    return e.partial;
  }
}

}  // namespace lpopt_b200
