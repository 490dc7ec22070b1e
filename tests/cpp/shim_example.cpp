// C++ caller of the drop-in header (include/halp_lpopt.hpp): reads a problem
// written by tests/test_cpp_shim.py, runs run_halp, prints the rows.  Mirrors
// the reference's own usage (proj/tests/test_optimizers.cpp style).
#include <cstdio>
#include <fstream>
#include <vector>

#include "halp_lpopt.hpp"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  std::ifstream in(argv[1], std::ios::binary);
  long n;
  int d;
  in.read(reinterpret_cast<char*>(&n), sizeof n);
  in.read(reinterpret_cast<char*>(&d), sizeof d);
  lpopt_b200::Dataset ds;
  ds.n = n;
  ds.d = d;
  ds.X.resize((size_t)n * d);
  ds.targets.resize(n);
  in.read(reinterpret_cast<char*>(ds.X.data()), sizeof(double) * ds.X.size());
  in.read(reinterpret_cast<char*>(ds.targets.data()), sizeof(double) * n);
  try {
    lpopt_b200::Objective obj(std::move(ds), lpopt_b200::LossFamily::Squared, 0.0);
    lpopt_b200::OptimizerConfig cfg;
    cfg.algorithm = lpopt_b200::Algorithm::Halp;
    cfg.alpha = 5e-3;
    cfg.epochs = 4;
    cfg.inner_steps = 2000;
    cfg.bits = 8;
    cfg.mu = 3.0;
    cfg.seed = 1;
    const auto rec = lpopt_b200::run(obj, cfg);
    for (const auto& r : rec.rows)
      std::printf("%.17g %.17g %.17g %.17g %llu\n", r.pass, r.loss, r.grad_norm, r.delta,
                  (unsigned long long)r.iterate_hash);
    // LM-HALP through run_prepared: the dataset is quantized on the fly
    lpopt_b200::OptimizerConfig lm = cfg;
    lm.algorithm = lpopt_b200::Algorithm::LmHalp;
    lm.epochs = 2;
    const auto lrec = lpopt_b200::run_prepared(obj, lm, 7);
    if (lrec.rows.size() != 3 || !(lrec.rows.back().loss < lrec.rows.front().loss) || !(lrec.rows[0].delta_aux > 0.0))
      return 4;
    std::printf("lm %.17g %.17g %.17g\n", lrec.rows.back().loss, lrec.rows.back().delta_inner,
                lrec.rows.back().delta_aux);
    // the reference's error behaviour: invalid configs throw InvalidInputError
    cfg.mu = 0.0;
    try {
      lpopt_b200::run(obj, cfg);
      return 3;
    } catch (const lpopt_b200::InvalidInputError&) {
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
