// halp_datasets.cpp -- the reference's own synthetic dataset generators, on the
// host (CPU-callable, no GPU): the harness builds its datasets with them
// (harness.cpp:70-93 build_dataset) before handing them to the device solver.
//
//   make_regression      objectives.cpp:27-45  (fill_gaussian_rowwise :17-23)
//   make_classification  objectives.cpp:46-76
//   QuantRng::next_normal stream for make_conditioned_regression
//                        (objectives.cpp:79-108; the QR factorisations are done
//                        by the Python harness with LAPACK)
//
// Draw order and arithmetic follow the reference: QuantRng (rng.hpp:27-64,
// xorshift64* seeded by splitmix), Box-Muller with std::log1p / std::cos, one
// variate per two uniforms; targets = X w_true as a sequential dot per row.
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/halp.h"
#include "rng_jump.hpp"

namespace {

struct QuantRng {  // rng.hpp:27-64
  uint64_t s;
  QuantRng(uint64_t seed, uint64_t stream) : s(halp::rng_seed_state(seed, stream)) {}
  uint64_t next_u64() {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    return s * 0x2545F4914F6CDD1DULL;
  }
  double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_normal() {
    const double u1 = next_uniform();
    const double u2 = next_uniform();
    const double r = std::sqrt(-2.0 * std::log1p(-u1));
    return r * std::cos(2.0 * 3.141592653589793 * u2);
  }
};

}  // namespace

extern "C" int halp_make_regression(int64_t n, int32_t d, double noise_sd, uint64_t seed, double* X, double* y) {
  if (n < 1 || d < 1 || !X || !y) return HALP_INVALID_INPUT;
  if (!(std::isfinite(noise_sd) && noise_sd >= 0.0)) return HALP_INVALID_INPUT;
  QuantRng rng(seed, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < d; ++j) X[i * d + j] = rng.next_normal();
  std::vector<double> w(d);
  for (int j = 0; j < d; ++j) w[j] = rng.next_normal();
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc += X[i * d + j] * w[j];
    y[i] = acc;
  }
  if (noise_sd > 0.0)
    for (int64_t i = 0; i < n; ++i) y[i] += noise_sd * rng.next_normal();
  return HALP_OK;
}

extern "C" int halp_make_classification(int64_t n, int32_t d, int32_t num_classes, double separation, uint64_t seed,
                                        double* X, int32_t* labels) {
  if (n < 1 || d < 1 || num_classes < 2 || !X || !labels) return HALP_INVALID_INPUT;
  if (!(std::isfinite(separation) && separation >= 0.0)) return HALP_INVALID_INPUT;
  QuantRng rng(seed, 0);
  const double center_sd = separation / std::sqrt(2.0 * d);
  std::vector<double> centers((size_t)num_classes * d);
  for (int c = 0; c < num_classes; ++c)
    for (int j = 0; j < d; ++j) centers[(size_t)c * d + j] = rng.next_normal();
  for (double& v : centers) v *= center_sd;
  for (int64_t i = 0; i < n; ++i) {
    const int c = static_cast<int>(i % num_classes);
    labels[i] = c;
    for (int j = 0; j < d; ++j) X[i * d + j] = centers[(size_t)c * d + j] + rng.next_normal();
  }
  return HALP_OK;
}

extern "C" int halp_normals(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  if (count < 0 || (count > 0 && !out)) return HALP_INVALID_INPUT;
  QuantRng rng(seed, stream);
  for (int64_t k = 0; k < count; ++k) out[k] = rng.next_normal();
  return HALP_OK;
}

// fixed_point.cpp:30-50 quantize_code (host copy for the dataset quantizer)
static int64_t q_code(double x, double delta, int bits, double u) {
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

// objectives.cpp:110-133 quantize_dataset: LPRepr(data_scale(X, bits), bits)
// with data_scale = max|X| / (2^(bits-1) - 1) (1 for an all-zero X), one
// stochastic rounding per element from QuantRng(seed, 2) in row order
extern "C" int halp_quantize_dataset(const double* X, int64_t n, int32_t d, int32_t bits, uint64_t seed,
                                     int64_t* codes, double* delta) {
  if (!X || !codes || !delta || n < 0 || d < 0) return HALP_INVALID_INPUT;
  if (bits < 2 || bits > 64) return HALP_INVALID_INPUT;
  double max_abs = 0.0;
  for (int64_t k = 0; k < n * (int64_t)d; ++k) {
    const double a = std::fabs(X[k]);
    if (!(a <= max_abs)) max_abs = a;
  }
  if (!std::isfinite(max_abs)) return HALP_INVALID_INPUT;
  const double span = std::ldexp(1.0, bits - 1) - 1.0;
  const double dl = max_abs == 0.0 ? 1.0 : max_abs / span;
  QuantRng rng(seed, 2);
  for (int64_t k = 0; k < n * (int64_t)d; ++k) codes[k] = q_code(X[k], dl, bits, rng.next_uniform());
  *delta = dl;
  return HALP_OK;
}
