// anisoq drop-in (B200): per-point loss coefficients and the eta proxy
// (reference geometry.hpp:119-145, 395-402). Host-side scalars; the data-parallel
// loss evaluation runs inside the device kernels.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <limits>
#include <span>
#include <utility>
#include <vector>

#include "error.hpp"

namespace anisoq {

// Score weight w(t) of the inner product (reference geometry.hpp:47-112):
// w = 1 (constant, the reconstruction loss), w = 1[t >= T] (indicator), or a
// non-decreasing staircase over strictly increasing knots (step). Host-side
// value type: the quadrature / Monte-Carlo theory built on it
// (geometry.hpp:202-467) is outside the device hot path; the
// type is here so that code written against the reference API (e.g. its test
// support, tests/support/oracles.hpp:212) compiles unchanged.
class WeightFunction {
 public:
  enum class Kind { constant, indicator, tabulated };

  static WeightFunction constant() { return WeightFunction(Kind::constant, {}, {}); }
  static WeightFunction indicator(double threshold) {
    if (!(threshold >= 0.0)) throw InvalidThreshold("indicator threshold must be >= 0");
    return WeightFunction(Kind::indicator, {threshold}, {1.0});
  }
  static WeightFunction step(std::vector<double> knots, std::vector<double> values) {
    if (knots.empty() || knots.size() != values.size())
      throw InvalidArgument("step weight needs matching non-empty knots/values");
    for (std::size_t i = 0; i < knots.size(); ++i) {
      if (!(knots[i] >= 0.0)) throw InvalidThreshold("step knots must be >= 0");
      if (!(values[i] >= 0.0)) throw InvalidArgument("step values must be >= 0");
      if (i > 0 && !(knots[i] > knots[i - 1]))
        throw InvalidArgument("step knots must be strictly increasing");
      if (i > 0 && values[i] < values[i - 1])
        throw InvalidArgument("step values must be non-decreasing");
    }
    return WeightFunction(Kind::tabulated, std::move(knots), std::move(values));
  }

  Kind kind() const { return kind_; }
  double threshold() const { return knots_.empty() ? 0.0 : knots_.front(); }
  const std::vector<double>& knots() const { return knots_; }
  const std::vector<double>& values() const { return values_; }

  // value of the last knot at or below t; 0 below the first knot
  double operator()(double t) const {
    if (kind_ == Kind::constant) return 1.0;
    if (t < knots_.front()) return 0.0;
    if (!(t >= knots_.front())) return values_.front();  // NaN
    const auto it = std::upper_bound(knots_.begin(), knots_.end(), t);
    return it == knots_.begin() ? 0.0 : values_[static_cast<std::size_t>(it - knots_.begin()) - 1];
  }

 private:
  WeightFunction(Kind kind, std::vector<double> knots, std::vector<double> values)
      : kind_(kind), knots_(std::move(knots)), values_(std::move(values)) {}
  Kind kind_;
  std::vector<double> knots_;
  std::vector<double> values_;
};

struct AnisotropicWeights {
  double h_parallel = 1.0;
  double h_perpendicular = 1.0;
  double eta = 1.0;

  bool is_isotropic() const { return h_parallel == h_perpendicular; }

  static AnisotropicWeights from_h(double h_parallel, double h_perpendicular) {
    if (!(h_parallel >= 0.0) || !(h_perpendicular >= 0.0) || !std::isfinite(h_parallel) ||
        !std::isfinite(h_perpendicular))
      throw InvalidArgument("h coefficients must be finite and >= 0");
    AnisotropicWeights w;
    w.h_parallel = h_parallel;
    w.h_perpendicular = h_perpendicular;
    w.eta = h_perpendicular > 0.0 ? h_parallel / h_perpendicular
                                  : std::numeric_limits<double>::infinity();
    return w;
  }
  static AnisotropicWeights from_eta(double eta) {
    if (!(eta >= 0.0)) throw InvalidArgument("eta must be >= 0");
    return from_h(eta, 1.0);
  }
  static AnisotropicWeights isotropic(double h = 1.0) { return from_h(h, h); }
};

// Large-d proxy (d-1) (T/|x|)^2 / (1 - (T/|x|)^2).
inline double eta_limit(double threshold, double norm, int d) {
  if (!(norm > 0.0)) throw InvalidArgument("norm must be positive");
  if (!(threshold >= 0.0) || threshold >= norm) throw InvalidThreshold("need 0 <= T < norm");
  if (d < 2) throw InvalidArgument("eta_limit needs d >= 2");
  const double rho = (threshold / norm) * (threshold / norm);
  return static_cast<double>(d - 1) * rho / (1.0 - rho);
}

namespace detail {
// geometry.hpp:170-176: inner product / squared norm in ascending component
// order (the host side of evaluate's relative error)
inline double dot(std::span<const double> a, std::span<const double> b) {
  double s = 0.0;
  for (std::size_t j = 0; j < a.size(); ++j) s += a[j] * b[j];
  return s;
}
inline double norm2(std::span<const double> a) { return dot(a, a); }

// geometry.hpp:182-200: the two scalars of a residual r = x - c (|r|^2 and
// <r, x>, ascending components) and the score-aware loss built from them —
// the float64 definitions the device kernels reproduce bit for bit.
inline void residual_terms(std::span<const double> x, std::span<const double> c, double& dist2,
                           double& rdot) {
  dist2 = 0.0;
  rdot = 0.0;
  for (std::size_t j = 0; j < x.size(); ++j) {
    const double r = x[j] - c[j];
    dist2 += r * r;
    rdot += r * x[j];
  }
}
inline double combined_loss(double dist2, double rdot, const AnisotropicWeights& w,
                            double inv_norm2) {
  return w.h_perpendicular * dist2 +
         (w.h_parallel - w.h_perpendicular) * (rdot * rdot) * inv_norm2;
}
}  // namespace detail

// geometry.hpp:404-415: the score-aware loss of one datapoint x against its
// quantization x_quant, h_par |r_par|^2 + h_perp |r_perp|^2 in the fused form
// the device kernels evaluate (residual_terms + combined_loss, clamped at 0).
// A single-point scalar helper, like adc_score; the batched losses of the hot
// path (pq_point_loss, pq.hpp:137-146) are computed on the device.
inline double anisotropic_loss(std::span<const double> x, std::span<const double> x_quant,
                               const AnisotropicWeights& w) {
  if (x.size() != x_quant.size())
    throw DimensionMismatch("datapoint and quantization dimensions differ");
  const double n2 = detail::norm2(x);
  if (n2 == 0.0) throw ZeroNormDatapoint("loss undefined at |x| = 0");
  double dist2 = 0.0, rdot = 0.0;
  detail::residual_terms(x, x_quant, dist2, rdot);
  return std::max(0.0, detail::combined_loss(dist2, rdot, w, 1.0 / n2));
}

}  // namespace anisoq
