// anisoq drop-in (B200): per-point loss coefficients and the eta proxy
// (reference geometry.hpp:119-145, 395-402). Host-side scalars; the data-parallel
// loss evaluation runs inside the device kernels.
#pragma once

#include <cmath>
#include <cstddef>
#include <limits>
#include <span>

#include "error.hpp"

namespace anisoq {

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

}  // namespace anisoq
