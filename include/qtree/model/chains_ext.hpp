// qtree/model/chains_ext.hpp -- the two chains BASELINE.json's configs need
// but the reference does not ship. Both satisfy the
// reference's MarkovChain concept (chains.hpp:17-26), so the reference's own
// estimate_alg* templates run them unchanged (that is how the oracle checks
// them, oracle/ref_harness.cpp), and the drop-in estimator maps them onto the
// device kinds QT_CHAIN_OU_1D / QT_CHAIN_GBM_3D.
#pragma once

#include <cmath>
#include <span>
#include <vector>

#include "qtree/errors.hpp"
#include "qtree/model/chains.hpp"
#include "qtree/model/two_factor.hpp"

namespace qtree::model {

/// Config 3: 1-D Ornstein-Uhlenbeck chain, defined as factor 1 of
/// TwoFactorChain so that its arithmetic is the reference's: step
/// a1 x + l11 eps (chains.hpp:51) with the exact AR(1) coefficients of
/// Ar1Spec::from_params (two_factor.hpp:90-101); marginal sd = l11 of
/// cholesky2(marginal_cov(k)) (chains.hpp:32-36,55-59).
class OuChain1d {
 public:
  explicit OuChain1d(const TwoFactorParams& p) : spec_(ar1_coefficients(p)) {
    marg_.reserve(static_cast<std::size_t>(spec_.steps()) + 1);
    for (int k = 0; k <= spec_.steps(); ++k) marg_.push_back(cholesky2(spec_.marginal_cov(k)).l11);
  }

  const Ar1Spec& spec() const { return spec_; }
  int dim() const { return 1; }
  int layers() const { return spec_.steps(); }
  int normals_per_step() const { return 1; }
  double marginal_sd(int k) const { return marg_[static_cast<std::size_t>(k)]; }

  void initial(std::span<double> out) const { out[0] = 0.0; }
  void step(int k, std::span<const double> x, std::span<double> out,
            std::span<const double> eps) const {
    const Ar1Step& op = spec_.step_op(k);
    out[0] = op.a1 * x[0] + op.chol.l11 * eps[0];
  }
  void sample_marginal(int k, std::span<double> out, std::span<const double> eps) const {
    out[0] = marg_[static_cast<std::size_t>(k)] * eps[0];
  }

 private:
  Ar1Spec spec_;
  std::vector<double> marg_;
};

/// Lower-triangular 3x3 factor.
struct Lower3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
};

/// Cholesky factor of the correlation matrix with off-diagonals
/// (rho12, rho13, rho23).
inline Lower3 corr_chol3(const double rho[3]) {
  Lower3 l;
  l.m[0][0] = 1.0;
  l.m[1][0] = rho[0];
  const double r11 = 1.0 - l.m[1][0] * l.m[1][0];
  if (!(r11 > 0.0)) throw NumericError("GbmChain3d: correlation matrix not positive definite");
  l.m[1][1] = std::sqrt(r11);
  l.m[2][0] = rho[1];
  l.m[2][1] = (rho[2] - l.m[2][0] * l.m[1][0]) / l.m[1][1];
  const double r22 = 1.0 - l.m[2][0] * l.m[2][0] - l.m[2][1] * l.m[2][1];
  if (!(r22 > 0.0)) throw NumericError("GbmChain3d: correlation matrix not positive definite");
  l.m[2][2] = std::sqrt(r22);
  return l;
}

inline Lower3 scaled(const Lower3& l, double s) {
  Lower3 o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c <= r; ++c) o.m[r][c] = s * l.m[r][c];
  return o;
}

/// Config 5: 3-D correlated Brownian log-state of a GBM basket,
/// X_{k+1} = X_k + sqrt(dt) L eps, marginal X_k = sqrt(t_k) L eps, with the
/// products and sums in the order written below (the device evaluates the
/// same order, csrc/qt_device.cuh Chain<3>).
class GbmChain3d {
 public:
  GbmChain3d(int steps, double horizon, const double rho[3]) : steps_(steps), horizon_(horizon) {
    if (steps < 1) throw NumericError("GbmChain3d: need at least one step");
    if (!(horizon > 0.0)) throw NumericError("GbmChain3d: horizon must be > 0");
    const Lower3 l = corr_chol3(rho);
    const double dt = horizon_ / steps_;
    step_ = scaled(l, std::sqrt(dt));
    marg_.reserve(static_cast<std::size_t>(steps_) + 1);
    for (int k = 0; k <= steps_; ++k) marg_.push_back(scaled(l, std::sqrt(k * dt)));
  }

  int dim() const { return 3; }
  int layers() const { return steps_; }
  int normals_per_step() const { return 3; }
  double dt() const { return horizon_ / steps_; }
  double time(int k) const { return k * dt(); }
  const Lower3& step_factor() const { return step_; }
  const Lower3& marginal(int k) const { return marg_[static_cast<std::size_t>(k)]; }

  void initial(std::span<double> out) const { out[0] = out[1] = out[2] = 0.0; }
  void step(int, std::span<const double> x, std::span<double> out,
            std::span<const double> e) const {
    const auto& c = step_.m;
    out[0] = x[0] + c[0][0] * e[0];
    out[1] = x[1] + (c[1][0] * e[0] + c[1][1] * e[1]);
    out[2] = x[2] + ((c[2][0] * e[0] + c[2][1] * e[1]) + c[2][2] * e[2]);
  }
  void sample_marginal(int k, std::span<double> out, std::span<const double> e) const {
    const auto& c = marg_[static_cast<std::size_t>(k)].m;
    out[0] = c[0][0] * e[0];
    out[1] = c[1][0] * e[0] + c[1][1] * e[1];
    out[2] = (c[2][0] * e[0] + c[2][1] * e[1]) + c[2][2] * e[2];
  }

 private:
  int steps_;
  double horizon_;
  Lower3 step_;
  std::vector<Lower3> marg_;
};

static_assert(MarkovChain<OuChain1d>);
static_assert(MarkovChain<GbmChain3d>);

}  // namespace qtree::model
