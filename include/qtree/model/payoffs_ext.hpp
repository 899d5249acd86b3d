// qtree/model/payoffs_ext.hpp -- the obstacles of the two BASELINE configs the
// reference has no factory for, as NodePayoffs
// (pricer/bdp.hpp:17) next to the reference's make_put/call/swing_payoff
// (pipeline.hpp:120-170), for C++ callers of the drop-in pricers.
//
//   config 3: make_ou_swing_payoff -- v_k = e^{-rt} (spot(p, t, x, 0) - K) with
//             sigma2 = 0, on the OuChain1d state (two_factor.hpp:144-152,172-176);
//   config 5: make_max_call_payoff -- e^{-rt} max(max_a S_a - K, 0),
//             S_a = s0 exp((r - sigma_a^2/2) t + sigma_a x_a), on the GbmChain3d state.
//
// The same expressions, in the same order, are tabulated by the C ABI's
// qt_payoff_table (QT_PAYOFF_SWING on QT_CHAIN_OU_1D, QT_PAYOFF_MAX_CALL), so
// a tree priced from C++ or from Python sees bit-identical obstacles.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <span>

#include "qtree/model/two_factor.hpp"
#include "qtree/pricer/bdp.hpp"

namespace qtree::model {

inline pricer::NodePayoff make_ou_swing_payoff(const TwoFactorParams& params) {
  TwoFactorParams p = params;
  p.sigma2 = 0.0;
  const double dt = p.horizon / p.steps;
  return [p, dt](int k, std::span<const double> x) {
    const double t = k * dt;
    return std::exp(-p.r * t) * (spot(p, t, x[0], 0.0) - p.strike);
  };
}

inline pricer::NodePayoff make_max_call_payoff(const TwoFactorParams& p,
                                               std::array<double, 3> sigma = {0.2, 0.2, 0.2}) {
  const double dt = p.horizon / p.steps;
  return [p, dt, sigma](int k, std::span<const double> x) {
    const double t = k * dt;
    double best = -std::numeric_limits<double>::infinity();
    for (int a = 0; a < 3; ++a) {
      const double s = p.s0 * std::exp((p.r - 0.5 * sigma[a] * sigma[a]) * t + sigma[a] * x[a]);
      best = std::max(best, s);
    }
    return std::exp(-p.r * t) * std::max(best - p.strike, 0.0);
  };
}

}  // namespace qtree::model
