// qtree/pricer/swing.hpp -- DROP-IN replacement of the reference's swing
// pricer (/root/reference/proj/include/qtree/pricer/swing.hpp) on the device
// kernels k_swing_cont / k_swing_decide (csrc/qt_bdp.cu, K5).
//
//   SwingProblem / SwingResult   swing.hpp:14-39
//   solve_swing                  swing.hpp:47-129 -> qt_bdp_swing
//
// Window rules, tie preference (take on >=) and the absorbing treatment of
// unvisited rows are the reference's; the payoff is tabulated on the host for
// the decision layers 0..n-1 (the reference never evaluates it at layer n).
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "qtree/cuda/capi.hpp"
#include "qtree/pricer/bdp.hpp"

namespace qtree::pricer {

struct SwingProblem {
  const tree::QuantTree* tree = nullptr;
  NodePayoff payoff;  // v_k
  int q_min = 0;
  int q_max = 0;
};

struct SwingResult {
  int q_min = 0, q_max = 0;
  std::vector<int> m_lo;                        // per layer 0..n
  std::vector<int> m_count;                     // per layer 0..n
  std::vector<std::vector<double>> value;       // [k][(m - m_lo) * N_k + i]
  std::vector<std::vector<std::uint8_t>> take;  // decisions, layers 0..n-1
  double price = 0.0;

  double value_at(int k, int m, std::size_t i, std::size_t nodes) const {
    return value[static_cast<std::size_t>(k)]
                [static_cast<std::size_t>(m - m_lo[static_cast<std::size_t>(k)]) * nodes + i];
  }
  bool take_at(int k, int m, std::size_t i, std::size_t nodes) const {
    return take[static_cast<std::size_t>(k)]
               [static_cast<std::size_t>(m - m_lo[static_cast<std::size_t>(k)]) * nodes + i] != 0;
  }
};

inline SwingResult solve_swing(const SwingProblem& problem) {
  if (!problem.tree || !problem.payoff) throw std::invalid_argument("solve_swing: incomplete problem");
  const tree::QuantTree& t = *problem.tree;
  const int n = t.layers();
  const int qmin = problem.q_min, qmax = problem.q_max;
  // swing.hpp:52-54 (checked again by the device entry with the same codes)
  if (qmin < 0 || qmin > qmax) throw ConfigError("swing: need 0 <= q_min <= q_max");
  if (qmax > n) throw ConfigError("swing: q_max exceeds the number of exercise dates");
  if (qmin > n) throw ConfigError("swing: q_min infeasible at the root");

  SwingResult res;
  res.q_min = qmin;
  res.q_max = qmax;
  res.m_lo.resize(static_cast<std::size_t>(n) + 1);
  res.m_count.resize(static_cast<std::size_t>(n) + 1);
  std::size_t total = 0, decisions = 0;
  for (int k = 0; k <= n; ++k) {
    const int lo = std::max(0, qmin - (n - k));
    const int hi = std::min(k, qmax);
    res.m_lo[static_cast<std::size_t>(k)] = lo;
    res.m_count[static_cast<std::size_t>(k)] = hi - lo + 1;
    const std::size_t s = static_cast<std::size_t>(hi - lo + 1) * t.layer_size(k);
    total += s;
    if (k < n) decisions += s;
  }
  const std::vector<double> phi = detail::tabulate(t, problem.payoff, n);
  std::vector<std::uint64_t> sizes, visits;
  std::vector<double> pi;
  cuda::flatten(t, sizes, visits, pi);
  std::vector<double> value(total);
  std::vector<std::uint8_t> take(decisions ? decisions : 1);
  cuda::check(qt_bdp_swing(n, sizes.data(), visits.data(), pi.data(), phi.data(), qmin, qmax,
                           &res.price, value.data(), take.data()),
              "solve_swing");
  res.value.resize(static_cast<std::size_t>(n) + 1);
  res.take.resize(static_cast<std::size_t>(n));
  std::size_t o = 0;
  for (int k = 0; k <= n; ++k) {
    const std::size_t s =
        static_cast<std::size_t>(res.m_count[static_cast<std::size_t>(k)]) * t.layer_size(k);
    res.value[static_cast<std::size_t>(k)].assign(value.begin() + o, value.begin() + o + s);
    if (k < n) res.take[static_cast<std::size_t>(k)].assign(take.begin() + o, take.begin() + o + s);
    o += s;
  }
  return res;
}

}  // namespace qtree::pricer
