// qtree/pricer/bdp.hpp -- DROP-IN replacement of the reference's optimal
// stopping pricer (/root/reference/proj/include/qtree/pricer/bdp.hpp) on the
// device backward-DP kernels of libqtree_cuda.so (csrc/qt_bdp.cu, K5).
//
//   NodePayoff                         bdp.hpp:17
//   StoppingProblem / StoppingResult   bdp.hpp:20-31
//   cond_expectation                   bdp.hpp:36-54  -> qt_bdp_cond_expectation
//   solve_stopping                     bdp.hpp:58-96  -> qt_bdp_stopping
//
// The payoff is a host std::function, so it is tabulated on the host into
// phi[k][i] (one call per node, as the reference makes) and handed to the
// device with the tree. Results are bit-identical to the reference: each
// conditional expectation is a sequential j-ascending sum over the row's
// non-zeros.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <span>
#include <stdexcept>
#include <vector>

#include "qtree/cuda/capi.hpp"
#include "qtree/tree/quant_tree.hpp"

namespace qtree::pricer {

/// Node payoff: layer index and the node's coordinates (bdp.hpp:17).
using NodePayoff = std::function<double(int layer, std::span<const double> node)>;

struct StoppingProblem {
  const tree::QuantTree* tree = nullptr;
  NodePayoff payoff;
};

struct StoppingResult {
  std::vector<std::vector<double>> value;
  std::vector<std::vector<std::uint8_t>> exercise;
  double price = 0.0;
};

/// E(f(X_{k+1}) | X_k = x_i) = pi^{k+1} f; quiet NaN on unvisited rows.
inline std::vector<double> cond_expectation(const tree::QuantTree& t, int k,
                                            std::span<const double> f) {
  if (k < 0 || k >= t.layers()) throw std::invalid_argument("cond_expectation: layer out of range");
  const std::size_t rows = t.layer_size(k);
  const std::size_t cols = t.layer_size(k + 1);
  if (f.size() != cols) throw std::invalid_argument("cond_expectation: value vector length mismatch");
  std::vector<double> out(rows);
  cuda::check(qt_bdp_cond_expectation(rows, cols, t.counts.visits[static_cast<std::size_t>(k)].data(),
                                      t.pi[static_cast<std::size_t>(k)].data(), f.data(), out.data()),
              "cond_expectation");
  return out;
}

namespace detail {

/// phi laid out like the flat visits array, layers [0, layers_to) (the rest 0).
inline std::vector<double> tabulate(const tree::QuantTree& t, const NodePayoff& payoff,
                                    int layers_to) {
  std::vector<double> phi;
  for (int k = 0; k <= t.layers(); ++k) {
    const quant::QuantGrid& g = t.grids[static_cast<std::size_t>(k)];
    for (std::size_t i = 0; i < g.size(); ++i)
      phi.push_back(k < layers_to ? payoff(k, g.point(i)) : 0.0);
  }
  return phi;
}

}  // namespace detail

/// V_n = phi_n; V_k = max(phi_k, E(V_{k+1} | node)), unvisited nodes absorb
/// at their payoff; exercise = phi >= continuation (terminal: phi > 0).
inline StoppingResult solve_stopping(const StoppingProblem& problem) {
  if (!problem.tree || !problem.payoff) throw std::invalid_argument("solve_stopping: incomplete problem");
  const tree::QuantTree& t = *problem.tree;
  const int n = t.layers();
  const std::vector<double> phi = detail::tabulate(t, problem.payoff, n + 1);
  std::vector<std::uint64_t> sizes, visits;
  std::vector<double> pi;
  cuda::flatten(t, sizes, visits, pi);
  std::vector<double> value(phi.size());
  std::vector<std::uint8_t> exercise(phi.size());
  StoppingResult res;
  cuda::check(qt_bdp_stopping(n, sizes.data(), visits.data(), pi.data(), phi.data(), value.data(),
                              exercise.data(), &res.price),
              "solve_stopping");
  res.value.resize(static_cast<std::size_t>(n) + 1);
  res.exercise.resize(static_cast<std::size_t>(n) + 1);
  std::size_t o = 0;
  for (int k = 0; k <= n; ++k) {
    const std::size_t s = sizes[static_cast<std::size_t>(k)];
    res.value[static_cast<std::size_t>(k)].assign(value.begin() + o, value.begin() + o + s);
    res.exercise[static_cast<std::size_t>(k)].assign(exercise.begin() + o, exercise.begin() + o + s);
    o += s;
  }
  return res;
}

}  // namespace qtree::pricer
