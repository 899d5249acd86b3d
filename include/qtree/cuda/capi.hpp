// qtree/cuda/capi.hpp -- C++ glue between the reference's host types and the
// C ABI of libqtree_cuda.so (include/qtree_cuda.h).
//
// Used by the drop-in headers include/qtree/tree/estimate.hpp,
// include/qtree/pricer/bdp.hpp and include/qtree/pricer/swing.hpp, which shadow
// the reference's headers of the same name when include/ precedes the
// reference's include directory on the compiler's search path.
// Everything here is marshalling: status -> exception mapping, chain
// coefficients taken from the reference's own chain objects (so the FP64
// constants are the reference's bit for bit), grid packing and unpacking of
// the flat count arrays into CountMatrixSet / QuantTree.
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "qtree/errors.hpp"
#include "qtree/model/chains.hpp"
#include "qtree/model/chains_ext.hpp"
#include "qtree/quant/grid.hpp"
#include "qtree/tree/quant_tree.hpp"
#include "qtree_cuda.h"

namespace qtree::cuda {

/// Status code -> the reference's exception taxonomy (errors.hpp:9-21;
/// include/qtree_cuda.h status table). Device failures keep CLI exit code 3.
inline void check(qt_status rc, const char* where) {
  if (rc == QT_OK) return;
  const std::string msg = std::string(where) + ": " + qt_last_error();
  switch (rc) {
    case QT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QT_ERR_CONFIG: throw ConfigError(msg);
    case QT_ERR_IO: throw IoError(msg);
    default: throw NumericError(msg);
  }
}

/// Per-chain device coefficients (qt_chain layout, include/qtree_cuda.h):
/// `step` n rows x 6, `marginal` n+1 rows x 6.
struct ChainCoefficients {
  qt_chain_kind kind{};
  int layers = 0;
  std::vector<double> step, marginal;

  qt_chain view() const { return {kind, layers, step.data(), marginal.data()}; }
};

template <class C>
inline constexpr bool kSupportedChain =
    std::is_same_v<C, model::BrownianChain1d> || std::is_same_v<C, model::TwoFactorChain> ||
    std::is_same_v<C, model::OuChain1d> || std::is_same_v<C, model::GbmChain3d>;

/// Coefficients read from the reference's chain objects with the same
/// expressions their step()/sample_marginal() evaluate (chains.hpp:48-59,
/// 83-90; two_factor.hpp:57-101), so the device multiplies by identical
/// doubles.
template <class C>
ChainCoefficients coefficients(const C& chain) {
  static_assert(kSupportedChain<C>,
                "qtree CUDA estimator: the device path implements BrownianChain1d, "
                "TwoFactorChain, OuChain1d and GbmChain3d (include/qtree_cuda.h qt_chain_kind)");
  ChainCoefficients c;
  const int n = chain.layers();
  c.layers = n;
  c.step.assign(static_cast<std::size_t>(n) * 6, 0.0);
  c.marginal.assign(static_cast<std::size_t>(n + 1) * 6, 0.0);
  auto S = [&](int t, int j) -> double& { return c.step[static_cast<std::size_t>(t) * 6 + j]; };
  auto Mg = [&](int k, int j) -> double& {
    return c.marginal[static_cast<std::size_t>(k) * 6 + j];
  };
  if constexpr (std::is_same_v<C, model::BrownianChain1d>) {
    c.kind = QT_CHAIN_BROWNIAN_1D;
    for (int t = 0; t < n; ++t) S(t, 0) = std::sqrt(chain.dt());       // chains.hpp:85
    for (int k = 0; k <= n; ++k)                                        // chains.hpp:89
      Mg(k, 0) = k == 0 ? 0.0 : std::sqrt(chain.time(k));
  } else if constexpr (std::is_same_v<C, model::TwoFactorChain>) {
    c.kind = QT_CHAIN_TWO_FACTOR;
    const model::Ar1Spec& spec = chain.spec();
    for (int t = 0; t < n; ++t) {
      const model::Ar1Step& op = spec.step_op(t);                        // chains.hpp:50-52
      S(t, 0) = op.a1;
      S(t, 1) = op.a2;
      S(t, 2) = op.chol.l11;
      S(t, 3) = op.chol.l21;
      S(t, 4) = op.chol.l22;
    }
    for (int k = 0; k <= n; ++k) {                                      // chains.hpp:32-36,55-59
      const model::LowerTri2 l = model::cholesky2(spec.marginal_cov(k));
      Mg(k, 0) = l.l11;
      Mg(k, 1) = l.l21;
      Mg(k, 2) = l.l22;
    }
  } else if constexpr (std::is_same_v<C, model::OuChain1d>) {
    c.kind = QT_CHAIN_OU_1D;
    for (int t = 0; t < n; ++t) {
      S(t, 0) = chain.spec().step_op(t).a1;
      S(t, 2) = chain.spec().step_op(t).chol.l11;
    }
    for (int k = 0; k <= n; ++k) Mg(k, 0) = chain.marginal_sd(k);
  } else {
    c.kind = QT_CHAIN_GBM_3D;
    const auto pack = [](const model::Lower3& l, double* o) {
      o[0] = l.m[0][0];
      o[1] = l.m[1][0];
      o[2] = l.m[1][1];
      o[3] = l.m[2][0];
      o[4] = l.m[2][1];
      o[5] = l.m[2][2];
    };
    for (int t = 0; t < n; ++t) pack(chain.step_factor(), &S(t, 0));
    for (int k = 0; k <= n; ++k) pack(chain.marginal(k), &Mg(k, 0));
  }
  return c;
}

/// Grids for layers 1..n packed for qt_grids, with the reference's
/// validation (estimate.hpp:52-64: one grid per layer, matching dimension).
struct PackedGrids {
  int dim = 0;
  std::vector<std::uint64_t> sizes;  // n+1, sizes[0] = 1
  std::vector<double> points;        // layers 1..n

  qt_grids view() const {
    return {dim, static_cast<int32_t>(sizes.size()) - 1, sizes.data(), points.data()};
  }
};

template <class C>
PackedGrids pack_grids(const C& chain, std::span<const quant::QuantGrid> grids) {
  if (static_cast<int>(grids.size()) != chain.layers())
    throw std::invalid_argument("estimate: need one grid per layer 1..n");
  for (const auto& g : grids)
    if (g.dim() != chain.dim()) throw std::invalid_argument("estimate: grid dimension mismatch");
  PackedGrids p;
  p.dim = chain.dim();
  p.sizes.reserve(grids.size() + 1);
  p.sizes.push_back(1);  // layer 0 is the singleton {x_0}
  std::size_t total = 0;
  for (const auto& g : grids) {
    p.sizes.push_back(g.size());
    total += g.data().size();
  }
  p.points.reserve(total);
  for (const auto& g : grids) p.points.insert(p.points.end(), g.data().begin(), g.data().end());
  return p;
}

/// Flat offsets of the visits (layers 0..n) and joint/pi (transitions 1..n)
/// arrays (include/qtree_cuda.h "Array layouts").
inline void flat_sizes(std::span<const std::uint64_t> sizes, std::uint64_t& n_visits,
                       std::uint64_t& n_joint) {
  n_visits = 0;
  n_joint = 0;
  for (std::size_t k = 0; k < sizes.size(); ++k) n_visits += sizes[k];
  for (std::size_t k = 1; k < sizes.size(); ++k) n_joint += sizes[k - 1] * sizes[k];
}

/// Flat arrays -> the reference's nested CountMatrixSet / pi layout.
inline void unflatten(std::span<const std::uint64_t> sizes, const std::vector<std::uint64_t>& visits,
                      const std::vector<std::uint64_t>& joint, const std::vector<double>* pi,
                      tree::CountMatrixSet& cs, std::vector<std::vector<double>>* pi_out) {
  const std::size_t L = sizes.size();
  cs.visits.resize(L);
  cs.joint.resize(L - 1);
  if (pi_out) pi_out->resize(L - 1);
  std::size_t vo = 0, jo = 0;
  for (std::size_t k = 0; k < L; ++k) {
    cs.visits[k].assign(visits.begin() + vo, visits.begin() + vo + sizes[k]);
    vo += sizes[k];
  }
  for (std::size_t t = 0; t + 1 < L; ++t) {
    const std::size_t e = sizes[t] * sizes[t + 1];
    cs.joint[t].assign(joint.begin() + jo, joint.begin() + jo + e);
    if (pi_out) (*pi_out)[t].assign(pi->begin() + jo, pi->begin() + jo + e);
    jo += e;
  }
}

/// QuantTree counts / pi -> flat arrays (for the pricer entry points).
inline void flatten(const tree::QuantTree& t, std::vector<std::uint64_t>& sizes,
                    std::vector<std::uint64_t>& visits, std::vector<double>& pi) {
  const int n = t.layers();
  sizes.resize(static_cast<std::size_t>(n) + 1);
  for (int k = 0; k <= n; ++k) sizes[static_cast<std::size_t>(k)] = t.layer_size(k);
  visits.clear();
  pi.clear();
  for (int k = 0; k <= n; ++k) {
    const auto& v = t.counts.visits[static_cast<std::size_t>(k)];
    visits.insert(visits.end(), v.begin(), v.end());
  }
  for (int k = 0; k < n; ++k) {
    const auto& p = t.pi[static_cast<std::size_t>(k)];
    pi.insert(pi.end(), p.begin(), p.end());
  }
}

}  // namespace qtree::cuda
