// qtree/tree/estimate.hpp -- DROP-IN replacement of the reference's
// estimator header (/root/reference/proj/include/qtree/tree/estimate.hpp),
// backed by libqtree_cuda.so (sm_100a) through the C ABI of qtree_cuda.h.
//
// Put this repository's include/ BEFORE the reference's include directory:
// every `#include "qtree/tree/estimate.hpp"` (pipeline.hpp, the CLI, the
// tests) then resolves here, while the reference keeps supplying the host
// types (QuantGrid, QuantTree, CountMatrixSet, the chains, the RNG enums).
// Names, signatures, defaults and exceptions are the reference's:
//
//   EstimatorKind, BuildPhases, EstimateOptions         estimate.hpp:18-36
//   detail::uniforms_per_path                            estimate.hpp:48-50
//   estimate_alg1 / estimate_alg2 / estimate_alg3        estimate.hpp:133-296
//   estimate                                             estimate.hpp:299-309
//
// Differences, all documented in INTEGRATION.md:
//   * EstimateOptions gains `int devices = 1` (GPUs of this process to shard
//     the paths over; counts are bit-identical for any value).
//   * `workers` is validated exactly as the reference does and otherwise
//     ignored (one launch covers all paths; Alg I already ignores it).
//   * `nn` is accepted; the device projection is the exact brute-force
//     argmin, equal to the kd-tree's answer (nn.hpp:127,138-140).
//   * the chain must be one of the device kinds (static_assert otherwise).
//   * detail::accumulate_paths takes the grids instead of NnIndex handles.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "qtree/cuda/capi.hpp"
#include "qtree/model/chains.hpp"
#include "qtree/model/chains_ext.hpp"
#include "qtree/quant/nn.hpp"
#include "qtree/rng/stream.hpp"
#include "qtree/tree/quant_tree.hpp"

namespace qtree::tree {

enum class EstimatorKind { AlgI, AlgII, AlgIII };

/// Phase attribution (estimate.hpp:22-28). On the device path: simulate = 0
/// (normals are generated inside the fused path kernel), nn = the path
/// kernel(s), merge = the NCCL reduction (devices > 1), normalize = visits +
/// row normalisation, total = the whole call including host<->device copies.
struct BuildPhases {
  double simulate_ms = 0.0;
  double nn_ms = 0.0;
  double merge_ms = 0.0;
  double normalize_ms = 0.0;
  double total_ms = 0.0;
};

struct EstimateOptions {
  rng::EngineKind engine = rng::EngineKind::Mrg32k3a;
  std::uint64_t seed = 12345;
  int workers = 1;
  quant::NnBackend nn = quant::NnBackend::BruteForce;
  BuildPhases* phases = nullptr;  // optional timing sink
  int devices = 1;                // new: GPUs of this process (paths sharded, one NCCL sum)
};

namespace detail {

/// estimate.hpp:48-50
inline std::uint64_t uniforms_per_path(std::uint64_t normals) { return 2 * ((normals + 1) / 2); }

template <class Chain>
QuantTree run_device_estimate(qt_estimator alg, const Chain& chain,
                              std::span<const quant::QuantGrid> grids, std::uint64_t samples,
                              const EstimateOptions& opt) {
  const cuda::PackedGrids pg = cuda::pack_grids(chain, grids);  // estimate.hpp:52-64
  const cuda::ChainCoefficients cc = cuda::coefficients(chain);
  std::uint64_t nv = 0, nj = 0;
  cuda::flat_sizes(pg.sizes, nv, nj);
  std::vector<std::uint64_t> visits(nv), joint(nj);
  std::vector<double> pi(nj);
  double ph[5] = {0, 0, 0, 0, 0};
  const qt_chain c = cc.view();
  const qt_grids g = pg.view();
  cuda::check(qt_estimate(alg, &c, &g, samples, static_cast<int32_t>(opt.engine), opt.seed,
                          opt.devices, visits.data(), joint.data(), pi.data(), ph),
              "estimate");
  // make_tree_shell (estimate.hpp:66-75): layer 0 is {initial()}
  QuantTree t;
  std::vector<double> x0(static_cast<std::size_t>(chain.dim()));
  chain.initial(x0);
  t.grids.reserve(grids.size() + 1);
  t.grids.emplace_back(chain.dim(), x0);
  for (const auto& gr : grids) t.grids.push_back(gr);
  t.samples = samples;
  cuda::unflatten(pg.sizes, visits, joint, &pi, t.counts, &t.pi);
  if (opt.phases) {
    opt.phases->simulate_ms = ph[0];
    opt.phases->nn_ms = ph[1];
    opt.phases->merge_ms = ph[2];
    opt.phases->normalize_ms = ph[3];
    opt.phases->total_ms = ph[4];
  }
  return t;
}

/// Path window [first_path, first_path + path_count) of a run of
/// `total_paths` paths, ADDED into `cs` (estimate.hpp:88-126); `cs` must have
/// the CountMatrixSet::zeros shape of the grids.
template <class Chain>
void accumulate_paths(const Chain& chain, std::span<const quant::QuantGrid> grids,
                      rng::EngineKind engine, std::uint64_t seed, std::uint64_t first_path,
                      std::uint64_t path_count, std::uint64_t total_paths, CountMatrixSet& cs) {
  const cuda::PackedGrids pg = cuda::pack_grids(chain, grids);
  const cuda::ChainCoefficients cc = cuda::coefficients(chain);
  std::uint64_t nv = 0, nj = 0;
  cuda::flat_sizes(pg.sizes, nv, nj);
  std::vector<std::uint64_t> visits(nv, 0), joint(nj, 0);
  const qt_chain c = cc.view();
  const qt_grids g = pg.view();
  cuda::check(qt_accumulate_paths(&c, &g, static_cast<int32_t>(engine), seed, first_path,
                                  path_count, total_paths, visits.data(), joint.data()),
              "accumulate_paths");
  CountMatrixSet part;
  cuda::unflatten(pg.sizes, visits, joint, nullptr, part, nullptr);
  cs.add(part);
}

}  // namespace detail

/// Algorithm I (estimate.hpp:133-157): same counts as the reference's serial
/// loop; on the device every path runs concurrently.
template <model::MarkovChain Chain>
QuantTree estimate_alg1(const Chain& chain, std::span<const quant::QuantGrid> grids,
                        std::uint64_t paths, const EstimateOptions& opt = {}) {
  if (paths == 0) throw std::invalid_argument("estimate: need at least one path");
  return detail::run_device_estimate(QT_ALG_I, chain, grids, paths, opt);
}

/// Algorithm II (estimate.hpp:163-207): bit-identical to Algorithm I for any
/// worker and device count.
template <model::MarkovChain Chain>
QuantTree estimate_alg2(const Chain& chain, std::span<const quant::QuantGrid> grids,
                        std::uint64_t paths, const EstimateOptions& opt = {}) {
  if (opt.workers < 1) throw std::invalid_argument("estimate_alg2: workers must be >= 1");
  if (paths == 0) throw std::invalid_argument("estimate: need at least one path");
  return detail::run_device_estimate(QT_ALG_II, chain, grids, paths, opt);
}

/// Algorithm III (estimate.hpp:213-296): `samples_per_layer` pair samples per
/// transition, sample (k, m) on substream (k-1) M + m.
template <model::MarkovChain Chain>
QuantTree estimate_alg3(const Chain& chain, std::span<const quant::QuantGrid> grids,
                        std::uint64_t samples_per_layer, const EstimateOptions& opt = {}) {
  if (opt.workers < 1) throw std::invalid_argument("estimate_alg3: workers must be >= 1");
  if (samples_per_layer == 0) throw std::invalid_argument("estimate: need at least one sample");
  return detail::run_device_estimate(QT_ALG_III, chain, grids, samples_per_layer, opt);
}

/// Dispatch by estimator kind (estimate.hpp:299-309).
template <model::MarkovChain Chain>
QuantTree estimate(EstimatorKind kind, const Chain& chain,
                   std::span<const quant::QuantGrid> grids, std::uint64_t paths,
                   const EstimateOptions& opt = {}) {
  switch (kind) {
    case EstimatorKind::AlgI: return estimate_alg1(chain, grids, paths, opt);
    case EstimatorKind::AlgII: return estimate_alg2(chain, grids, paths, opt);
    case EstimatorKind::AlgIII: return estimate_alg3(chain, grids, paths, opt);
  }
  throw std::invalid_argument("estimate: unknown estimator kind");
}

}  // namespace qtree::tree
