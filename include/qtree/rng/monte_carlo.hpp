// qtree/rng/monte_carlo.hpp -- DROP-IN for the reference's rng/monte_carlo.hpp:
// estimate_pi_partitioned (monte_carlo.hpp:51-77, `qtree bench-rng`) runs on
// the GPU through qt_bench_pi (include/qtree_cuda.h); the estimate equals the
// reference's exactly (integer inside-count over bit-exact uniforms).
// estimate_pi(RngStream&, samples) on a caller-owned serial stream is the
// reference's own (it advances the caller's stream object), pulled in with
// #include_next under a renamed partitioned entry.
#pragma once

#define estimate_pi_partitioned estimate_pi_partitioned_reference
#include_next "qtree/rng/monte_carlo.hpp"
#undef estimate_pi_partitioned

#include <stdexcept>

#include "qtree_cuda.h"

namespace qtree::rng {

inline PiEstimate estimate_pi_partitioned(EngineKind kind, std::uint64_t seed,
                                          std::uint64_t samples, std::uint64_t streams,
                                          PartitionMode mode) {
  const int engine = kind == EngineKind::Lcg48 ? QT_ENGINE_LCG48
                     : kind == EngineKind::Mrg32k3a ? QT_ENGINE_MRG32K3A
                                                    : QT_ENGINE_XORWOW;
  std::uint64_t inside = 0;
  double est = 0.0, se = 0.0, ms = 0.0;
  const qt_status rc = qt_bench_pi(engine, seed, samples, streams,
                                   mode == PartitionMode::SkipAhead ? 1 : 0, &inside, &est, &se,
                                   &ms);
  if (rc != QT_OK) {
    const std::string msg = qt_last_error();
    if (rc == QT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  return {est, se, samples / 2};
}

}  // namespace qtree::rng
