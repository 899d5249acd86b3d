// qtree/quant/lloyd.hpp -- DROP-IN replacement of the reference's grid builder
// (/root/reference/proj/include/qtree/quant/lloyd.hpp) on libqtree_cuda.so.
//
//   PointSampler, QuantError, GaussianSampler, LloydResult   lloyd.hpp:16-24,55-58,110-117
//   distortion                                                lloyd.hpp:30-48
//   lloyd_build                                               lloyd.hpp:59-107
//
// GaussianSampler on an MRG32k3a stream in block mode (what pipeline.hpp's
// build_*_grids pass, pipeline.hpp:27-77) runs entirely on the device:
// qt_lloyd_build_stream / qt_distortion_stream generate the stream's normals
// (the glibc-exact Box-Muller), project exactly and recenter with per-cell sums
// in sample order, and hand back the stream state, so g ends where the
// reference leaves it and the grid is the reference's bit for bit. Any other
// sampler or stream keeps its draws on the host (the sampler is caller code)
// and sends every iteration's nearest-point and recentering work to the device
// (qt_lloyd_iterate, qt_distortion_points) -- the same arithmetic, the same
// results. `backend` is accepted: the device projection is the exact
// brute-force argmin the kd-tree also returns (nn.hpp:127,138-140).
#pragma once

#include <algorithm>
#include <limits>
#include <cmath>
#include <concepts>
#include <cstdint>
#include <set>
#include <span>
#include <stdexcept>
#include <type_traits>
#include <variant>
#include <vector>

#include "qtree/cuda/capi.hpp"
#include "qtree/errors.hpp"
#include "qtree/quant/grid.hpp"
#include "qtree/quant/nn.hpp"
#include "qtree/rng/stream.hpp"

namespace qtree::quant {

/// Anything that can fill a d-vector with a fresh draw from a target law.
template <class S>
concept PointSampler = requires(const S s, rng::RngStream& g, std::span<double> out) {
  { s.dim() } -> std::convertible_to<int>;
  s.sample(g, out);
};

/// Monte Carlo estimate of the quadratic distortion E min_i |X - x_i|^2.
struct QuantError {
  double distortion = 0.0;
  double std_error = 0.0;
  std::uint64_t samples = 0;
};

struct LloydResult {
  QuantGrid grid;
  std::vector<double> distortion;  // per-iteration estimate, under the old centers
};

/// Standard-normal product sampler (lloyd.hpp:110-117).
struct GaussianSampler {
  int dimension = 1;
  int dim() const { return dimension; }
  void sample(rng::RngStream& g, std::span<double> out) const {
    for (auto& v : out) v = g.next_gaussian();
  }
};

namespace b200 {

// RngStream keeps its engine state and cached mate private (stream.hpp:112-121)
// and befriends only split_stream / PathStreamer. The device path must read and
// write them to continue the caller's stream; an explicit instantiation may
// name private members ([temp.spec]), which is how these accessors reach them.
template <class Tag, typename Tag::type M>
struct Reach {
  friend typename Tag::type member(Tag) { return M; }
};
struct EngineOf {
  using type = std::variant<rng::Lcg48State, rng::Mrg32k3aState, rng::XorwowState> rng::RngStream::*;
  friend type member(EngineOf);
};
struct InterleavedOf {
  using type = bool rng::RngStream::*;
  friend type member(InterleavedOf);
};
struct SpareOf {
  using type = double rng::RngStream::*;
  friend type member(SpareOf);
};
struct HasSpareOf {
  using type = bool rng::RngStream::*;
  friend type member(HasSpareOf);
};
template struct Reach<EngineOf, &rng::RngStream::engine_>;
template struct Reach<InterleavedOf, &rng::RngStream::interleaved_>;
template struct Reach<SpareOf, &rng::RngStream::spare_>;
template struct Reach<HasSpareOf, &rng::RngStream::has_spare_>;

/// The MRG32k3a block-mode state of g, or null when the device stream cannot
/// continue it (another engine, or skip-ahead interleaving).
inline rng::Mrg32k3aState* device_stream(rng::RngStream& g) {
  if (g.*member(InterleavedOf{})) return nullptr;
  return std::get_if<rng::Mrg32k3aState>(&(g.*member(EngineOf{})));
}

/// Runs `call(state6, has_spare, spare)` on g's state and writes the result back.
template <class F>
void with_stream(rng::RngStream& g, rng::Mrg32k3aState& st, F&& call) {
  std::uint64_t s6[6] = {st.s1[0], st.s1[1], st.s1[2], st.s2[0], st.s2[1], st.s2[2]};
  std::int32_t has = (g.*member(HasSpareOf{})) ? 1 : 0;
  double spare = g.*member(SpareOf{});
  call(s6, &has, &spare);
  st.s1 = {s6[0], s6[1], s6[2]};
  st.s2 = {s6[3], s6[4], s6[5]};
  g.*member(HasSpareOf{}) = has != 0;
  g.*member(SpareOf{}) = spare;
}

/// `count` draws of the sampler, sample-major.
template <class S>
std::vector<double> draw(const S& sampler, std::uint64_t count, std::size_t d, rng::RngStream& g) {
  std::vector<double> x(static_cast<std::size_t>(count) * d);
  for (std::uint64_t m = 0; m < count; ++m)
    sampler.sample(g, std::span<double>(x.data() + m * d, d));
  return x;
}

}  // namespace b200

template <PointSampler S>
QuantError distortion(const QuantGrid& grid, const S& sampler, std::uint64_t samples,
                      rng::RngStream& g, NnBackend backend = NnBackend::KdTree) {
  if (samples == 0) throw std::invalid_argument("distortion: samples must be >= 1");
  if (sampler.dim() != grid.dim()) throw NumericError("distortion: sampler dimension mismatch");
  (void)backend;
  const auto pts = grid.data();
  QuantError e;
  e.samples = samples;
  rng::Mrg32k3aState* st = std::is_same_v<S, GaussianSampler> ? b200::device_stream(g) : nullptr;
  if (st) {
    b200::with_stream(g, *st, [&](std::uint64_t* s6, std::int32_t* has, double* spare) {
      cuda::check(qt_distortion_stream(grid.dim(), grid.size(), pts.data(), samples, s6, has, spare,
                                       &e.distortion, &e.std_error),
                  "distortion");
    });
  } else {
    const auto x = b200::draw(sampler, samples, static_cast<std::size_t>(grid.dim()), g);
    cuda::check(qt_distortion_points(grid.dim(), grid.size(), pts.data(), samples, x.data(),
                                     &e.distortion, &e.std_error),
                "distortion");
  }
  return e;
}

template <PointSampler S>
LloydResult lloyd_build(const S& sampler, std::size_t n_points, int dim, int iterations,
                        std::uint64_t samples_per_iter, rng::RngStream& g,
                        NnBackend backend = NnBackend::KdTree) {
  if (n_points == 0) throw std::invalid_argument("lloyd_build: need at least one center");
  if (iterations < 0) throw std::invalid_argument("lloyd_build: iterations must be >= 0");
  if (sampler.dim() != dim) throw NumericError("lloyd_build: sampler dimension mismatch");
  (void)backend;
  const std::size_t d = static_cast<std::size_t>(dim);
  LloydResult result;
  std::vector<double> centers(n_points * d);
  rng::Mrg32k3aState* st =
      std::is_same_v<S, GaussianSampler> && dim <= 3 ? b200::device_stream(g) : nullptr;
  if (st) {  // the whole build on the device, continuing g's own stream
    std::vector<double> dist(static_cast<std::size_t>(std::max(iterations, 1)));
    b200::with_stream(g, *st, [&](std::uint64_t* s6, std::int32_t* has, double* spare) {
      cuda::check(qt_lloyd_build_stream(dim, n_points, iterations, samples_per_iter, s6, has,
                                        spare, centers.data(), dist.data()),
                  "lloyd_build");
    });
    result.distortion.assign(dist.begin(), dist.begin() + iterations);
    result.grid = QuantGrid(dim, std::move(centers));
    return result;
  }
  // host draws (caller sampler), device iterations. Initial centers: distinct
  // samples in stream order (lloyd.hpp:72-83).
  centers.clear();
  std::set<std::vector<double>> seen;
  std::vector<double> x(d);
  std::uint64_t attempts = 0;
  while (centers.size() < n_points * d) {
    sampler.sample(g, x);
    if (seen.insert(x).second) centers.insert(centers.end(), x.begin(), x.end());
    if (++attempts > 100 * n_points + 100)
      throw NumericError("lloyd_build: sampler cannot produce enough distinct centers");
  }
  for (int it = 0; it < iterations; ++it) {
    const QuantGrid snapshot(dim, centers);  // the reference's grid checks
    if (samples_per_iter == 0) {  // nothing assigned: centers kept, 0 / 0 (lloyd.hpp:97)
      volatile double zero = 0.0;
      result.distortion.push_back(zero / zero);
      continue;
    }
    const auto xs = b200::draw(sampler, samples_per_iter, d, g);
    double dist = 0.0;
    cuda::check(qt_lloyd_iterate(dim, n_points, centers.data(), samples_per_iter, xs.data(), &dist),
                "lloyd_build");
    result.distortion.push_back(dist);
  }
  result.grid = QuantGrid(dim, std::move(centers));
  return result;
}

}  // namespace qtree::quant
