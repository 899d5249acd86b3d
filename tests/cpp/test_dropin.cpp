// test_dropin.cpp -- TEST INFRASTRUCTURE: the C++ drop-in headers in
// include/qtree/ driven the way a reference user drives them (unchanged
// reference callers: pipeline.hpp's build_tree / run_pipeline, the reference
// chains and grids), checked against the reference itself: oracle/_ref's
// libqtree_ref.so (the unmodified reference headers, loaded with dlopen so
// its template instances never meet ours at link time).
#include <catch2/catch_amalgamated.hpp>

#include <dlfcn.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "oracle_api.h"
#include "qtree/model/chains_ext.hpp"
#include "qtree/pipeline.hpp"
#include "qtree/pricer/bdp.hpp"
#include "qtree/pricer/swing.hpp"
#include "qtree/tree/estimate.hpp"

using namespace qtree;

namespace {

// --- the reference oracle (oracle/_ref/libqtree_ref.so) ----------------------
struct RefLib {
  decltype(&oq_estimate) estimate = nullptr;
  decltype(&oq_accumulate_paths) accumulate = nullptr;
  decltype(&oq_solve_swing) swing = nullptr;
  decltype(&oq_solve_stopping) stopping = nullptr;
  decltype(&oq_payoff_table) payoff_table = nullptr;
  decltype(&oq_build_grids) build_grids = nullptr;
  RefLib() {
    const char* p = std::getenv("QTREE_REF_LIB");
    void* h = dlopen(p ? p : "oracle/_ref/libqtree_ref.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      std::fprintf(stderr, "cannot load the reference oracle: %s\n", dlerror());
      std::abort();
    }
    estimate = reinterpret_cast<decltype(estimate)>(dlsym(h, "oq_estimate"));
    accumulate = reinterpret_cast<decltype(accumulate)>(dlsym(h, "oq_accumulate_paths"));
    swing = reinterpret_cast<decltype(swing)>(dlsym(h, "oq_solve_swing"));
    stopping = reinterpret_cast<decltype(stopping)>(dlsym(h, "oq_solve_stopping"));
    payoff_table = reinterpret_cast<decltype(payoff_table)>(dlsym(h, "oq_payoff_table"));
    build_grids = reinterpret_cast<decltype(build_grids)>(dlsym(h, "oq_build_grids"));
  }
};

const RefLib& ref() {
  static RefLib r;
  return r;
}

oq_chain oq_of(int kind, const model::TwoFactorParams& p) {
  oq_chain c{};
  c.kind = kind;
  c.steps = p.steps;
  c.horizon = p.horizon;
  c.s0 = p.s0;
  c.sigma1 = p.sigma1;
  c.sigma2 = p.sigma2;
  c.alpha1 = p.alpha1;
  c.alpha2 = p.alpha2;
  c.rho = p.rho;
  c.r = p.r;
  c.strike = p.strike;
  return c;
}

struct Flat {
  std::vector<std::uint64_t> sizes, visits, joint;
  std::vector<double> pts, pi;
};

Flat flat_of(std::span<const quant::QuantGrid> grids) {
  Flat f;
  f.sizes.push_back(1);
  for (const auto& g : grids) {
    f.sizes.push_back(g.size());
    f.pts.insert(f.pts.end(), g.data().begin(), g.data().end());
  }
  std::uint64_t nv = 0, nj = 0;
  cuda::flat_sizes(f.sizes, nv, nj);
  f.visits.assign(nv, 0);
  f.joint.assign(nj, 0);
  f.pi.assign(nj, 0.0);
  return f;
}

// QuantTree (drop-in output) == flat oracle arrays, bit for bit.
bool same_tree(const tree::QuantTree& t, const Flat& f) {
  std::size_t vo = 0, jo = 0;
  for (int k = 0; k <= t.layers(); ++k)
    for (std::uint64_t v : t.counts.visits[static_cast<std::size_t>(k)])
      if (v != f.visits[vo++]) return false;
  for (int k = 0; k < t.layers(); ++k) {
    const auto& J = t.counts.joint[static_cast<std::size_t>(k)];
    const auto& P = t.pi[static_cast<std::size_t>(k)];
    for (std::size_t e = 0; e < J.size(); ++e, ++jo)
      if (J[e] != f.joint[jo] || P[e] != f.pi[jo]) return false;
  }
  return vo == f.visits.size() && jo == f.joint.size();
}

}  // namespace

TEST_CASE("pipeline.hpp build_tree on the drop-in equals the reference", "[dropin]") {
  RunConfig cfg;
  cfg.params.steps = 24;
  cfg.grid_size = 60;
  cfg.samples = 30000;
  cfg.algorithm = 2;
  cfg.workers = 8;
  tree::BuildPhases ph;
  const tree::QuantTree t = build_tree(cfg, &ph);  // reference caller, device estimator
  REQUIRE(t.layers() == 24);
  CHECK(ph.total_ms > 0.0);
  std::vector<quant::QuantGrid> grids(t.grids.begin() + 1, t.grids.end());
  Flat f = flat_of(grids);
  const oq_chain c = oq_of(OQ_CHAIN_TWO_FACTOR, cfg.params);
  REQUIRE(ref().estimate(OQ_ALG_II, &c, f.sizes.data(), f.pts.data(), cfg.samples,
                         OQ_ENGINE_MRG32K3A, cfg.seed, 4, f.visits.data(), f.joint.data(),
                         f.pi.data(), nullptr) == 0);
  CHECK(same_tree(t, f));
  SECTION("swing price through run_pipeline's pricer equals the reference") {
    pricer::SwingProblem prob{&t, make_swing_payoff(cfg, 2), 2, 10};
    const pricer::SwingResult res = pricer::solve_swing(prob);
    std::vector<double> phi(f.visits.size());
    std::vector<double> all;
    for (const auto& g : t.grids)
      all.insert(all.end(), g.data().begin(), g.data().end());
    REQUIRE(ref().payoff_table(&c, OQ_PAYOFF_SWING, f.sizes.data(), all.data(), phi.data()) == 0);
    double ref_price = 0.0;
    std::vector<double> ref_vals(res.value.size() * 0 + 1);
    std::size_t total = 0;
    for (std::size_t k = 0; k < res.value.size(); ++k) total += res.value[k].size();
    ref_vals.assign(total, 0.0);
    REQUIRE(ref().swing(t.layers(), f.sizes.data(), f.visits.data(), f.pi.data(), phi.data(), 2, 10,
                        &ref_price, ref_vals.data()) == 0);
    CHECK(std::abs(res.price - ref_price) <= 1e-12 * std::max(1.0, std::abs(ref_price)));
    std::size_t o = 0;
    double worst = 0.0;
    for (const auto& layer : res.value)
      for (double v : layer) worst = std::max(worst, std::abs(v - ref_vals[o++]));
    CHECK(worst <= 1e-9);
    REQUIRE(res.take.size() == static_cast<std::size_t>(t.layers()));
  }
  SECTION("american put through make_put_payoff equals the reference") {
    pricer::StoppingProblem prob{&t, make_put_payoff(cfg, 2)};
    const pricer::StoppingResult res = pricer::solve_stopping(prob);
    std::vector<double> phi(f.visits.size()), all;
    for (const auto& g : t.grids) all.insert(all.end(), g.data().begin(), g.data().end());
    REQUIRE(ref().payoff_table(&c, OQ_PAYOFF_PUT, f.sizes.data(), all.data(), phi.data()) == 0);
    double ref_price = 0.0;
    REQUIRE(ref().stopping(t.layers(), f.sizes.data(), f.visits.data(), f.pi.data(), phi.data(),
                           nullptr, nullptr, &ref_price) == 0);
    CHECK(res.price == ref_price);
  }
}

TEST_CASE("run_pipeline end to end on the drop-in", "[dropin]") {
  RunConfig cfg;
  cfg.params.steps = 10;
  cfg.grid_size = 40;
  cfg.samples = 20000;
  PipelineOptions po;
  po.contract = Contract::Swing;
  po.q_max = 4;
  const PipelineResult r = run_pipeline(cfg, po);
  CHECK(std::isfinite(r.price));
  CHECK(r.price > 0.0);
  CHECK(r.report.price == r.price);
}

TEST_CASE("config-1 Brownian put: counts and price bit-exact vs the reference", "[dropin]") {
  const model::BrownianChain1d chain(10);
  const auto grids = build_brownian_grids(chain, 100, 12345);
  tree::EstimateOptions opt;
  opt.workers = 8;
  const tree::QuantTree t = tree::estimate(tree::EstimatorKind::AlgII, chain, grids, 200000, opt);
  Flat f = flat_of(grids);
  model::TwoFactorParams p;
  p.steps = 10;
  p.sigma1 = 0.2;
  p.r = 0.05;
  const oq_chain c = oq_of(OQ_CHAIN_BROWNIAN1D, p);
  REQUIRE(ref().estimate(OQ_ALG_I, &c, f.sizes.data(), f.pts.data(), 200000, OQ_ENGINE_MRG32K3A,
                         12345, 1, f.visits.data(), f.joint.data(), f.pi.data(), nullptr) == 0);
  CHECK(same_tree(t, f));
  SECTION("path window through detail::accumulate_paths") {
    tree::CountMatrixSet cs;
    std::vector<std::size_t> sz{1};
    for (const auto& g : grids) sz.push_back(g.size());
    cs = tree::CountMatrixSet::zeros(sz);
    tree::detail::accumulate_paths(chain, grids, rng::EngineKind::Mrg32k3a, 12345, 123456789,
                                   5000, 1000000000, cs);
    Flat w = flat_of(grids);
    REQUIRE(ref().accumulate(&c, w.sizes.data(), w.pts.data(), OQ_ENGINE_MRG32K3A, 12345,
                             123456789, 5000, 1000000000, w.visits.data(), w.joint.data()) == 0);
    std::size_t jo = 0;
    bool same = true;
    for (const auto& J : cs.joint)
      for (std::uint64_t v : J) same &= v == w.joint[jo++];
    CHECK(same);
  }
  SECTION("cond_expectation: NaN exactly on unvisited rows") {
    const tree::QuantTree few = tree::estimate_alg1(chain, grids, 7);
    std::vector<double> f1(few.layer_size(6), 1.0);
    const auto out = pricer::cond_expectation(few, 5, f1);
    for (std::size_t i = 0; i < out.size(); ++i)
      CHECK(std::isnan(out[i]) == !few.row_visited(6, i));
  }
}

TEST_CASE("new chains (configs 3 and 5) through the reference's templates", "[dropin]") {
  model::TwoFactorParams p;
  p.steps = 12;
  SECTION("OuChain1d, Algorithm III") {
    const model::OuChain1d chain(p);
    std::vector<quant::QuantGrid> grids;
    for (int k = 1; k <= 12; ++k) {
      std::vector<double> pts;
      for (int i = 0; i < 30; ++i) pts.push_back((-1.5 + 0.1 * i) * std::sqrt(k / 12.0) * 0.5);
      grids.emplace_back(1, std::move(pts));
    }
    const tree::QuantTree t = tree::estimate_alg3(chain, grids, 40000);
    Flat f = flat_of(grids);
    const oq_chain c = oq_of(OQ_CHAIN_OU1D, p);
    REQUIRE(ref().estimate(OQ_ALG_III, &c, f.sizes.data(), f.pts.data(), 40000, OQ_ENGINE_MRG32K3A,
                           12345, 4, f.visits.data(), f.joint.data(), f.pi.data(), nullptr) == 0);
    CHECK(same_tree(t, f));
  }
  SECTION("GbmChain3d, Algorithm II, all three engines") {
    const double rho[3] = {0.3, 0.1, -0.2};
    const model::GbmChain3d chain(6, 1.0, rho);
    std::vector<quant::QuantGrid> grids;
    rng::RngStream g = rng::split_stream(rng::EngineKind::Mrg32k3a, 7, rng::StreamPartition{});
    for (int k = 1; k <= 6; ++k) {
      std::vector<double> pts(3 * 64);
      for (auto& v : pts) v = g.next_gaussian() * std::sqrt(k / 6.0);
      grids.emplace_back(3, std::move(pts));
    }
    oq_chain c = oq_of(OQ_CHAIN_GBM3D, p);
    c.steps = 6;
    c.gbm_rho[0] = rho[0];
    c.gbm_rho[1] = rho[1];
    c.gbm_rho[2] = rho[2];
    for (int e : {0, 1, 2}) {
      tree::EstimateOptions opt;
      opt.engine = static_cast<rng::EngineKind>(e);
      opt.seed = 99;
      const tree::QuantTree t = tree::estimate_alg2(chain, grids, 20000, opt);
      Flat f = flat_of(grids);
      REQUIRE(ref().estimate(OQ_ALG_II, &c, f.sizes.data(), f.pts.data(), 20000, e, 99, 4,
                             f.visits.data(), f.joint.data(), f.pi.data(), nullptr) == 0);
      CHECK(same_tree(t, f));
    }
  }
}

TEST_CASE("errors keep the reference's exception types", "[dropin]") {
  const model::BrownianChain1d chain(3);
  std::vector<quant::QuantGrid> grids;
  for (int k = 0; k < 3; ++k) grids.emplace_back(1, std::vector<double>{-1.0, 1.0});
  CHECK_THROWS_AS(tree::estimate_alg3(chain, grids, 0), std::invalid_argument);
  tree::EstimateOptions opt;
  opt.workers = 0;
  CHECK_THROWS_AS(tree::estimate_alg3(chain, grids, 10, opt), std::invalid_argument);
  const tree::QuantTree t = tree::estimate_alg1(chain, grids, 100);
  pricer::SwingProblem bad{&t, [](int, std::span<const double>) { return 1.0; }, 3, 2};
  CHECK_THROWS_AS(pricer::solve_swing(bad), ConfigError);
  pricer::StoppingProblem nan_payoff{&t, [](int, std::span<const double>) { return NAN; }};
  CHECK_THROWS_AS(pricer::solve_stopping(nan_payoff), NumericError);
  CHECK_THROWS_AS(pricer::cond_expectation(t, 3, std::vector<double>(2, 0.0)),
                  std::invalid_argument);
}

// ---- quant/lloyd.hpp drop-in (lloyd.hpp:30-107) ------------------------------

TEST_CASE("pipeline.hpp grid builders on the drop-in Lloyd equal the reference's", "[dropin]") {
  // build_brownian_grids / build_two_factor_grids call lloyd_build(GaussianSampler, ...)
  // on an MRG32k3a block stream: the drop-in runs it on the device
  model::TwoFactorParams p;
  p.steps = 6;
  for (int kind : {OQ_CHAIN_BROWNIAN1D, OQ_CHAIN_TWO_FACTOR}) {
    std::vector<quant::QuantGrid> grids;
    const std::size_t N = kind == OQ_CHAIN_BROWNIAN1D ? 150 : 120;
    if (kind == OQ_CHAIN_BROWNIAN1D)
      grids = build_brownian_grids(model::BrownianChain1d(p.steps), N, 777);
    else
      grids = build_two_factor_grids(model::ar1_coefficients(p), N, 777);
    const oq_chain c = oq_of(kind, p);
    std::vector<double> want(static_cast<std::size_t>(p.steps) * N * grids[0].dim());
    REQUIRE(ref().build_grids(&c, N, 777, 0, 40, want.data()) == 0);
    std::vector<double> got;
    for (const auto& g : grids) got.insert(got.end(), g.data().begin(), g.data().end());
    REQUIRE(got.size() == want.size());
    for (std::size_t i = 0; i < got.size(); ++i) CHECK(got[i] == want[i]);
  }
}

TEST_CASE("drop-in lloyd_build and distortion leave the stream where the reference does",
          "[dropin]") {
  // N = 7 centers of d = 3 and 2 x 5 samples consume 21 + 30 = 51 normals: an odd
  // count, so the stream ends holding a cached Box-Muller mate
  for (bool spare_first : {false, true}) {
    auto g = rng::split_stream(rng::EngineKind::Mrg32k3a, 99, rng::StreamPartition{});
    auto h = g;  // the reference's view: draw the same normals on the host
    if (spare_first) {  // start with a cached mate
      (void)g.next_gaussian();
      (void)h.next_gaussian();
    }
    const auto res = quant::lloyd_build(quant::GaussianSampler{3}, 7, 3, 2, 5, g);
    for (int k = 0; k < 51; ++k) (void)h.next_gaussian();
    for (int k = 0; k < 5; ++k) CHECK(g.next_gaussian() == h.next_gaussian());
    CHECK(res.distortion.size() == 2);
    const auto e = quant::distortion(res.grid, quant::GaussianSampler{3}, 9, g);
    for (int k = 0; k < 27; ++k) (void)h.next_gaussian();
    CHECK(g.next_gaussian() == h.next_gaussian());
    CHECK(e.samples == 9);
  }
}

TEST_CASE("drop-in lloyd_build with a host sampler matches the device stream path", "[dropin]") {
  // a sampler that is not GaussianSampler draws on the host; here it draws the same
  // normals, so the grid and the distortions must equal the all-device build
  struct HostGauss {
    int d;
    int dim() const { return d; }
    void sample(rng::RngStream& g, std::span<double> out) const {
      for (auto& v : out) v = g.next_gaussian();
    }
  };
  auto g1 = rng::split_stream(rng::EngineKind::Mrg32k3a, 5, rng::StreamPartition{});
  auto g2 = g1;
  const auto a = quant::lloyd_build(quant::GaussianSampler{2}, 40, 2, 6, 3000, g1);
  const auto b = quant::lloyd_build(HostGauss{2}, 40, 2, 6, 3000, g2);
  REQUIRE(a.grid.size() == b.grid.size());
  for (std::size_t i = 0; i < a.grid.data().size(); ++i) CHECK(a.grid.data()[i] == b.grid.data()[i]);
  for (std::size_t i = 0; i < a.distortion.size(); ++i) CHECK(a.distortion[i] == b.distortion[i]);
  const auto ea = quant::distortion(a.grid, quant::GaussianSampler{2}, 5000, g1);
  const auto eb = quant::distortion(b.grid, HostGauss{2}, 5000, g2);
  CHECK(ea.distortion == eb.distortion);
  CHECK(ea.std_error == eb.std_error);
}
