// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// Drives the UNMODIFIED reference library (header-only C++20 under
// /root/reference/proj/include, included in place, never copied) through the
// plain-C interface of oracle/oracle_api.h. Built by oracle/Makefile into
// oracle/_ref/libqtree_ref.so with the reference's Release flags
// (-std=c++20 -O3 -DNDEBUG, no -march: SURVEY.md §8(c) build rule).
//
// Used to (1) pin the C restatement oracle/qtree_oracle.c, (2) generate the
// golden fixtures under tests/golden/ and (3) time the reference CPU path for
// bench.py --impl reference. Only the two chains the reference lacks (C3 OU,
// C5 GBM basket, BASELINE.json configs 3 and 5) are new code here: they are
// MarkovChain classes fed through the reference's own estimate_alg* templates.

#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "qtree/errors.hpp"
#include "qtree/model/chains.hpp"
#include "qtree/pipeline.hpp"
#include "qtree/pricer/bdp.hpp"
#include "qtree/pricer/swing.hpp"
#include "qtree/quant/lloyd.hpp"
#include "qtree/quant/nn.hpp"
#include "qtree/rng/stream.hpp"
#include "qtree/rng/monte_carlo.hpp"
#include "qtree/tree/estimate.hpp"

#include "oracle_api.h"

using namespace qtree;

namespace oqx {

// Config 3: 1-D Ornstein-Uhlenbeck, defined as factor 1 of TwoFactorChain so
// its arithmetic is the reference's (chains.hpp:51, two_factor.hpp:57-101).
class OuChain1d {
 public:
  explicit OuChain1d(const model::TwoFactorParams& p) : spec_(model::ar1_coefficients(p)) {
    for (int k = 0; k <= spec_.steps(); ++k)
      marg_.push_back(model::cholesky2(spec_.marginal_cov(k)).l11);
  }
  int dim() const { return 1; }
  int layers() const { return spec_.steps(); }
  int normals_per_step() const { return 1; }
  void initial(std::span<double> out) const { out[0] = 0.0; }
  void step(int k, std::span<const double> x, std::span<double> out,
            std::span<const double> eps) const {
    const model::Ar1Step& op = spec_.step_op(k);
    out[0] = op.a1 * x[0] + op.chol.l11 * eps[0];
  }
  void sample_marginal(int k, std::span<double> out, std::span<const double> eps) const {
    out[0] = marg_[static_cast<std::size_t>(k)] * eps[0];
  }

 private:
  model::Ar1Spec spec_;
  std::vector<double> marg_;
};

// Config 5: 3-D correlated Brownian log-state of a GBM basket,
// X_{k+1} = X_k + sqrt(dt) L eps with L = chol(corr); marginal sqrt(t_k) L eps.
struct Lower3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
};

inline Lower3 corr_chol3(const double rho[3]) {
  Lower3 l;
  l.m[0][0] = 1.0;
  l.m[1][0] = rho[0];
  l.m[1][1] = std::sqrt(1.0 - l.m[1][0] * l.m[1][0]);
  l.m[2][0] = rho[1];
  l.m[2][1] = (rho[2] - l.m[2][0] * l.m[1][0]) / l.m[1][1];
  l.m[2][2] = std::sqrt(1.0 - l.m[2][0] * l.m[2][0] - l.m[2][1] * l.m[2][1]);
  return l;
}

inline Lower3 scaled(const Lower3& l, double s) {
  Lower3 o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c <= r; ++c) o.m[r][c] = s * l.m[r][c];
  return o;
}

class GbmChain3d {
 public:
  GbmChain3d(int steps, double horizon, const double rho[3]) : steps_(steps), horizon_(horizon) {
    if (steps < 1) throw NumericError("GbmChain3d: need at least one step");
    const Lower3 l = corr_chol3(rho);
    const double dt = horizon_ / steps_;
    step_ = scaled(l, std::sqrt(dt));
    for (int k = 0; k <= steps_; ++k) marg_.push_back(scaled(l, std::sqrt(k * dt)));
  }
  int dim() const { return 3; }
  int layers() const { return steps_; }
  int normals_per_step() const { return 3; }
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
  const Lower3& marginal(int k) const { return marg_[static_cast<std::size_t>(k)]; }

 private:
  int steps_;
  double horizon_;
  Lower3 step_;
  std::vector<Lower3> marg_;
};

static_assert(model::MarkovChain<OuChain1d>);
static_assert(model::MarkovChain<GbmChain3d>);

model::TwoFactorParams params_of(const oq_chain& c) {
  model::TwoFactorParams p;
  p.s0 = c.s0;
  p.sigma1 = c.sigma1;
  p.sigma2 = c.sigma2;
  p.alpha1 = c.alpha1;
  p.alpha2 = c.alpha2;
  p.rho = c.rho;
  p.r = c.r;
  p.strike = c.strike;
  p.horizon = c.horizon;
  p.steps = c.steps;
  return p;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const ConfigError&) {
    return 2;
  } catch (const IoError&) {
    return 3;
  } catch (const NumericError&) {
    return 4;
  } catch (...) {
    return 9;
  }
}

// Calls f(chain) with the reference chain object the description names.
template <class F>
void with_chain(const oq_chain& c, F&& f) {
  switch (c.kind) {
    case OQ_CHAIN_BROWNIAN1D: f(model::BrownianChain1d(c.steps, c.horizon)); return;
    case OQ_CHAIN_TWO_FACTOR:
      f(model::TwoFactorChain(model::ar1_coefficients(params_of(c))));
      return;
    case OQ_CHAIN_OU1D: f(OuChain1d(params_of(c))); return;
    case OQ_CHAIN_GBM3D: f(GbmChain3d(c.steps, c.horizon, c.gbm_rho)); return;
  }
  throw std::invalid_argument("unknown chain kind");
}

std::vector<quant::QuantGrid> grids_of(int dim, int n, const uint64_t* sizes, const double* pts) {
  std::vector<quant::QuantGrid> g;
  std::size_t off = 0;
  for (int k = 1; k <= n; ++k) {
    const std::size_t len = static_cast<std::size_t>(sizes[k]) * static_cast<std::size_t>(dim);
    g.emplace_back(dim, std::vector<double>(pts + off, pts + off + len));
    off += len;
  }
  return g;
}

void export_counts(const tree::CountMatrixSet& cs, uint64_t* visits, uint64_t* joint, bool add) {
  std::size_t o = 0;
  for (const auto& v : cs.visits)
    for (auto x : v) {
      visits[o] = add ? visits[o] + x : x;
      ++o;
    }
  o = 0;
  for (const auto& j : cs.joint)
    for (auto x : j) {
      joint[o] = add ? joint[o] + x : x;
      ++o;
    }
}

rng::EngineKind engine_of(int e) {
  switch (e) {
    case OQ_ENGINE_LCG48: return rng::EngineKind::Lcg48;
    case OQ_ENGINE_MRG32K3A: return rng::EngineKind::Mrg32k3a;
    case OQ_ENGINE_XORWOW: return rng::EngineKind::Xorwow;
  }
  throw std::invalid_argument("unknown engine");
}

// QuantTree whose nodes are the indices 0..N_k-1 (1-D), so a tabulated
// payoff can be keyed on the node coordinate (the test_pricer.cpp:26-65 trick).
tree::QuantTree index_tree(int n, const uint64_t* sizes, const uint64_t* visits, const double* pi) {
  tree::QuantTree t;
  std::size_t vo = 0, po = 0;
  t.counts.visits.resize(static_cast<std::size_t>(n) + 1);
  t.counts.joint.resize(static_cast<std::size_t>(n));
  t.pi.resize(static_cast<std::size_t>(n));
  for (int k = 0; k <= n; ++k) {
    std::vector<double> nodes(sizes[k]);
    for (std::size_t i = 0; i < nodes.size(); ++i) nodes[i] = static_cast<double>(i);
    t.grids.emplace_back(1, std::move(nodes));
    t.counts.visits[static_cast<std::size_t>(k)].assign(visits + vo, visits + vo + sizes[k]);
    vo += sizes[k];
  }
  for (int k = 1; k <= n; ++k) {
    const std::size_t len = static_cast<std::size_t>(sizes[k - 1] * sizes[k]);
    t.pi[static_cast<std::size_t>(k - 1)].assign(pi + po, pi + po + len);
    t.counts.joint[static_cast<std::size_t>(k - 1)].assign(len, 0);
    po += len;
  }
  return t;
}

pricer::NodePayoff table_payoff(int n, const uint64_t* sizes, const double* phi) {
  std::vector<std::vector<double>> tab;
  std::size_t o = 0;
  for (int k = 0; k <= n; ++k) {
    tab.emplace_back(phi + o, phi + o + sizes[k]);
    o += sizes[k];
  }
  return [tab = std::move(tab)](int k, std::span<const double> x) {
    return tab[static_cast<std::size_t>(k)][static_cast<std::size_t>(x[0])];
  };
}

}  // namespace oqx

using namespace oqx;

extern "C" {

int oq_chain_dims(const oq_chain* c, int* dim, int* nps) {
  return guarded([&] {
    with_chain(*c, [&](const auto& ch) {
      *dim = ch.dim();
      *nps = ch.normals_per_step();
    });
  });
}

int oq_estimate(int alg, const oq_chain* c, const uint64_t* sizes, const double* pts,
                uint64_t paths, int engine, uint64_t seed, int workers, uint64_t* visits,
                uint64_t* joint, double* pi, double* phases5) {
  return guarded([&] {
    with_chain(*c, [&](const auto& ch) {
      const auto grids = grids_of(ch.dim(), ch.layers(), sizes, pts);
      tree::BuildPhases ph;
      tree::EstimateOptions opt;
      opt.engine = engine_of(engine);
      opt.seed = seed;
      opt.workers = workers;
      opt.phases = &ph;
      const auto kind = alg == OQ_ALG_I    ? tree::EstimatorKind::AlgI
                        : alg == OQ_ALG_II ? tree::EstimatorKind::AlgII
                        : alg == OQ_ALG_III ? tree::EstimatorKind::AlgIII
                                            : static_cast<tree::EstimatorKind>(alg);
      const tree::QuantTree t = tree::estimate(kind, ch, grids, paths, opt);
      export_counts(t.counts, visits, joint, false);
      std::size_t o = 0;
      for (const auto& p : t.pi)
        for (double v : p) pi[o++] = v;
      if (phases5) {
        phases5[0] = ph.simulate_ms;
        phases5[1] = ph.nn_ms;
        phases5[2] = ph.merge_ms;
        phases5[3] = ph.normalize_ms;
        phases5[4] = ph.total_ms;
      }
    });
  });
}

int oq_accumulate_paths(const oq_chain* c, const uint64_t* sizes, const double* pts, int engine,
                        uint64_t seed, uint64_t first, uint64_t count, uint64_t total,
                        uint64_t* visits, uint64_t* joint) {
  return guarded([&] {
    with_chain(*c, [&](const auto& ch) {
      const auto grids = grids_of(ch.dim(), ch.layers(), sizes, pts);
      const auto lsz = tree::detail::layer_sizes(ch, std::span<const quant::QuantGrid>(grids));
      const auto idx = tree::detail::build_indices(grids, quant::NnBackend::BruteForce);
      auto cs = tree::CountMatrixSet::zeros(lsz);
      tree::detail::accumulate_paths(ch, std::span<const quant::NnIndex>(idx),
                                     std::span<const std::size_t>(lsz), engine_of(engine), seed,
                                     first, count, total, cs, nullptr, nullptr);
      export_counts(cs, visits, joint, true);
    });
  });
}

int oq_path_normals(int engine, uint64_t seed, uint64_t normals, uint64_t first, uint64_t count,
                    uint64_t total, double* out) {
  return guarded([&] {
    rng::PathStreamer ps(engine_of(engine), seed, tree::detail::uniforms_per_path(normals), first,
                         total);
    for (uint64_t m = 0; m < count; ++m) {
      rng::RngStream g = ps.next_path();
      for (uint64_t e = 0; e < normals; ++e) *out++ = g.next_gaussian();
    }
  });
}

int oq_uniforms(int engine, uint64_t seed, int skip_ahead, uint64_t streams, uint64_t index,
                uint64_t block, uint64_t n, double* out) {
  return guarded([&] {
    rng::StreamPartition part;
    part.mode = skip_ahead ? rng::PartitionMode::SkipAhead : rng::PartitionMode::Block;
    part.stream_count = streams;
    part.stream_index = index;
    part.block_size = block;
    rng::RngStream g = rng::split_stream(engine_of(engine), seed, part);
    for (uint64_t i = 0; i < n; ++i) out[i] = g.next_uniform();
  });
}

int oq_nearest_brute(int dim, uint64_t npts, const double* pts, uint64_t nq, const double* q,
                     uint64_t* out) {
  return guarded([&] {
    const quant::QuantGrid g(dim, std::vector<double>(pts, pts + npts * static_cast<uint64_t>(dim)));
    for (uint64_t i = 0; i < nq; ++i)
      out[i] = quant::nearest_brute(
          g, std::span<const double>(q + i * static_cast<uint64_t>(dim), static_cast<std::size_t>(dim)));
  });
}

int oq_normalize(int n, const uint64_t* sizes, const uint64_t* visits, const uint64_t* joint,
                 double* pi) {
  return guarded([&] {
    tree::QuantTree t;
    std::size_t vo = 0, jo = 0;
    for (int k = 0; k <= n; ++k) {
      t.counts.visits.emplace_back(visits + vo, visits + vo + sizes[k]);
      vo += sizes[k];
    }
    for (int k = 1; k <= n; ++k) {
      const std::size_t len = static_cast<std::size_t>(sizes[k - 1] * sizes[k]);
      t.counts.joint.emplace_back(joint + jo, joint + jo + len);
      jo += len;
    }
    t.normalize();
    std::size_t o = 0;
    for (const auto& p : t.pi)
      for (double v : p) pi[o++] = v;
  });
}

int oq_payoff_table(const oq_chain* c, int payoff, const uint64_t* sizes, const double* pts_all,
                    double* phi) {
  return guarded([&] {
    int dim = 0, nps = 0;
    with_chain(*c, [&](const auto& ch) {
      dim = ch.dim();
      nps = ch.normals_per_step();
    });
    (void)nps;
    RunConfig cfg;
    cfg.params = params_of(*c);
    pricer::NodePayoff f;
    if (c->kind == OQ_CHAIN_GBM3D || payoff == OQ_PAYOFF_MAXCALL) {
      // C5 obstacle (new): discounted max-call on the 3 GBM assets.
      const model::TwoFactorParams p = cfg.params;
      const double sig[3] = {c->gbm_sigma[0], c->gbm_sigma[1], c->gbm_sigma[2]};
      const double dt = p.horizon / p.steps;
      f = [p, dt, sig](int k, std::span<const double> x) {
        const double t = k * dt;
        double best = -std::numeric_limits<double>::infinity();
        for (int a = 0; a < 3; ++a) {
          const double s = p.s0 * std::exp((p.r - 0.5 * sig[a] * sig[a]) * t + sig[a] * x[a]);
          best = std::max(best, s);
        }
        return std::exp(-p.r * t) * std::max(best - p.strike, 0.0);
      };
    } else if (c->kind == OQ_CHAIN_OU1D) {
      // C3 obstacle: factor-1 spot with sigma2 = 0.
      model::TwoFactorParams p = cfg.params;
      p.sigma2 = 0.0;
      const double dt = p.horizon / p.steps;
      if (payoff == OQ_PAYOFF_SWING)
        f = [p, dt](int k, std::span<const double> x) {
          const double t = k * dt;
          return std::exp(-p.r * t) * (model::spot(p, t, x[0], 0.0) - p.strike);
        };
      else if (payoff == OQ_PAYOFF_PUT)
        f = [p, dt](int k, std::span<const double> x) {
          const double t = k * dt;
          return std::exp(-p.r * t) * std::max(p.strike - model::spot(p, t, x[0], 0.0), 0.0);
        };
      else
        f = [p, dt](int k, std::span<const double> x) {
          const double t = k * dt;
          return std::exp(-p.r * t) * std::max(model::spot(p, t, x[0], 0.0) - p.strike, 0.0);
        };
    } else if (payoff == OQ_PAYOFF_PUT) {
      f = make_put_payoff(cfg, dim);
    } else if (payoff == OQ_PAYOFF_CALL) {
      f = make_call_payoff(cfg, dim);
    } else {
      f = make_swing_payoff(cfg, dim);
    }
    std::size_t o = 0, po = 0;
    for (int k = 0; k <= c->steps; ++k) {
      for (uint64_t i = 0; i < sizes[k]; ++i) {
        phi[o++] = f(k, std::span<const double>(pts_all + po, static_cast<std::size_t>(dim)));
        po += static_cast<std::size_t>(dim);
      }
    }
  });
}

int oq_solve_stopping(int n, const uint64_t* sizes, const uint64_t* visits, const double* pi,
                      const double* phi, double* value, uint8_t* exercise, double* price) {
  return guarded([&] {
    const tree::QuantTree t = index_tree(n, sizes, visits, pi);
    const pricer::StoppingProblem prob{&t, table_payoff(n, sizes, phi)};
    const auto res = pricer::solve_stopping(prob);
    std::size_t o = 0;
    for (int k = 0; k <= n; ++k)
      for (std::size_t i = 0; i < sizes[k]; ++i, ++o) {
        if (value) value[o] = res.value[static_cast<std::size_t>(k)][i];
        if (exercise) exercise[o] = res.exercise[static_cast<std::size_t>(k)][i];
      }
    *price = res.price;
  });
}

int oq_build_grids(const oq_chain* c, uint64_t grid_size, uint64_t seed, uint64_t per_iter,
                   int iterations, double* out) {
  return guarded([&] {
    LloydOptions lo;
    lo.iterations = iterations;
    lo.samples_per_iter = per_iter;
    std::vector<quant::QuantGrid> grids;
    if (c->kind == OQ_CHAIN_BROWNIAN1D) {
      grids = build_brownian_grids(model::BrownianChain1d(c->steps, c->horizon), grid_size, seed, lo);
    } else if (c->kind == OQ_CHAIN_TWO_FACTOR) {
      grids = build_two_factor_grids(model::ar1_coefficients(params_of(*c)), grid_size, seed, lo);
    } else {
      // New chains: one standard-normal Lloyd base grid (same stream convention
      // as pipeline.hpp:35,63) mapped by each layer's marginal factor.
      const int dim = c->kind == OQ_CHAIN_OU1D ? 1 : 3;
      const uint64_t spi = per_iter ? per_iter : std::max<uint64_t>(20000, 200 * grid_size);
      rng::RngStream g = rng::split_stream(rng::EngineKind::Mrg32k3a, seed ^ 0x9E3779B9ull,
                                           rng::StreamPartition{});
      quant::GaussianSampler sampler{dim};
      const auto base = quant::lloyd_build(sampler, grid_size, dim, iterations, spi, g);
      if (c->kind == OQ_CHAIN_OU1D) {
        const OuChain1d ch(params_of(*c));
        const auto spec = model::ar1_coefficients(params_of(*c));
        for (int k = 1; k <= c->steps; ++k) {
          const double sd = model::cholesky2(spec.marginal_cov(k)).l11;
          std::vector<double> pts(base.grid.data().begin(), base.grid.data().end());
          for (auto& v : pts) v *= sd;
          grids.emplace_back(1, std::move(pts));
        }
      } else {
        const GbmChain3d ch(c->steps, c->horizon, c->gbm_rho);
        for (int k = 1; k <= c->steps; ++k) {
          const auto& m = ch.marginal(k).m;
          std::vector<double> pts(base.grid.data().begin(), base.grid.data().end());
          for (std::size_t i = 0; i < base.grid.size(); ++i) {
            const double z0 = pts[3 * i], z1 = pts[3 * i + 1], z2 = pts[3 * i + 2];
            pts[3 * i] = m[0][0] * z0;
            pts[3 * i + 1] = m[1][0] * z0 + m[1][1] * z1;
            pts[3 * i + 2] = (m[2][0] * z0 + m[2][1] * z1) + m[2][2] * z2;
          }
          grids.emplace_back(3, std::move(pts));
        }
      }
    }
    std::size_t o = 0;
    for (const auto& g : grids)
      for (double v : g.data()) out[o++] = v;
  });
}

int oq_lloyd_base(int dim, uint64_t grid_size, uint64_t seed, uint64_t per_iter, int iterations,
                  double* out) {
  return guarded([&] {
    const uint64_t spi = per_iter ? per_iter : std::max<uint64_t>(20000, 200 * grid_size);
    rng::RngStream g = rng::split_stream(rng::EngineKind::Mrg32k3a, seed ^ 0x9E3779B9ull,
                                         rng::StreamPartition{});
    quant::GaussianSampler sampler{dim};
    const auto base = quant::lloyd_build(sampler, grid_size, dim, iterations, spi, g);
    std::size_t o = 0;
    for (double v : base.grid.data()) out[o++] = v;
  });
}

int oq_solve_swing(int n, const uint64_t* sizes, const uint64_t* visits, const double* pi,
                   const double* phi, int qmin, int qmax, double* price, double* value_all) {
  return guarded([&] {
    const tree::QuantTree t = index_tree(n, sizes, visits, pi);
    const pricer::SwingProblem prob{&t, table_payoff(n, sizes, phi), qmin, qmax};
    const auto res = pricer::solve_swing(prob);
    *price = res.price;
    if (value_all) {
      std::size_t o = 0;
      for (const auto& v : res.value)
        for (double x : v) value_all[o++] = x;
    }
  });
}

// tree::save_tree / load_tree (quant_tree.hpp:138-207) and quant::save_grid /
// load_grid (grid.hpp:84-117), the reference's own writers and readers.
int oq_save_tree(const char* path, int n, int dim, const uint64_t* sizes, const double* pts_all,
                 uint64_t samples, const uint64_t* visits, const uint64_t* joint,
                 const double* pi) {
  return guarded([&] {
    tree::QuantTree t;
    t.samples = samples;
    t.counts.visits.resize(static_cast<std::size_t>(n) + 1);
    t.counts.joint.resize(static_cast<std::size_t>(n));
    t.pi.resize(static_cast<std::size_t>(n));
    std::size_t vo = 0, jo = 0, go = 0;
    for (int k = 0; k <= n; ++k) {
      const std::size_t N = sizes[k];
      t.grids.emplace_back(dim, std::vector<double>(pts_all + go, pts_all + go + N * dim));
      go += N * dim;
      t.counts.visits[static_cast<std::size_t>(k)].assign(visits + vo, visits + vo + N);
      vo += N;
    }
    for (int k = 1; k <= n; ++k) {
      const std::size_t len = static_cast<std::size_t>(sizes[k - 1] * sizes[k]);
      t.counts.joint[static_cast<std::size_t>(k - 1)].assign(joint + jo, joint + jo + len);
      t.pi[static_cast<std::size_t>(k - 1)].assign(pi + jo, pi + jo + len);
      jo += len;
    }
    tree::save_tree(t, path);
  });
}

int oq_load_tree(const char* path, int* n, int* dim, uint64_t* samples, uint64_t* sizes,
                 double* pts_all, uint64_t* visits, uint64_t* joint, double* pi) {
  return guarded([&] {
    const tree::QuantTree t = tree::load_tree(path);
    *n = t.layers();
    *dim = t.grids[0].dim();
    *samples = t.samples;
    std::size_t vo = 0, jo = 0, go = 0;
    for (int k = 0; k <= *n; ++k) {
      const auto& g = t.grids[static_cast<std::size_t>(k)];
      sizes[k] = g.size();
      for (double v : g.data()) pts_all[go++] = v;
      for (auto v : t.counts.visits[static_cast<std::size_t>(k)]) visits[vo++] = v;
    }
    for (int k = 1; k <= *n; ++k) {
      const auto& J = t.counts.joint[static_cast<std::size_t>(k - 1)];
      const auto& P = t.pi[static_cast<std::size_t>(k - 1)];
      for (std::size_t e = 0; e < J.size(); ++e, ++jo) {
        joint[jo] = J[e];
        pi[jo] = P[e];
      }
    }
  });
}

int oq_save_grid(const char* path, int dim, uint64_t npts, const double* pts) {
  return guarded([&] {
    quant::save_grid(quant::QuantGrid(dim, std::vector<double>(pts, pts + npts * dim)), path);
  });
}

// bench-rng / bench-nn bodies (qtree_main.cpp:136-191) on the reference code
int oq_bench_pi(int engine, uint64_t seed, uint64_t samples, uint64_t streams, int skip,
                double* estimate, double* std_error) {
  return guarded([&] {
    const auto est = rng::estimate_pi_partitioned(
        engine_of(engine), seed, samples, streams,
        skip ? rng::PartitionMode::SkipAhead : rng::PartitionMode::Block);
    *estimate = est.estimate;
    *std_error = est.std_error;
  });
}

int oq_bench_nn(uint64_t n, uint64_t queries, uint64_t seed, uint64_t* sink) {
  return guarded([&] {
    rng::RngStream g = rng::split_stream(rng::EngineKind::Mrg32k3a, seed, rng::StreamPartition{});
    std::vector<double> pts(2 * n);
    for (auto& v : pts) v = g.next_gaussian();
    const quant::QuantGrid grid(2, std::move(pts));
    const quant::NnIndex index(grid, quant::NnBackend::BruteForce);
    std::vector<double> qs(2 * queries);
    for (auto& v : qs) v = g.next_gaussian();
    std::size_t s = 0;
    for (std::uint64_t q = 0; q < queries; ++q)
      s += index.nearest(std::span<const double>(qs.data() + 2 * q, 2));
    *sink = s;
  });
}

}  // extern "C"
