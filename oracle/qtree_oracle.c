/*
 * qtree_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker for the CUDA
 * path. Plain-C restatement of the reference hot path (arXiv 1101.3228
 * quantization-tree transition estimator + backward-DP pricer), written from
 * the reference's behaviour, each function citing the file:line it follows
 * (paths relative to /root/reference/proj/include/qtree/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker. It is pinned against the reference
 * itself (oracle/_ref, built from the unmodified reference headers) by
 * tests/test_oracle.py and against the committed fixtures in tests/golden/.
 *
 * Build: gcc -std=c11 -O3 -ffp-contract=off (no -march): the reference is
 * compiled without FMA contraction, and every product/sum below must round
 * separately exactly as it does there.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle_api.h"

typedef unsigned __int128 u128;

enum { E_OK = 0, E_INVALID = 1, E_CONFIG = 2, E_IO = 3, E_NUMERIC = 4, E_OTHER = 9 };

/* ------------------------------------------------------------------------ */
/* RNG engines                                                               */
/* ------------------------------------------------------------------------ */

/* splitmix64 finaliser, rng/mrg32k3a.hpp:23-29 */
static uint64_t sm64(uint64_t* z) {
  *z += 0x9E3779B97F4A7C15ull;
  uint64_t v = *z;
  v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ull;
  v = (v ^ (v >> 27)) * 0x94D049BB133111EBull;
  return v ^ (v >> 31);
}

/* MRG32k3a constants, rng/mrg32k3a.hpp:8-13 */
#define M1 4294967087ull
#define M2 4294944443ull
#define A12 1403580ll
#define A13N 810728ll
#define A21 527612ll
#define A23N 1370589ll

typedef struct { uint64_t s1[3], s2[3]; } mrg_t;
typedef struct { uint64_t a[3][3]; } mat3;
typedef struct { mat3 m1, m2; } mrg_jump_t;

/* rng/mrg32k3a.hpp:34-40: both histories seeded from one splitmix sequence */
static mrg_t mrg_seed(uint64_t seed) {
  mrg_t s;
  uint64_t z = seed;
  for (int i = 0; i < 3; ++i) s.s1[i] = 1 + sm64(&z) % (M1 - 1);
  for (int i = 0; i < 3; ++i) s.s2[i] = 1 + sm64(&z) % (M2 - 1);
  return s;
}

/* rng/mrg32k3a.hpp:44-63: signed-64 recurrences, output (x+1)/(m1+1) */
static double mrg_next(mrg_t* s) {
  int64_t p1 = (A12 * (int64_t)s->s1[1] - A13N * (int64_t)s->s1[0]) % (int64_t)M1;
  if (p1 < 0) p1 += (int64_t)M1;
  s->s1[0] = s->s1[1];
  s->s1[1] = s->s1[2];
  s->s1[2] = (uint64_t)p1;
  int64_t p2 = (A21 * (int64_t)s->s2[2] - A23N * (int64_t)s->s2[0]) % (int64_t)M2;
  if (p2 < 0) p2 += (int64_t)M2;
  s->s2[0] = s->s2[1];
  s->s2[1] = s->s2[2];
  s->s2[2] = (uint64_t)p2;
  const uint64_t x = (uint64_t)p1 >= (uint64_t)p2 ? (uint64_t)(p1 - p2)
                                                  : (uint64_t)p1 + M1 - (uint64_t)p2;
  return (double)(x + 1) / (double)(M1 + 1);
}

static mat3 mat3_eye(void) {
  mat3 r;
  memset(&r, 0, sizeof r);
  for (int i = 0; i < 3; ++i) r.a[i][i] = 1;
  return r;
}

/* rng/mrg32k3a.hpp:73-84: 128-bit accumulate then reduce */
static mat3 mat3_mul(const mat3* x, const mat3* y, uint64_t m) {
  mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      u128 acc = 0;
      for (int k = 0; k < 3; ++k) acc += (u128)x->a[i][k] * y->a[k][j];
      r.a[i][j] = (uint64_t)(acc % m);
    }
  return r;
}

static void mat3_apply(const mat3* x, uint64_t v[3], uint64_t m) {
  uint64_t r[3];
  for (int i = 0; i < 3; ++i) {
    u128 acc = 0;
    for (int k = 0; k < 3; ++k) acc += (u128)x->a[i][k] * v[k];
    r[i] = (uint64_t)(acc % m);
  }
  memcpy(v, r, sizeof r);
}

static mat3 mat3_pow(mat3 b, uint64_t e, uint64_t m) {
  mat3 acc = mat3_eye();
  while (e) {
    if (e & 1) acc = mat3_mul(&acc, &b, m);
    b = mat3_mul(&b, &b, m);
    e >>= 1;
  }
  return acc;
}

/* companion matrices on (x_{n-3}, x_{n-2}, x_{n-1}), rng/mrg32k3a.hpp:109-119 */
static mrg_jump_t mrg_jump(uint64_t steps) {
  mat3 c1, c2;
  memset(&c1, 0, sizeof c1);
  memset(&c2, 0, sizeof c2);
  c1.a[0][1] = 1; c1.a[1][2] = 1; c1.a[2][0] = M1 - (uint64_t)A13N; c1.a[2][1] = (uint64_t)A12;
  c2.a[0][1] = 1; c2.a[1][2] = 1; c2.a[2][0] = M2 - (uint64_t)A23N; c2.a[2][2] = (uint64_t)A21;
  mrg_jump_t j;
  j.m1 = mat3_pow(c1, steps, M1);
  j.m2 = mat3_pow(c2, steps, M2);
  return j;
}

static void mrg_jump_apply(const mrg_jump_t* j, mrg_t* s) {
  mat3_apply(&j->m1, s->s1, M1);
  mat3_apply(&j->m2, s->s2, M2);
}

/* LCG48 = drand48 constants, rng/lcg48.hpp:8-34 */
#define LCG_MASK ((1ull << 48) - 1)
typedef struct { uint64_t x, a, c; } lcg_t;
typedef struct { uint64_t A, C; } lcg_jump_t;

static lcg_t lcg_seed(uint64_t seed) {
  lcg_t s = {((seed << 16) | 0x330Eull) & LCG_MASK, 0x5DEECE66Dull, 0xBull};
  return s;
}
static double lcg_next(lcg_t* s) {
  s->x = (s->a * s->x + s->c) & LCG_MASK;
  return (double)s->x * 0x1p-48;
}
/* binary splitting of the affine map, rng/lcg48.hpp:46-61 */
static lcg_jump_t lcg_jump(uint64_t a, uint64_t c, uint64_t steps) {
  lcg_jump_t acc = {1, 0}, base = {a & LCG_MASK, c & LCG_MASK};
  while (steps) {
    if (steps & 1) {
      lcg_jump_t t = {(base.A * acc.A) & LCG_MASK, (base.A * acc.C + base.C) & LCG_MASK};
      acc = t;
    }
    lcg_jump_t b2 = {(base.A * base.A) & LCG_MASK, (base.A * base.C + base.C) & LCG_MASK};
    base = b2;
    steps >>= 1;
  }
  return acc;
}
static void lcg_jump_apply(const lcg_jump_t* j, lcg_t* s) { s->x = (j->A * s->x + j->C) & LCG_MASK; }

/* XORWOW, rng/xorwow.hpp:16-47 */
typedef struct { uint32_t v, w, x, y, z, d; } xw_t;
static xw_t xw_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed ^ (0x9E3779B97F4A7C15ull * (stream + 1));
  const uint64_t a = sm64(&z), b = sm64(&z), c = sm64(&z);
  xw_t s = {(uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32), (uint32_t)c,
            (uint32_t)(c >> 32)};
  if ((s.v | s.w | s.x | s.y | s.z) == 0) s.v = 1;
  return s;
}
static uint32_t xw_next(xw_t* s) {
  const uint32_t t = s->x ^ (s->x >> 2);
  s->x = s->y; s->y = s->z; s->z = s->w; s->w = s->v;
  s->v = (s->v ^ (s->v << 4)) ^ (t ^ (t << 1));
  s->d += 362437u;
  return s->v + s->d;
}

/* ------------------------------------------------------------------------ */
/* Streams (rng/stream.hpp)                                                  */
/* ------------------------------------------------------------------------ */

typedef struct {
  int engine;
  mrg_t mrg;
  lcg_t lcg;
  xw_t xw;
  int interleaved;
  mrg_jump_t mj;
  lcg_jump_t lj;
  double spare;
  int has_spare;
} stream_t;

/* next_uniform, stream.hpp:81-93 */
static double st_uniform(stream_t* g) {
  double u;
  if (g->engine == OQ_ENGINE_LCG48) {
    u = lcg_next(&g->lcg);
    if (g->interleaved) lcg_jump_apply(&g->lj, &g->lcg);
  } else if (g->engine == OQ_ENGINE_MRG32K3A) {
    u = mrg_next(&g->mrg);
    if (g->interleaved) mrg_jump_apply(&g->mj, &g->mrg);
  } else {
    u = (double)xw_next(&g->xw) * 0x1p-32;
  }
  return u;
}

/* Box-Muller with clamp, stream.hpp:57-62; cached mate, stream.hpp:97-108 */
static double st_gaussian(stream_t* g) {
  if (g->has_spare) {
    g->has_spare = 0;
    return g->spare;
  }
  double u1 = st_uniform(g);
  const double u2 = st_uniform(g);
  if (u1 <= 0.0) u1 = 0x1p-64;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.14159265358979323846 * u2;
  g->spare = r * sin(a);
  g->has_spare = 1;
  return r * cos(a);
}

/* split_stream, stream.hpp:143-178 */
static int st_split(int engine, uint64_t seed, int skip, uint64_t count, uint64_t index,
                    uint64_t block, stream_t* g) {
  if (count == 0 || index >= count || (!skip && block == 0)) return E_INVALID;
  memset(g, 0, sizeof *g);
  g->engine = engine;
  if (engine == OQ_ENGINE_XORWOW) {
    if (skip) return E_INVALID;
    g->xw = xw_seed(seed, index);
    for (int i = 0; i < 64; ++i) xw_next(&g->xw);
    return E_OK;
  }
  const uint64_t offset = skip ? index : index * block;
  if (engine == OQ_ENGINE_LCG48) {
    g->lcg = lcg_seed(seed);
    if (offset) {
      lcg_jump_t j = lcg_jump(g->lcg.a, g->lcg.c, offset);
      lcg_jump_apply(&j, &g->lcg);
    }
    if (skip && count > 1) {
      g->lj = lcg_jump(g->lcg.a, g->lcg.c, count - 1);
      g->interleaved = 1;
    }
  } else if (engine == OQ_ENGINE_MRG32K3A) {
    g->mrg = mrg_seed(seed);
    if (offset) {
      mrg_jump_t j = mrg_jump(offset);
      mrg_jump_apply(&j, &g->mrg);
    }
    if (skip && count > 1) {
      g->mj = mrg_jump(count - 1);
      g->interleaved = 1;
    }
  } else {
    return E_INVALID;
  }
  return E_OK;
}

/* PathStreamer, stream.hpp:182-231: path m = block substream m of size D */
typedef struct {
  int engine;
  uint64_t seed, draws, next, total;
  mrg_t mrg;
  lcg_t lcg;
  mrg_jump_t mj;
  lcg_jump_t lj;
} paths_t;

static int ps_init(paths_t* p, int engine, uint64_t seed, uint64_t draws, uint64_t first,
                   uint64_t total) {
  if (draws == 0) return E_INVALID;
  memset(p, 0, sizeof *p);
  p->engine = engine;
  p->seed = seed;
  p->draws = draws;
  p->next = first;
  p->total = total;
  if (engine == OQ_ENGINE_LCG48) {
    p->lcg = lcg_seed(seed);
    if (first * draws != 0) {
      lcg_jump_t j = lcg_jump(p->lcg.a, p->lcg.c, first * draws);
      lcg_jump_apply(&j, &p->lcg);
    }
    p->lj = lcg_jump(p->lcg.a, p->lcg.c, draws);
  } else if (engine == OQ_ENGINE_MRG32K3A) {
    p->mrg = mrg_seed(seed);
    if (first * draws != 0) {
      mrg_jump_t j = mrg_jump(first * draws);
      mrg_jump_apply(&j, &p->mrg);
    }
    p->mj = mrg_jump(draws);
  } else if (engine != OQ_ENGINE_XORWOW) {
    return E_INVALID;
  }
  return E_OK;
}

static void ps_next(paths_t* p, stream_t* g) {
  if (p->engine == OQ_ENGINE_XORWOW) {
    st_split(OQ_ENGINE_XORWOW, p->seed, 0, p->total, p->next, p->draws, g);
  } else {
    memset(g, 0, sizeof *g);
    g->engine = p->engine;
    if (p->engine == OQ_ENGINE_LCG48) {
      g->lcg = p->lcg;
      lcg_jump_apply(&p->lj, &p->lcg);
    } else {
      g->mrg = p->mrg;
      mrg_jump_apply(&p->mj, &p->mrg);
    }
  }
  ++p->next;
}

/* uniforms_per_path, tree/estimate.hpp:48-50 */
static uint64_t draws_for(uint64_t normals) { return 2 * ((normals + 1) / 2); }

/* ------------------------------------------------------------------------ */
/* Chains (model/chains.hpp, model/two_factor.hpp)                           */
/* ------------------------------------------------------------------------ */

typedef struct {
  int kind, dim, nps, n;
  double* step;  /* per transition t=0..n-1, 5 doubles (see below) */
  double* marg;  /* per layer k=0..n, 6 doubles */
} chain_t;

/* ou_covariance, two_factor.hpp:57-63 */
static void ou_cov(double t, double a1, double a2, double rho, double c[3]) {
  c[0] = -expm1(-2.0 * a1 * t) / (2.0 * a1);
  c[2] = -expm1(-2.0 * a2 * t) / (2.0 * a2);
  c[1] = -rho * expm1(-(a1 + a2) * t) / (a1 + a2);
}

/* cholesky2, two_factor.hpp:67-77 (l11, l21, l22) */
static int chol2(const double c[3], double l[3]) {
  if (c[0] < 0.0 || c[2] < 0.0) return E_NUMERIC;
  l[0] = sqrt(c[0]);
  l[1] = l[0] > 0.0 ? c[1] / l[0] : 0.0;
  const double rem = c[2] - l[1] * l[1];
  if (rem < -1e-12 * (1.0 > c[2] ? 1.0 : c[2])) return E_NUMERIC;
  l[2] = sqrt(rem > 0.0 ? rem : 0.0);
  return E_OK;
}

/* TwoFactorParams::validate, two_factor.hpp:28-42 */
static int validate_params(const oq_chain* c) {
  if (!(c->s0 > 0.0) || !(c->sigma1 >= 0.0) || !(c->sigma2 >= 0.0) || !(c->alpha1 > 0.0) ||
      !(c->alpha2 > 0.0) || !(c->rho >= -1.0 && c->rho <= 1.0) || !isfinite(c->r) ||
      !(c->strike > 0.0) || !(c->horizon > 0.0) || c->steps < 1)
    return E_CONFIG;
  return E_OK;
}

static void chain_free(chain_t* ch) {
  free(ch->step);
  free(ch->marg);
}

/* 3x3 correlation Cholesky for the C5 basket (new chain, see oracle_api.h) */
static void corr_chol3(const double rho[3], double L[3][3]) {
  memset(L, 0, 9 * sizeof(double));
  L[0][0] = 1.0;
  L[1][0] = rho[0];
  L[1][1] = sqrt(1.0 - L[1][0] * L[1][0]);
  L[2][0] = rho[1];
  L[2][1] = (rho[2] - L[2][0] * L[1][0]) / L[1][1];
  L[2][2] = sqrt(1.0 - L[2][0] * L[2][0] - L[2][1] * L[2][1]);
}

static int chain_make(const oq_chain* c, chain_t* ch) {
  memset(ch, 0, sizeof *ch);
  ch->kind = c->kind;
  ch->n = c->steps;
  const int n = c->steps;
  if (c->kind == OQ_CHAIN_BROWNIAN1D) {
    /* BrownianChain1d, chains.hpp:68-95 */
    if (n < 1 || !(c->horizon > 0.0)) return E_NUMERIC;
    ch->dim = 1;
    ch->nps = 1;
  } else if (c->kind == OQ_CHAIN_TWO_FACTOR || c->kind == OQ_CHAIN_OU1D) {
    const int rc = validate_params(c);
    if (rc) return rc;
    ch->dim = c->kind == OQ_CHAIN_TWO_FACTOR ? 2 : 1;
    ch->nps = ch->dim;
  } else if (c->kind == OQ_CHAIN_GBM3D) {
    if (n < 1) return E_NUMERIC;
    ch->dim = 3;
    ch->nps = 3;
  } else {
    return E_INVALID;
  }
  ch->step = calloc((size_t)n * 6, sizeof(double));
  ch->marg = calloc((size_t)(n + 1) * 6, sizeof(double));
  if (!ch->step || !ch->marg) return E_OTHER;
  if (c->kind == OQ_CHAIN_BROWNIAN1D) {
    const double dt = c->horizon / n; /* dt(), chains.hpp:78 */
    for (int k = 0; k < n; ++k) ch->step[6 * k] = sqrt(dt);
    for (int k = 0; k <= n; ++k) ch->marg[6 * k] = k == 0 ? 0.0 : sqrt(k * dt);
  } else if (c->kind == OQ_CHAIN_TWO_FACTOR || c->kind == OQ_CHAIN_OU1D) {
    /* Ar1Spec::from_params, two_factor.hpp:90-101; marginals chains.hpp:32-36 */
    const double dt = c->horizon / c->steps;
    double cv[3], l[3];
    ou_cov(dt, c->alpha1, c->alpha2, c->rho, cv);
    if (chol2(cv, l)) return E_NUMERIC;
    const double a1 = exp(-c->alpha1 * dt), a2 = exp(-c->alpha2 * dt);
    for (int k = 0; k < n; ++k) {
      double* s = ch->step + 6 * k;
      s[0] = a1; s[1] = a2; s[2] = l[0]; s[3] = l[1]; s[4] = l[2];
    }
    for (int k = 0; k <= n; ++k) {
      ou_cov(k * dt, c->alpha1, c->alpha2, c->rho, cv); /* time(k) = k*dt() */
      if (chol2(cv, l)) return E_NUMERIC;
      double* m = ch->marg + 6 * k;
      m[0] = l[0]; m[1] = l[1]; m[2] = l[2];
    }
  } else {
    double L[3][3];
    corr_chol3(c->gbm_rho, L);
    const double dt = c->horizon / n;
    const double sdt = sqrt(dt);
    for (int k = 0; k < n; ++k) {
      double* s = ch->step + 6 * k;
      s[0] = sdt * L[0][0]; s[1] = sdt * L[1][0]; s[2] = sdt * L[1][1];
      s[3] = sdt * L[2][0]; s[4] = sdt * L[2][1]; s[5] = sdt * L[2][2];
    }
    for (int k = 0; k <= n; ++k) {
      const double st = sqrt(k * dt);
      double* m = ch->marg + 6 * k;
      m[0] = st * L[0][0]; m[1] = st * L[1][0]; m[2] = st * L[1][1];
      m[3] = st * L[2][0]; m[4] = st * L[2][1]; m[5] = st * L[2][2];
    }
  }
  return E_OK;
}

/* Chain::step (chains.hpp:48-53, :83-86; new chains per oracle_api.h) */
static void chain_step(const chain_t* ch, int k, const double* x, double* out, const double* e) {
  const double* s = ch->step + 6 * k;
  switch (ch->kind) {
    case OQ_CHAIN_BROWNIAN1D: out[0] = x[0] + s[0] * e[0]; break;
    case OQ_CHAIN_TWO_FACTOR:
      out[0] = s[0] * x[0] + s[2] * e[0];
      out[1] = s[1] * x[1] + s[3] * e[0] + s[4] * e[1];
      break;
    case OQ_CHAIN_OU1D: out[0] = s[0] * x[0] + s[2] * e[0]; break;
    default:
      out[0] = x[0] + s[0] * e[0];
      out[1] = x[1] + (s[1] * e[0] + s[2] * e[1]);
      out[2] = x[2] + ((s[3] * e[0] + s[4] * e[1]) + s[5] * e[2]);
  }
}

/* Chain::sample_marginal (chains.hpp:55-59, :88-90) */
static void chain_marginal(const chain_t* ch, int k, double* out, const double* e) {
  const double* m = ch->marg + 6 * k;
  switch (ch->kind) {
    case OQ_CHAIN_BROWNIAN1D: out[0] = k == 0 ? 0.0 : m[0] * e[0]; break;
    case OQ_CHAIN_TWO_FACTOR:
      out[0] = m[0] * e[0];
      out[1] = m[1] * e[0] + m[2] * e[1];
      break;
    case OQ_CHAIN_OU1D: out[0] = m[0] * e[0]; break;
    default:
      out[0] = m[0] * e[0];
      out[1] = m[1] * e[0] + m[2] * e[1];
      out[2] = (m[3] * e[0] + m[4] * e[1]) + m[5] * e[2];
  }
}

/* ------------------------------------------------------------------------ */
/* Grids and nearest neighbour (quant/grid.hpp, quant/nn.hpp)                */
/* ------------------------------------------------------------------------ */

static int cmp_lex_dim;
static const double* cmp_lex_pts;
static int cmp_lex(const void* a, const void* b) {
  const double* pa = cmp_lex_pts + (size_t)(*(const uint64_t*)a) * cmp_lex_dim;
  const double* pb = cmp_lex_pts + (size_t)(*(const uint64_t*)b) * cmp_lex_dim;
  for (int j = 0; j < cmp_lex_dim; ++j) {
    if (pa[j] < pb[j]) return -1;
    if (pa[j] > pb[j]) return 1;
  }
  return 0;
}

/* QuantGrid invariants, grid.hpp:24-31,41-55: finite and pairwise distinct */
static pthread_mutex_t cmp_mu = PTHREAD_MUTEX_INITIALIZER;
static int grid_check(int dim, uint64_t npts, const double* pts) {
  if (dim < 1 || npts == 0) return E_NUMERIC;
  for (uint64_t i = 0; i < npts * (uint64_t)dim; ++i)
    if (!isfinite(pts[i])) return E_NUMERIC;
  uint64_t* ord = malloc(npts * sizeof *ord);
  if (!ord) return E_OTHER;
  for (uint64_t i = 0; i < npts; ++i) ord[i] = i;
  pthread_mutex_lock(&cmp_mu);
  cmp_lex_dim = dim;
  cmp_lex_pts = pts;
  qsort(ord, npts, sizeof *ord, cmp_lex);
  int rc = E_OK;
  for (uint64_t i = 1; i < npts && rc == E_OK; ++i)
    if (cmp_lex(&ord[i - 1], &ord[i]) == 0) rc = E_NUMERIC;
  pthread_mutex_unlock(&cmp_mu);
  free(ord);
  return rc;
}

/* nearest_brute, nn.hpp:18-46: strict < keeps the smallest index on ties;
 * d=2 fast path dx*dx+dy*dy, otherwise squared_distance (grid.hpp:65-72). */
static uint64_t nearest(int dim, uint64_t npts, const double* pts, const double* q) {
  uint64_t best = 0;
  double best_d2 = INFINITY;
  if (dim == 2) {
    const double qx = q[0], qy = q[1];
    for (uint64_t i = 0; i < npts; ++i) {
      const double dx = qx - pts[2 * i];
      const double dy = qy - pts[2 * i + 1];
      const double d2 = dx * dx + dy * dy;
      if (d2 < best_d2) {
        best_d2 = d2;
        best = i;
      }
    }
    return best;
  }
  for (uint64_t i = 0; i < npts; ++i) {
    double acc = 0.0;
    for (int j = 0; j < dim; ++j) {
      const double diff = q[j] - pts[i * (uint64_t)dim + (uint64_t)j];
      acc += diff * diff;
    }
    if (acc < best_d2) {
      best_d2 = acc;
      best = i;
    }
  }
  return best;
}

/* ------------------------------------------------------------------------ */
/* Estimator (tree/estimate.hpp)                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
  int n, dim;
  const uint64_t* sizes;
  const double** layer_pts;  /* [1..n] */
  uint64_t* voff;            /* visits offset per layer 0..n */
  uint64_t* joff;            /* joint offset per transition t=0..n-1 */
  uint64_t nvis, njoint;
} layout_t;

static int layout_make(const chain_t* ch, const uint64_t* sizes, const double* pts, layout_t* L) {
  memset(L, 0, sizeof *L);
  L->n = ch->n;
  L->dim = ch->dim;
  L->sizes = sizes;
  if (sizes[0] != 1) return E_INVALID;
  L->layer_pts = calloc((size_t)ch->n + 1, sizeof(double*));
  L->voff = calloc((size_t)ch->n + 2, sizeof(uint64_t));
  L->joff = calloc((size_t)ch->n + 1, sizeof(uint64_t));
  if (!L->layer_pts || !L->voff || !L->joff) return E_OTHER;
  uint64_t off = 0;
  for (int k = 1; k <= ch->n; ++k) {
    L->layer_pts[k] = pts + off;
    const int rc = grid_check(ch->dim, sizes[k], pts + off);
    if (rc) return rc;
    off += sizes[k] * (uint64_t)ch->dim;
  }
  for (int k = 0; k <= ch->n; ++k) L->voff[k + 1] = L->voff[k] + sizes[k];
  for (int t = 0; t < ch->n; ++t) L->joff[t + 1] = L->joff[t] + sizes[t] * sizes[t + 1];
  L->nvis = L->voff[ch->n + 1];
  L->njoint = L->joff[ch->n];
  return E_OK;
}

static void layout_free(layout_t* L) {
  free(L->layer_pts);
  free(L->voff);
  free(L->joff);
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

/* detail::accumulate_paths, estimate.hpp:88-126 */
static int accumulate(const chain_t* ch, const layout_t* L, int engine, uint64_t seed,
                      uint64_t first, uint64_t count, uint64_t total, uint64_t* visits,
                      uint64_t* joint, double* sim_ms, double* nn_ms) {
  const int n = ch->n, d = ch->dim, nps = ch->nps;
  const uint64_t normals = (uint64_t)n * (uint64_t)nps;
  paths_t ps;
  int rc = ps_init(&ps, engine, seed, draws_for(normals), first, total);
  if (rc) return rc;
  double* eps = malloc(normals * sizeof(double));
  if (!eps) return E_OTHER;
  double x[3], xn[3], ts = 0.0, tn = 0.0;
  for (uint64_t m = 0; m < count; ++m) {
    stream_t g;
    ps_next(&ps, &g);
    const double t0 = now_ms();
    for (uint64_t e = 0; e < normals; ++e) eps[e] = st_gaussian(&g);
    const double t1 = now_ms();
    ts += t1 - t0;
    x[0] = x[1] = x[2] = 0.0; /* initial(): the origin for every chain */
    uint64_t i = 0;
    ++visits[L->voff[0]];
    for (int k = 1; k <= n; ++k) {
      chain_step(ch, k - 1, x, xn, eps + (size_t)(k - 1) * (size_t)nps);
      memcpy(x, xn, sizeof x);
      const uint64_t j = nearest(d, L->sizes[k], L->layer_pts[k], x);
      ++joint[L->joff[k - 1] + i * L->sizes[k] + j];
      ++visits[L->voff[k] + j];
      i = j;
    }
    tn += now_ms() - t1;
  }
  free(eps);
  if (sim_ms) *sim_ms = ts;
  if (nn_ms) *nn_ms = tn;
  return E_OK;
}

typedef struct {
  const chain_t* ch;
  const layout_t* L;
  int engine;
  uint64_t seed, first, count, total;
  uint64_t *visits, *joint;
  double sim, nn;
  int rc;
  /* Alg III task queue */
  int* next_layer;
  pthread_mutex_t* mu;
  uint64_t per_layer;
} work_t;

static void* alg2_worker(void* arg) {
  work_t* w = arg;
  w->rc = accumulate(w->ch, w->L, w->engine, w->seed, w->first, w->count, w->total, w->visits,
                     w->joint, &w->sim, &w->nn);
  return NULL;
}

/* estimate_alg3 worker body, estimate.hpp:237-265 */
static void* alg3_worker(void* arg) {
  work_t* w = arg;
  const chain_t* ch = w->ch;
  const layout_t* L = w->L;
  const int n = ch->n, d = ch->dim, nps = ch->nps;
  const uint64_t normals = (uint64_t)d + (uint64_t)nps;
  const uint64_t M = w->per_layer;
  double eps[8], x[3], xn[3];
  for (;;) {
    pthread_mutex_lock(w->mu);
    const int k = (*w->next_layer)++;
    pthread_mutex_unlock(w->mu);
    if (k > n) return NULL;
    const int tk = k - 1;
    paths_t ps;
    w->rc = ps_init(&ps, w->engine, w->seed, draws_for(normals), (uint64_t)tk * M,
                    (uint64_t)n * M);
    if (w->rc) return NULL;
    const uint64_t cols = L->sizes[k];
    for (uint64_t m = 0; m < M; ++m) {
      stream_t g;
      ps_next(&ps, &g);
      const double s0 = now_ms();
      for (uint64_t e = 0; e < normals; ++e) eps[e] = st_gaussian(&g);
      chain_marginal(ch, k - 1, x, eps);
      chain_step(ch, k - 1, x, xn, eps + d);
      const double s1 = now_ms();
      w->sim += s1 - s0;
      const uint64_t i = k - 1 == 0 ? 0 : nearest(d, L->sizes[k - 1], L->layer_pts[k - 1], x);
      const uint64_t j = nearest(d, L->sizes[k], L->layer_pts[k], xn);
      ++w->joint[L->joff[tk] + i * cols + j];
      ++w->visits[L->voff[tk] + i];
      w->nn += now_ms() - s1;
    }
  }
}

/* QuantTree::normalize, quant_tree.hpp:69-83 */
static void normalize(const layout_t* L, const uint64_t* visits, const uint64_t* joint, double* pi) {
  for (int t = 0; t < L->n; ++t) {
    const uint64_t rows = L->sizes[t], cols = L->sizes[t + 1];
    for (uint64_t i = 0; i < rows; ++i) {
      const uint64_t den = visits[L->voff[t] + i];
      double* row = pi + L->joff[t] + i * cols;
      const uint64_t* jr = joint + L->joff[t] + i * cols;
      for (uint64_t j = 0; j < cols; ++j) row[j] = den == 0 ? 0.0 : (double)jr[j] / (double)den;
    }
  }
}

OQ_EXPORT int oq_chain_dims(const oq_chain* c, int* dim, int* nps) {
  chain_t ch;
  const int rc = chain_make(c, &ch);
  if (!rc) {
    *dim = ch.dim;
    *nps = ch.nps;
  }
  chain_free(&ch);
  return rc;
}

OQ_EXPORT int oq_estimate(int alg, const oq_chain* c, const uint64_t* sizes, const double* pts,
                          uint64_t paths, int engine, uint64_t seed, int workers,
                          uint64_t* visits, uint64_t* joint, double* pi, double* phases5) {
  if (alg < OQ_ALG_I || alg > OQ_ALG_III) return E_INVALID;
  if (alg != OQ_ALG_I && workers < 1) return E_INVALID; /* estimate.hpp:166,216 */
  if (paths == 0) return E_INVALID;                      /* estimate.hpp:136,167,217 */
  const double t0 = now_ms();
  chain_t ch;
  layout_t L;
  int rc = chain_make(c, &ch);
  if (!rc) rc = layout_make(&ch, sizes, pts, &L);
  if (rc) {
    chain_free(&ch);
    return rc;
  }
  memset(visits, 0, L.nvis * sizeof(uint64_t));
  memset(joint, 0, L.njoint * sizeof(uint64_t));
  double sim = 0.0, nn = 0.0, merge = 0.0, tm = 0.0;
  if (alg == OQ_ALG_I) {
    rc = accumulate(&ch, &L, engine, seed, 0, paths, paths, visits, joint, &sim, &nn);
    tm = now_ms();
  } else {
    const uint64_t W = alg == OQ_ALG_II ? ((uint64_t)workers < paths ? (uint64_t)workers : paths)
                                        : (uint64_t)(workers < ch.n ? workers : ch.n);
    work_t* w = calloc(W, sizeof *w);
    pthread_t* th = calloc(W, sizeof *th);
    int next_layer = 1;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    for (uint64_t i = 0; i < W; ++i) {
      w[i].ch = &ch;
      w[i].L = &L;
      w[i].engine = engine;
      w[i].seed = seed;
      w[i].total = paths;
      if (alg == OQ_ALG_II) {
        /* contiguous blocks [M w/W, M (w+1)/W), estimate.hpp:180-181 */
        w[i].first = (uint64_t)((u128)paths * i / W);
        w[i].count = (uint64_t)((u128)paths * (i + 1) / W) - w[i].first;
        w[i].visits = calloc(L.nvis, sizeof(uint64_t));
        w[i].joint = calloc(L.njoint, sizeof(uint64_t));
        pthread_create(&th[i], NULL, alg2_worker, &w[i]);
      } else {
        /* layer tasks write disjoint slices of the shared set, estimate.hpp:244-245 */
        w[i].visits = visits;
        w[i].joint = joint;
        w[i].next_layer = &next_layer;
        w[i].mu = &mu;
        w[i].per_layer = paths;
        pthread_create(&th[i], NULL, alg3_worker, &w[i]);
      }
    }
    for (uint64_t i = 0; i < W; ++i) pthread_join(th[i], NULL);
    tm = now_ms();
    uint64_t busiest = 0;
    for (uint64_t i = 0; i < W; ++i) {
      if (w[i].rc) rc = w[i].rc;
      if (w[i].sim + w[i].nn > w[busiest].sim + w[busiest].nn) busiest = i;
    }
    sim = w[busiest].sim;
    nn = w[busiest].nn;
    if (alg == OQ_ALG_II) {
      /* CountMatrixSet::add merge, quant_tree.hpp:35-40 */
      for (uint64_t i = 0; i < W; ++i) {
        for (uint64_t e = 0; e < L.nvis; ++e) visits[e] += w[i].visits[e];
        for (uint64_t e = 0; e < L.njoint; ++e) joint[e] += w[i].joint[e];
        free(w[i].visits);
        free(w[i].joint);
      }
    } else {
      /* visits[n] = column sums of the last joint, estimate.hpp:275-281 */
      const int n = ch.n;
      const uint64_t rows = sizes[n - 1], cols = sizes[n];
      for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j)
          visits[L.voff[n] + j] += joint[L.joff[n - 1] + i * cols + j];
    }
    merge = now_ms() - tm;
    free(w);
    free(th);
  }
  const double tn = now_ms();
  if (!rc) normalize(&L, visits, joint, pi);
  if (phases5) {
    phases5[0] = sim;
    phases5[1] = nn;
    phases5[2] = merge;
    phases5[3] = now_ms() - tn;
    phases5[4] = now_ms() - t0;
  }
  layout_free(&L);
  chain_free(&ch);
  return rc;
}

OQ_EXPORT int oq_accumulate_paths(const oq_chain* c, const uint64_t* sizes, const double* pts,
                                  int engine, uint64_t seed, uint64_t first, uint64_t count,
                                  uint64_t total, uint64_t* visits, uint64_t* joint) {
  chain_t ch;
  layout_t L;
  int rc = chain_make(c, &ch);
  if (!rc) rc = layout_make(&ch, sizes, pts, &L);
  if (!rc) {
    rc = accumulate(&ch, &L, engine, seed, first, count, total, visits, joint, NULL, NULL);
    layout_free(&L);
  }
  chain_free(&ch);
  return rc;
}

OQ_EXPORT int oq_path_normals(int engine, uint64_t seed, uint64_t normals, uint64_t first,
                              uint64_t count, uint64_t total, double* out) {
  paths_t ps;
  const int rc = ps_init(&ps, engine, seed, draws_for(normals), first, total);
  if (rc) return rc;
  for (uint64_t m = 0; m < count; ++m) {
    stream_t g;
    ps_next(&ps, &g);
    for (uint64_t e = 0; e < normals; ++e) *out++ = st_gaussian(&g);
  }
  return E_OK;
}

OQ_EXPORT int oq_uniforms(int engine, uint64_t seed, int skip_ahead, uint64_t streams,
                          uint64_t index, uint64_t block, uint64_t n, double* out) {
  stream_t g;
  const int rc = st_split(engine, seed, skip_ahead, streams, index, block, &g);
  if (rc) return rc;
  for (uint64_t i = 0; i < n; ++i) out[i] = st_uniform(&g);
  return E_OK;
}

OQ_EXPORT int oq_nearest_brute(int dim, uint64_t npts, const double* pts, uint64_t nq,
                               const double* q, uint64_t* out) {
  const int rc = grid_check(dim, npts, pts);
  if (rc) return rc;
  for (uint64_t i = 0; i < nq; ++i) out[i] = nearest(dim, npts, pts, q + i * (uint64_t)dim);
  return E_OK;
}

OQ_EXPORT int oq_normalize(int n, const uint64_t* sizes, const uint64_t* visits,
                           const uint64_t* joint, double* pi) {
  layout_t L;
  memset(&L, 0, sizeof L);
  L.n = n;
  L.sizes = sizes;
  L.voff = calloc((size_t)n + 2, sizeof(uint64_t));
  L.joff = calloc((size_t)n + 1, sizeof(uint64_t));
  for (int k = 0; k <= n; ++k) L.voff[k + 1] = L.voff[k] + sizes[k];
  for (int t = 0; t < n; ++t) L.joff[t + 1] = L.joff[t] + sizes[t] * sizes[t + 1];
  normalize(&L, visits, joint, pi);
  free(L.voff);
  free(L.joff);
  return E_OK;
}

/* ------------------------------------------------------------------------ */
/* Obstacles (pipeline.hpp:124-170, two_factor.hpp:144-176)                  */
/* ------------------------------------------------------------------------ */

/* spot(), two_factor.hpp:144-152 */
static double spot2(const oq_chain* p, double sigma2, double t, double x1, double x2) {
  double cv[3];
  ou_cov(t, p->alpha1, p->alpha2, p->rho, cv);
  const double mu = p->sigma1 * p->sigma1 * cv[0] + 2.0 * p->sigma1 * sigma2 * cv[1] +
                    sigma2 * sigma2 * cv[2];
  return p->s0 * exp(p->sigma1 * x1 + sigma2 * x2 - 0.5 * mu);
}

/* std::max(a, b) semantics: (a < b) ? b : a */
static double std_max(double a, double b) { return a < b ? b : a; }

static double payoff_at(const oq_chain* p, int dim, int kind, int k, const double* x) {
  const double dt = p->horizon / p->steps;
  const double t = k * dt;
  const double disc = exp(-p->r * t);
  if (p->kind == OQ_CHAIN_GBM3D || kind == OQ_PAYOFF_MAXCALL) {
    double best = -INFINITY;
    for (int a = 0; a < 3; ++a) {
      const double sg = p->gbm_sigma[a];
      const double s = p->s0 * exp((p->r - 0.5 * sg * sg) * t + sg * x[a]);
      if (s > best) best = s;
    }
    return disc * std_max(best - p->strike, 0.0);
  }
  double s;
  if (p->kind == OQ_CHAIN_OU1D) {
    s = spot2(p, 0.0, t, x[0], 0.0);
  } else if (dim == 1) {
    /* amer_*_payoff / 1-D swing: s0 exp((r - sigma1^2/2) t + sigma1 x) */
    s = p->s0 * exp((p->r - 0.5 * p->sigma1 * p->sigma1) * t + p->sigma1 * x[0]);
  } else {
    s = spot2(p, p->sigma2, t, x[0], x[1]);
  }
  if (kind == OQ_PAYOFF_PUT) return disc * std_max(p->strike - s, 0.0);
  if (kind == OQ_PAYOFF_CALL) return disc * std_max(s - p->strike, 0.0);
  return disc * (s - p->strike);
}

OQ_EXPORT int oq_payoff_table(const oq_chain* c, int payoff, const uint64_t* sizes,
                              const double* pts_all, double* phi) {
  chain_t ch;
  const int rc = chain_make(c, &ch);
  const int dim = ch.dim;
  chain_free(&ch);
  if (rc) return rc;
  for (int k = 0; k <= c->steps; ++k)
    for (uint64_t i = 0; i < sizes[k]; ++i) {
      *phi++ = payoff_at(c, dim, payoff, k, pts_all);
      pts_all += dim;
    }
  return E_OK;
}

OQ_EXPORT int oq_build_grids(const oq_chain* c, uint64_t grid_size, uint64_t seed,
                             uint64_t per_iter, int iterations, double* out) {
  (void)c; (void)grid_size; (void)seed; (void)per_iter; (void)iterations; (void)out;
  return E_OTHER; /* Lloyd is not on the hot path */
}

OQ_EXPORT int oq_lloyd_base(int dim, uint64_t grid_size, uint64_t seed, uint64_t per_iter,
                            int iterations, double* out) {
  (void)dim; (void)grid_size; (void)seed; (void)per_iter; (void)iterations; (void)out;
  return E_OTHER;
}

/* ------------------------------------------------------------------------ */
/* Backward dynamic programming (pricer/bdp.hpp, pricer/swing.hpp)            */
/* ------------------------------------------------------------------------ */

/* cond_expectation, bdp.hpp:36-54: dense row . f in ascending j, NaN if unvisited */
static void cond_exp(uint64_t rows, uint64_t cols, const uint64_t* vis, const double* pi,
                     const double* f, double* out) {
  for (uint64_t i = 0; i < rows; ++i) {
    if (vis[i] == 0) {
      out[i] = NAN;
      continue;
    }
    double acc = 0.0;
    for (uint64_t j = 0; j < cols; ++j) acc += pi[i * cols + j] * f[j];
    out[i] = acc;
  }
}

OQ_EXPORT int oq_solve_stopping(int n, const uint64_t* sizes, const uint64_t* visits,
                                const double* pi, const double* phi, double* value,
                                uint8_t* exercise, double* price) {
  uint64_t* voff = calloc((size_t)n + 2, sizeof(uint64_t));
  uint64_t* poff = calloc((size_t)n + 1, sizeof(uint64_t));
  for (int k = 0; k <= n; ++k) voff[k + 1] = voff[k] + sizes[k];
  for (int t = 0; t < n; ++t) poff[t + 1] = poff[t] + sizes[t] * sizes[t + 1];
  double* V = malloc(voff[n + 1] * sizeof(double));
  uint8_t* X = malloc(voff[n + 1]);
  int rc = E_OK;
  /* terminal layer, bdp.hpp:71-77 */
  for (uint64_t i = 0; i < sizes[n]; ++i) {
    const double f = phi[voff[n] + i];
    if (!isfinite(f)) rc = E_NUMERIC;
    V[voff[n] + i] = f;
    X[voff[n] + i] = f > 0.0;
  }
  double* cont = malloc(sizeof(double) * (sizes[0] > 1 ? sizes[0] : 1));
  for (int k = n - 1; k >= 0 && rc == E_OK; --k) {
    cont = realloc(cont, sizes[k] * sizeof(double));
    cond_exp(sizes[k], sizes[k + 1], visits + voff[k], pi + poff[k], V + voff[k + 1], cont);
    for (uint64_t i = 0; i < sizes[k]; ++i) {
      const double f = phi[voff[k] + i];
      if (!isfinite(f)) rc = E_NUMERIC;
      if (isnan(cont[i])) { /* absorbing, bdp.hpp:85-88 */
        V[voff[k] + i] = f;
        X[voff[k] + i] = 1;
      } else {
        V[voff[k] + i] = std_max(f, cont[i]);
        X[voff[k] + i] = f >= cont[i];
      }
    }
  }
  if (rc == E_OK) {
    *price = V[0];
    if (value) memcpy(value, V, voff[n + 1] * sizeof(double));
    if (exercise) memcpy(exercise, X, voff[n + 1]);
  }
  free(cont);
  free(V);
  free(X);
  free(voff);
  free(poff);
  return rc;
}

/* solve_swing, swing.hpp:47-129 */
OQ_EXPORT int oq_solve_swing(int n, const uint64_t* sizes, const uint64_t* visits,
                             const double* pi, const double* phi, int qmin, int qmax,
                             double* price, double* value_all) {
  if (qmin < 0 || qmin > qmax || qmax > n || qmin > n) return E_CONFIG;
  uint64_t* voff = calloc((size_t)n + 2, sizeof(uint64_t));
  uint64_t* poff = calloc((size_t)n + 1, sizeof(uint64_t));
  int* lo = calloc((size_t)n + 1, sizeof(int));
  int* cnt = calloc((size_t)n + 1, sizeof(int));
  uint64_t* soff = calloc((size_t)n + 2, sizeof(uint64_t));
  for (int k = 0; k <= n; ++k) voff[k + 1] = voff[k] + sizes[k];
  for (int t = 0; t < n; ++t) poff[t + 1] = poff[t] + sizes[t] * sizes[t + 1];
  for (int k = 0; k <= n; ++k) {
    const int l = qmin - (n - k) > 0 ? qmin - (n - k) : 0;
    const int h = k < qmax ? k : qmax;
    lo[k] = l;
    cnt[k] = h - l + 1;
    soff[k + 1] = soff[k] + (uint64_t)cnt[k] * sizes[k];
  }
  double* P = calloc(soff[n + 1], sizeof(double)); /* terminal P_n = 0 */
  int rc = E_OK;
  for (int k = n - 1; k >= 0 && rc == E_OK; --k) {
    const uint64_t nodes = sizes[k], nn = sizes[k + 1];
    double* cont = malloc((size_t)cnt[k + 1] * nodes * sizeof(double));
    for (int mi = 0; mi < cnt[k + 1]; ++mi)
      cond_exp(nodes, nn, visits + voff[k], pi + poff[k], P + soff[k + 1] + (uint64_t)mi * nn,
               cont + (uint64_t)mi * nodes);
    for (int m = lo[k]; m < lo[k] + cnt[k]; ++m) {
      const int can_wait = m + (n - k - 1) >= qmin;
      const int can_take = m + 1 <= qmax;
      for (uint64_t i = 0; i < nodes; ++i) {
        const double v = phi[voff[k] + i];
        if (!isfinite(v)) rc = E_NUMERIC;
        double best = -INFINITY;
        if (can_wait) {
          const double c = cont[(uint64_t)(m - lo[k + 1]) * nodes + i];
          best = isnan(c) ? 0.0 : c;
        }
        if (can_take) {
          const double c = cont[(uint64_t)(m + 1 - lo[k + 1]) * nodes + i];
          const double cand = v + (isnan(c) ? 0.0 : c);
          if (cand >= best) best = cand;
        }
        P[soff[k] + (uint64_t)(m - lo[k]) * nodes + i] = best;
      }
    }
    free(cont);
  }
  if (rc == E_OK) {
    *price = P[0];
    if (value_all) memcpy(value_all, P, soff[n + 1] * sizeof(double));
  }
  free(P);
  free(voff);
  free(poff);
  free(lo);
  free(cnt);
  free(soff);
  return rc;
}
