// qt_capi.cu -- host runtime behind include/qtree_cuda.h.
//
// Owns: validation with the reference's error taxonomy; the per-layer device
// tables (sorted 1-D threshold records + bucket index, FP32 scan tables for
// d >= 2, fast-path records); the RNG jump tables; device plans and the kernel
// selection (k_paths_x / k_paths_scan / k_alg3_* / k_paths, opt-in fast path);
// multi-GPU sharding with one NCCL all-reduce; the one-call host-buffer entry
// points with pinned staging; grid construction, micro-benchmarks and the
// batch projection. No CPU compute fallback exists: every count comes from a
// kernel (file I/O lives in qt_io.cu).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <numeric>
#include <set>
#include <thread>
#include <string>
#include <memory>
#include <vector>

#include "../../include/qtree_cuda.h"
#include "qt_internal.h"
#include "qt_layout.h"
#include "qt_math_fast.h"

namespace {

using qt::LayerTable;
using qt::Rec1;

thread_local std::string g_error;
std::atomic<uint64_t> g_launches{0};
// fast 1-D path: enabled unless QT_FAST_PATH=0 or qt_set_fast_path(0)
std::atomic<int> g_fast{-1};
// cumulative fast-path evidence of destroyed plans: paths, replayed, inline-replayed
std::atomic<uint64_t> g_fast_paths{0}, g_fast_replayed{0}, g_fast_inline{0};

// 1-D MRG32k3a lockstep exact kernel: enabled unless QT_XKERNEL=0 (then k_paths)
bool xkernel_enabled() {
  const char* e = std::getenv("QT_XKERNEL");
  return !(e && e[0] == '0');
}

// d >= 2 FP32-scan kernel: enabled unless QT_SCAN=0
bool scan_enabled() {
  const char* e = std::getenv("QT_SCAN");
  return !(e && e[0] == '0');
}

// d >= 2 cell-list projection: enabled unless QT_NN=scan (then the FP32 scan)
bool cell_enabled() {
  const char* e = std::getenv("QT_NN");
  return !(e && std::strcmp(e, "scan") == 0);
}

// 1-D MRG32k3a Alg I/II kernel: 0 = exact k_paths_x (glibc-exact Box-Muller for every
// draw), 1 = k_paths_fast (FP32 Box-Muller, certified, exact replay), 2 = k_paths_x<CERT>
// (approximate FP64 Box-Muller, certified, exact replay; the default).
// QT_FAST_PATH=0/1/2 or qt_set_fast_path(mode).
int mode1d() {
  int v = g_fast.load();
  if (v < 0) {
    const char* e = std::getenv("QT_FAST_PATH");
    v = (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 1 : 2;
    g_fast.store(v);
  }
  return v;
}
bool fast_enabled() { return mode1d() == 1; }
bool cert_enabled() { return mode1d() == 2; }

struct Failure {
  qt_status code;
  std::string msg;
};

[[noreturn]] void raise(qt_status c, const std::string& m) { throw Failure{c, m}; }

#define QT_CUDA(expr)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      raise(QT_ERR_DEVICE, std::string("cuda: ") + cudaGetErrorString(e_) + " (" #expr ")"); \
  } while (0)

template <class F>
qt_status guarded(F&& f) {
  qt::DeviceRestore keep_device;  // every entry point leaves the caller's current device as it was
  try {
    f();
    return QT_OK;
  } catch (const Failure& e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return QT_ERR_DEVICE;
  } catch (const std::exception& e) {
    g_error = e.what();
    return QT_ERR_DEVICE;
  }
}

// ---------------------------------------------------------------------------
// RNG jump tables (host side of mrg32k3a_skip / lcg48_skip)
// ---------------------------------------------------------------------------
using u128 = unsigned __int128;
constexpr uint64_t kM1 = 4294967087ull, kM2 = 4294944443ull;

struct Mat3 {
  uint64_t a[3][3];
};

Mat3 mat_mul(const Mat3& x, const Mat3& y, uint64_t m) {
  Mat3 r{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      u128 acc = 0;
      for (int k = 0; k < 3; ++k) acc += static_cast<u128>(x.a[i][k]) * y.a[k][j];
      r.a[i][j] = static_cast<uint64_t>(acc % m);
    }
  return r;
}

// J^(d 16^w), w = 0..15 (4-bit windows of the jump), d = 1..15, both components:
// entry 15 w + d - 1 = [0..8] the m1 part, [9..17] the m2 part. A jump by e applies
// one entry per non-zero hex digit of e (at most 16 instead of 64 squarings' worth).
std::vector<uint32_t> mrg_jump_table() {
  Mat3 p1{{{0, 1, 0}, {0, 0, 1}, {kM1 - 810728ull, 1403580ull, 0}}};  // J^(16^w)
  Mat3 p2{{{0, 1, 0}, {0, 0, 1}, {kM2 - 1370589ull, 0, 527612ull}}};
  std::vector<uint32_t> t(16 * 15 * 18);
  for (int w = 0; w < 16; ++w) {
    Mat3 c1 = p1, c2 = p2;  // J^(d 16^w)
    for (int d = 1; d <= 15; ++d) {
      const int b = 15 * w + d - 1;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          t[b * 18 + 3 * i + j] = static_cast<uint32_t>(c1.a[i][j]);
          t[b * 18 + 9 + 3 * i + j] = static_cast<uint32_t>(c2.a[i][j]);
        }
      c1 = mat_mul(c1, p1, kM1);
      c2 = mat_mul(c2, p2, kM2);
    }
    for (int q = 0; q < 4; ++q) {  // p <- p^16
      p1 = mat_mul(p1, p1, kM1);
      p2 = mat_mul(p2, p2, kM2);
    }
  }
  return t;
}

uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  b %= m;
  for (; e; e >>= 1) {
    if (e & 1) r = static_cast<uint64_t>(static_cast<u128>(r) * b % m);
    b = static_cast<uint64_t>(static_cast<u128>(b) * b % m);
  }
  return r;
}

// (J^e)^-1 mod m (m prime) by the adjugate
Mat3 mat_pow_inv(Mat3 c, uint64_t e, uint64_t m) {
  Mat3 r{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  for (; e; e >>= 1) {
    if (e & 1) r = mat_mul(r, c, m);
    c = mat_mul(c, c, m);
  }
  auto mm = [&](uint64_t x, uint64_t y) { return static_cast<uint64_t>(static_cast<u128>(x) * y % m); };
  auto sub = [&](uint64_t x, uint64_t y) { return (x + m - y) % m; };
  Mat3 adj{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      // cofactor of (j, i)
      const int r0 = (j + 1) % 3, r1 = (j + 2) % 3, c0 = (i + 1) % 3, c1 = (i + 2) % 3;
      adj.a[i][j] = sub(mm(r.a[r0][c0], r.a[r1][c1]), mm(r.a[r0][c1], r.a[r1][c0]));
    }
  uint64_t det = 0;
  for (int k = 0; k < 3; ++k) det = (det + mm(r.a[0][k], adj.a[k][0])) % m;
  const uint64_t inv = powmod(det, m - 2, m);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) adj.a[i][j] = mm(adj.a[i][j], inv);
  return adj;
}

// MRG32k3a state <- (J^D)^-1 state: from the end of a path back to its start
// state <- J^e state on the host (mrg32k3a_skip, mrg32k3a.hpp:124-146):
// s[0..2] component 1, s[3..5] component 2, oldest first.
void mrg_skip_host(uint64_t s[6], uint64_t e) {
  static const std::vector<uint32_t> J = mrg_jump_table();
  for (int w = 0; e != 0; ++w, e >>= 4) {
    const int d = static_cast<int>(e & 15u);
    if (!d) continue;
    for (int c = 0; c < 2; ++c) {
      const uint64_t m = c ? kM2 : kM1;
      const uint32_t* M = J.data() + (15 * w + d - 1) * 18 + 9 * c;
      uint64_t r[3];
      for (int i = 0; i < 3; ++i) {
        u128 acc = 0;
        for (int j = 0; j < 3; ++j) acc += static_cast<u128>(M[3 * i + j]) * s[3 * c + j];
        r[i] = static_cast<uint64_t>(acc % m);
      }
      for (int i = 0; i < 3; ++i) s[3 * c + i] = r[i];
    }
  }
}

void mrg_back_jump(uint64_t D, uint32_t out[18]) {
  const Mat3 c1{{{0, 1, 0}, {0, 0, 1}, {kM1 - 810728ull, 1403580ull, 0}}};
  const Mat3 c2{{{0, 1, 0}, {0, 0, 1}, {kM2 - 1370589ull, 0, 527612ull}}};
  const Mat3 i1 = mat_pow_inv(c1, D, kM1), i2 = mat_pow_inv(c2, D, kM2);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      out[3 * i + j] = static_cast<uint32_t>(i1.a[i][j]);
      out[9 + 3 * i + j] = static_cast<uint32_t>(i2.a[i][j]);
    }
}

constexpr uint64_t kLcgMask = (1ull << 48) - 1;
std::vector<unsigned long long> lcg_jump_table() {
  std::vector<unsigned long long> t(128);
  uint64_t A = 0x5DEECE66Dull, C = 0xBull;
  for (int b = 0; b < 64; ++b) {
    t[2 * b] = A;
    t[2 * b + 1] = C;
    const uint64_t A2 = (A * A) & kLcgMask, C2 = (A * C + C) & kLcgMask;
    A = A2;
    C = C2;
  }
  return t;
}

uint64_t splitmix64(uint64_t& z) {
  z += 0x9E3779B97F4A7C15ull;
  uint64_t v = z;
  v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ull;
  v = (v ^ (v >> 27)) * 0x94D049BB133111EBull;
  return v ^ (v >> 31);
}

// Device-resident copies of the jump tables, one per device.
struct DeviceTables {
  uint32_t* mrg = nullptr;
  unsigned long long* lcg = nullptr;
};
std::mutex g_dev_mu;
DeviceTables g_dev_tables[64];

const DeviceTables& device_tables(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceTables& t = g_dev_tables[dev];
  if (!t.mrg) {
    const auto m = mrg_jump_table();
    const auto l = lcg_jump_table();
    QT_CUDA(cudaMalloc(&t.mrg, m.size() * sizeof(uint32_t)));
    QT_CUDA(cudaMalloc(&t.lcg, l.size() * sizeof(unsigned long long)));
    QT_CUDA(cudaMemcpy(t.mrg, m.data(), m.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    QT_CUDA(cudaMemcpy(t.lcg, l.data(), l.size() * sizeof(unsigned long long),
                       cudaMemcpyHostToDevice));
  }
  return t;
}

qt::SrcArgs make_src(int dev, int engine, uint64_t seed, uint64_t draws, uint32_t per_unit,
                     const double* normals, uint64_t normals_first) {
  qt::SrcArgs a{};
  // mrg32k3a_seed (mrg32k3a.hpp:34-40)
  uint64_t z = seed;
  for (int i = 0; i < 3; ++i) a.mrg_seed[i] = static_cast<uint32_t>(1 + splitmix64(z) % (kM1 - 1));
  for (int i = 0; i < 3; ++i)
    a.mrg_seed[3 + i] = static_cast<uint32_t>(1 + splitmix64(z) % (kM2 - 1));
  a.lcg_seed = ((seed << 16) | 0x330Eull) & kLcgMask;  // lcg48_seed (lcg48.hpp:20-22)
  a.seed = seed;
  const DeviceTables& t = device_tables(dev);
  a.mrg_table = t.mrg;
  a.lcg_table = t.lcg;
  a.normals = normals;
  a.normals_first = normals_first;
  a.draws = draws;
  a.per_unit = per_unit;
  (void)engine;
  return a;
}

// ---------------------------------------------------------------------------
// chains
// ---------------------------------------------------------------------------
int chain_dim(int kind) {
  switch (kind) {
    case QT_CHAIN_BROWNIAN_1D: return 1;
    case QT_CHAIN_TWO_FACTOR: return 2;
    case QT_CHAIN_OU_1D: return 1;
    case QT_CHAIN_GBM_3D: return 3;
  }
  raise(QT_ERR_INVALID_ARGUMENT, "estimate: unknown chain kind");
}

// ou_covariance (two_factor.hpp:57-63)
void ou_cov(double t, double a1, double a2, double rho, double c[3]) {
  c[0] = -std::expm1(-2.0 * a1 * t) / (2.0 * a1);
  c[2] = -std::expm1(-2.0 * a2 * t) / (2.0 * a2);
  c[1] = -rho * std::expm1(-(a1 + a2) * t) / (a1 + a2);
}

// cholesky2 (two_factor.hpp:67-77)
void chol2(const double c[3], double l[3]) {
  if (c[0] < 0.0 || c[2] < 0.0) raise(QT_ERR_NUMERIC, "cholesky2: negative variance");
  l[0] = std::sqrt(c[0]);
  l[1] = l[0] > 0.0 ? c[1] / l[0] : 0.0;
  const double rem = c[2] - l[1] * l[1];
  if (rem < -1e-12 * std::max(1.0, c[2]))
    raise(QT_ERR_NUMERIC, "cholesky2: covariance not positive semi-definite");
  l[2] = std::sqrt(std::max(0.0, rem));
}

void validate_params(const qt_model_params& p) {
  auto fail = [](const char* key, const char* what) {
    raise(QT_ERR_CONFIG, std::string("parameter '") + key + "' " + what);
  };
  if (!(p.s0 > 0.0)) fail("s0", "must be > 0");
  if (!(p.sigma1 >= 0.0)) fail("sigma1", "must be >= 0");
  if (!(p.sigma2 >= 0.0)) fail("sigma2", "must be >= 0");
  if (!(p.alpha1 > 0.0)) fail("alpha1", "must be > 0");
  if (!(p.alpha2 > 0.0)) fail("alpha2", "must be > 0");
  if (!(p.rho >= -1.0 && p.rho <= 1.0)) fail("rho", "must lie in [-1, 1]");
  if (!std::isfinite(p.r)) fail("r", "must be finite");
  if (!(p.strike > 0.0)) fail("K", "must be > 0");
  if (!(p.horizon > 0.0)) fail("T", "must be > 0");
  if (p.steps < 1) fail("n", "must be >= 1");
}

void chain_coefficients(int kind, const qt_model_params& p, double* step, double* marg) {
  const int n = p.steps;
  if (kind == QT_CHAIN_BROWNIAN_1D) {
    if (n < 1) raise(QT_ERR_NUMERIC, "BrownianChain1d: need at least one step");
    if (!(p.horizon > 0.0)) raise(QT_ERR_NUMERIC, "BrownianChain1d: horizon must be > 0");
  } else if (kind == QT_CHAIN_TWO_FACTOR || kind == QT_CHAIN_OU_1D) {
    validate_params(p);
  } else if (kind == QT_CHAIN_GBM_3D) {
    if (n < 1) raise(QT_ERR_NUMERIC, "GbmChain3d: need at least one step");
  } else {
    raise(QT_ERR_INVALID_ARGUMENT, "unknown chain kind");
  }
  std::fill(step, step + static_cast<size_t>(n) * 6, 0.0);
  std::fill(marg, marg + static_cast<size_t>(n + 1) * 6, 0.0);
  if (kind == QT_CHAIN_BROWNIAN_1D) {
    const double dt = p.horizon / n;  // dt(), chains.hpp:78
    for (int k = 0; k < n; ++k) step[6 * k] = std::sqrt(dt);
    for (int k = 0; k <= n; ++k) marg[6 * k] = k == 0 ? 0.0 : std::sqrt(k * dt);
  } else if (kind == QT_CHAIN_TWO_FACTOR || kind == QT_CHAIN_OU_1D) {
    const double dt = p.horizon / p.steps;
    double c[3], l[3];
    ou_cov(dt, p.alpha1, p.alpha2, p.rho, c);
    chol2(c, l);
    const double a1 = std::exp(-p.alpha1 * dt), a2 = std::exp(-p.alpha2 * dt);
    for (int k = 0; k < n; ++k) {
      double* s = step + 6 * k;
      s[0] = a1;
      s[1] = a2;
      s[2] = l[0];
      s[3] = l[1];
      s[4] = l[2];
    }
    for (int k = 0; k <= n; ++k) {
      ou_cov(k * dt, p.alpha1, p.alpha2, p.rho, c);  // marginal_cov(k), time(k) = k dt
      chol2(c, l);
      marg[6 * k] = l[0];
      marg[6 * k + 1] = l[1];
      marg[6 * k + 2] = l[2];
    }
  } else {
    double L[3][3] = {{1.0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    L[1][0] = p.gbm_rho[0];
    L[1][1] = std::sqrt(1.0 - L[1][0] * L[1][0]);
    L[2][0] = p.gbm_rho[1];
    L[2][1] = (p.gbm_rho[2] - L[2][0] * L[1][0]) / L[1][1];
    L[2][2] = std::sqrt(1.0 - L[2][0] * L[2][0] - L[2][1] * L[2][1]);
    const double dt = p.horizon / n;
    auto fill = [&](double* o, double s) {
      o[0] = s * L[0][0];
      o[1] = s * L[1][0];
      o[2] = s * L[1][1];
      o[3] = s * L[2][0];
      o[4] = s * L[2][1];
      o[5] = s * L[2][2];
    };
    for (int k = 0; k < n; ++k) fill(step + 6 * k, std::sqrt(dt));
    for (int k = 0; k <= n; ++k) fill(marg + 6 * k, std::sqrt(k * dt));
  }
}

// ---------------------------------------------------------------------------
// grid tables
// ---------------------------------------------------------------------------
uint32_t round16(uint64_t b) { return static_cast<uint32_t>((b + 15) & ~uint64_t(15)); }

// QuantGrid invariants (grid.hpp:24-31,41-55): finite, pairwise distinct.
void check_grid(int dim, uint64_t npts, const double* pts, int layer) {
  if (npts == 0) raise(QT_ERR_NUMERIC, "grid: point data size is not a positive multiple of dim");
  for (uint64_t i = 0; i < npts * static_cast<uint64_t>(dim); ++i)
    if (!std::isfinite(pts[i]))
      raise(QT_ERR_NUMERIC, "grid: non-finite point coordinate (layer " + std::to_string(layer) + ")");
  std::vector<uint32_t> ord(npts);
  std::iota(ord.begin(), ord.end(), 0u);
  auto less = [&](uint32_t a, uint32_t b) {
    return std::lexicographical_compare(pts + a * dim, pts + (a + 1) * dim, pts + b * dim,
                                        pts + (b + 1) * dim);
  };
  std::sort(ord.begin(), ord.end(), less);
  for (uint64_t i = 1; i < npts; ++i)
    if (std::equal(pts + ord[i - 1] * dim, pts + (ord[i - 1] + 1) * dim, pts + ord[i] * dim))
      raise(QT_ERR_NUMERIC, "grid: duplicate points (layer " + std::to_string(layer) + ")");
}

// Ordered 64-bit key of a double: monotone in numeric order (-0 just below +0).
uint64_t dkey(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
double dfromkey(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
  double x;
  std::memcpy(&x, &b, 8);
  return x;
}

// The reference's pairwise choice between sorted neighbours vl < vh for a
// query x in [vl, vh]: separately rounded d2 (nn.hpp:38-45), smaller index on
// ties (strict < in index order).
bool choose_hi(double x, double vl, double vh, uint32_t ol, uint32_t oh) {
  volatile double dl = x - vl, dh = x - vh;
  volatile double d2l = dl * dl, d2h = dh * dh;
  return d2h < d2l || (d2h == d2l && oh < ol);
}

// FP32 value >= x (round toward +inf)
float f32_up(double x) {
  float f = static_cast<float>(x);
  if (static_cast<double>(f) < x) f = std::nextafter(f, std::numeric_limits<float>::infinity());
  return f;
}
// FP32 value >= |x| (round toward +inf)
float f32_up_abs(double x) {
  const double a = std::fabs(x);
  float f = static_cast<float>(a);
  if (static_cast<double>(f) < a) f = std::nextafter(f, std::numeric_limits<float>::infinity());
  return f;
}

struct TableBlob {
  std::vector<uint8_t> hot;   // staged into shared memory
  std::vector<uint8_t> cold;  // d == 1 exact-scan records (global memory only)
  std::vector<uint8_t> fast;  // d == 1 fast-path table (FastHdr + FRec[nb])
};

float f32_down(double x) {
  float f = static_cast<float>(x);
  if (static_cast<double>(f) > x) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
  return f == 0.0f ? 0.0f : f;  // never -0 (the device's up() step assumes t0 >= 0 -> bits + 1)
}

// Fast-path table of one 1-D layer from the exact decision thresholds t[0..N-1]
// (t[N-1] = +inf) in sorted-cell order, ord = original index of each sorted cell.
std::vector<uint8_t> build_fast_table(int kind, const std::vector<double>& t,
                                      const std::vector<uint32_t>& ord, double x_safe,
                                      const double* step, uint64_t joff) {
  const uint64_t N = t.size();
  qt::FastHdr h{};
  h.c0 = step[0];
  h.c2 = kind == QT_CHAIN_OU_1D ? step[2] : 0.0;
  h.joff = joff;
  h.fa = kind == QT_CHAIN_OU_1D ? f32_up_abs(step[0]) : 1.0f;
  h.fs = f32_up_abs(kind == QT_CHAIN_OU_1D ? step[2] : step[0]);
  h.x_safe = x_safe > 0.0 ? std::max(0.0f, f32_down(x_safe)) : 0.0f;
  h.n_pts = static_cast<uint32_t>(N);
  // bucket map over g(t_0) .. g(t_{N-2}), g(x) = x / sqrt(1 + gc x^2): the
  // fewest buckets (over a few gc) that hold at most one threshold each
  uint32_t nb = 1;
  double bk_a = 0.0, bk_b = 0.0, gc = 0.0;
  if (N > 2 && std::isfinite(t[0]) && std::isfinite(t[N - 2]) && t[N - 2] > t[0]) {
    std::vector<double> mags;
    for (uint64_t c = 0; c + 1 < N; ++c) mags.push_back(std::fabs(t[c]));
    std::nth_element(mags.begin(), mags.begin() + mags.size() / 2, mags.end());
    const double scale = std::max(mags[mags.size() / 2] / 0.6745, 1e-300);  // ~ sd of the cells
    uint32_t best = 0;
    std::vector<double> u(N - 1);
    for (double q : {0.0, 0.03, 0.06, 0.1, 0.15, 0.22, 0.3}) {
      const double g = q / (scale * scale);
      for (uint64_t c = 0; c + 1 < N; ++c) u[c] = qt::fmap_g(t[c], g);
      const double u0 = u[0], u1 = u[N - 2];
      if (!(u1 > u0) || !std::isfinite(u1 - u0)) continue;
      // one threshold per bucket needs a bucket width below the smallest gap
      double gap = u1 - u0;
      for (uint64_t c = 1; c + 1 < N; ++c) gap = std::min(gap, u[c] - u[c - 1]);
      if (!(gap > 0.0)) continue;
      double want = std::ceil((u1 - u0) / gap) + 1.0;
      for (int tries = 0; tries < 8 && want <= 8.0 * N; ++tries, want = std::ceil(want * 1.02) + 1) {
        const uint32_t cand = static_cast<uint32_t>(want);
        if (best && cand >= best) break;
        const double a = cand / (u1 - u0), bb = -u0 * a;
        uint32_t prev = 0xFFFFFFFFu, worst = 0, run = 0;
        for (uint64_t c = 0; c + 1 < N; ++c) {
          const uint32_t b = qt::fbucket_host(t[c], g, a, bb, cand - 1);
          run = b == prev ? run + 1 : 1;
          prev = b;
          worst = std::max(worst, run);
        }
        if (worst <= 1) {
          best = cand;
          nb = cand;
          bk_a = a;
          bk_b = bb;
          gc = g;
          break;
        }
      }
    }
    if (!best) {  // no map found: uniform, 8N (records still certify correctly)
      nb = static_cast<uint32_t>(8 * N);
      bk_a = nb / (t[N - 2] - t[0]);
      bk_b = -t[0] * bk_a;
      gc = 0.0;
    }
  }
  h.bk_a = static_cast<float>(bk_a);
  h.bk_b = static_cast<float>(bk_b);
  h.gc = static_cast<float>(gc);
  h.nb1 = nb - 1;
  h.bytes = round16(sizeof(qt::FastHdr) + 16ull * nb);
  std::vector<uint8_t> out(h.bytes, 0);
  std::memcpy(out.data(), &h, sizeof h);
  qt::FRec* R = reinterpret_cast<qt::FRec*>(out.data() + sizeof(qt::FastHdr));
  const float inf = std::numeric_limits<float>::infinity();
  uint64_t c = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    while (c + 1 < N && qt::fbucket_host(t[c], gc, bk_a, bk_b, nb - 1) < b) ++c;
    qt::FRec r;
    r.tl = c ? f32_up(t[c - 1]) : -inf;
    r.t0 = f32_down(t[c]);
    r.t1 = c + 1 < N ? f32_down(t[c + 1]) : inf;
    // sorted positions: the certified counts land in sorted-cell space, where a
    // layer's hits crowd a band around the diagonal (Brownian steps are small
    // against the grid), so the count array's hot lines stay L2-resident
    (void)ord;
    r.o0 = static_cast<uint16_t>(c);
    r.o1 = static_cast<uint16_t>(std::min<uint64_t>(c + 1, N - 1));
    R[b] = r;
  }
  return out;
}

// One layer's table (layout in qt_layout.h). header.cold_off is patched by
// the caller once the cold block's position is known.
// FP32 scan table of one d >= 2 layer (ScanHdr + paired FP32 points), qt_layout.h
// Bucket geometry of one d >= 2 layer's cell-list index (CellHdr,
// qt_layout.h): the box of the points plus a 10 % margin, per N^(1/d)
// buckets per axis (measured on B200: per = 6 for d = 2 (C4: 1.90e10
// transitions/s; 4: 1.72e10, 1.5: 1.15e10), 5 for d = 3 (C5: 4.86e9; 4: 4.31e9,
// 1.2: 8.4e8)). The lists themselves are built on the device
// (qt::build_cell_lists).
qt::CellHdr cell_geometry(int dim, uint64_t N, const double* pts) {
  qt::CellHdr h{};
  for (int c = 0; c < 3; ++c) {
    h.g[c] = 1;
    h.w[c] = 1.0;
  }
  if (dim < 2 || dim > 3 || N < 2 || N > 65535) return h;  // ok = 0: full scan
  double mn[3] = {0, 0, 0}, mx[3] = {0, 0, 0};
  for (int c = 0; c < dim; ++c) {
    mn[c] = std::numeric_limits<double>::infinity();
    mx[c] = -mn[c];
    for (uint64_t i = 0; i < N; ++i) {
      const double v = pts[i * dim + c];
      if (!std::isfinite(v) || std::fabs(v) > 1e100) return h;
      mn[c] = std::min(mn[c], v);
      mx[c] = std::max(mx[c], v);
    }
  }
  double per = 6.0;  // d = 3: 6 measured 5.87e9 at C5 (5: 5.56e9, 7: 5.90e9 with a larger index)
  if (const char* e = std::getenv(dim == 2 ? "QT_CELL_G2" : "QT_CELL_G3")) per = std::atof(e);
  const uint32_t gax = static_cast<uint32_t>(
      std::min(dim == 2 ? 1024.0 : 96.0, std::max(1.0, std::round(per * std::pow(double(N), 1.0 / dim)))));
  for (int c = 0; c < dim; ++c) {
    const double span = mx[c] - mn[c];
    const double pad = span > 0.0 ? 0.1 * span : 0.5;
    h.lo[c] = mn[c] - pad;
    const double hi = mx[c] + pad;
    h.g[c] = span > 0.0 ? gax : 1;
    h.w[c] = (hi - h.lo[c]) / h.g[c];
    h.inv_w[c] = h.g[c] / (hi - h.lo[c]);
    // bucket corners lo + c w must resolve far below the 1e-6 w inflation
    if (!(h.w[c] > 1e-9 * (std::fabs(h.lo[c]) + std::fabs(hi)))) {
      h.ok = 0;
      return h;
    }
  }
  h.ok = 1;
  return h;
}

std::vector<uint8_t> build_scan_table(int dim, uint64_t N, const double* pts, const double* step,
                                      uint64_t joff, uint64_t exact_off) {
  qt::ScanHdr h{};
  std::memcpy(h.step, step, sizeof h.step);
  h.joff = joff;
  h.exact_off = exact_off;
  h.n_pts = static_cast<uint32_t>(N);
  h.n_chunks = static_cast<uint32_t>((N + 2 * qt::kScanChunkPairs - 1) / (2 * qt::kScanChunkPairs));
  const uint64_t npairs = static_cast<uint64_t>(h.n_chunks) * qt::kScanChunkPairs;
  h.off_b = static_cast<uint32_t>(sizeof(qt::ScanHdr) + 16 * npairs);
  h.bytes = round16(h.off_b + (dim == 2 ? 8 : 16) * npairs);
  std::vector<uint8_t> out(h.bytes, 0);
  float* XY = reinterpret_cast<float*>(out.data() + sizeof(qt::ScanHdr));
  float* B = reinterpret_cast<float*>(out.data() + h.off_b);
  const float inf = std::numeric_limits<float>::infinity();
  double hmax = 0.0, pmax[3] = {0.0, 0.0, 0.0};
  bool ok = true;
  for (uint64_t idx = 0; idx < 2 * npairs; ++idx) {
    const uint64_t pr = idx / 2, ln = idx % 2;
    if (idx < N) {
      const double* pp = pts + idx * dim;
      double hh = 0.0;
      for (int c = 0; c < dim; ++c) {
        hh += pp[c] * pp[c];
        pmax[c] = std::max(pmax[c], std::fabs(pp[c]));
        ok = ok && std::fabs(pp[c]) < 0x1p40;
      }
      hh *= 0.5;
      hmax = std::max(hmax, hh);
      XY[4 * pr + ln] = static_cast<float>(pp[0]);
      XY[4 * pr + 2 + ln] = static_cast<float>(pp[1]);
      if (dim == 2) {
        B[2 * pr + ln] = static_cast<float>(hh);
      } else {
        B[4 * pr + ln] = static_cast<float>(pp[2]);
        B[4 * pr + 2 + ln] = static_cast<float>(hh);
      }
    } else {  // padding: p = 0, h = +inf (never a candidate)
      if (dim == 2) B[2 * pr + ln] = inf;
      else B[4 * pr + 2 + ln] = inf;
    }
  }
  h.hmax = f32_up(hmax * (1.0 + 0x1p-50));
  for (int c = 0; c < dim; ++c) h.pmax[c] = f32_up(pmax[c]);
  h.fp32_ok = ok && std::isfinite(h.hmax) ? 1u : 0u;
  std::memcpy(out.data(), &h, sizeof h);
  return out;
}

TableBlob build_table(int kind, int dim, uint64_t npts, const double* pts, const double* step,
                      const double* marg_prev, uint64_t joff, uint64_t n_prev, uint32_t layer) {
  LayerTable h{};
  if (kind == QT_CHAIN_BROWNIAN_1D) {  // x' = x + s eps
    h.fa = 1.0f;
    h.fs = f32_up_abs(step[0]);
  } else if (kind == QT_CHAIN_OU_1D) {  // x' = a x + s eps
    h.fa = f32_up_abs(step[0]);
    h.fs = f32_up_abs(step[2]);
  }
  std::memcpy(h.step, step, sizeof h.step);
  std::memcpy(h.marg_prev, marg_prev, sizeof h.marg_prev);
  h.joff = joff;
  h.n_pts = static_cast<uint32_t>(npts);
  h.n_prev = static_cast<uint32_t>(n_prev);
  h.layer = layer;
  h.dim = static_cast<uint32_t>(dim);
  h.off_rec = sizeof(LayerTable);
  TableBlob out;
  if (dim == 1) {
    std::vector<uint32_t> ord(npts);
    std::iota(ord.begin(), ord.end(), 0u);
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return pts[a] < pts[b]; });
    std::vector<double> v(npts);
    for (uint64_t s = 0; s < npts; ++s) v[s] = pts[ord[s]];
    // x_safe: |x| below it rules out equal d2 between same-side neighbours
    // (gap > 2^-51 (|x| + max|v|) suffices; 8x margin) and d2 overflow.
    double gmin = std::numeric_limits<double>::infinity();
    for (uint64_t s = 1; s < npts; ++s) gmin = std::min(gmin, v[s] - v[s - 1]);
    const double vmax = std::max(std::fabs(v.front()), std::fabs(v.back()));
    double x_safe;
    if (npts == 1) x_safe = vmax <= 1e150 ? 1e150 : 0.0;
    else if (gmin >= 1e-150 && vmax <= 1e150) x_safe = std::min(gmin * 0x1p48 - vmax, 1e150);
    else x_safe = 0.0;
    if (!(x_safe > 0.0) || npts > 65534) x_safe = 0.0;  // exact scan only
    // decision thresholds t_c between sorted c and c+1 (bisection over doubles)
    std::vector<double> t(npts, std::numeric_limits<double>::infinity());
    for (uint64_t c = 0; c + 1 < npts && x_safe > 0.0; ++c) {
      const double vl = v[c], vh = v[c + 1];
      if (choose_hi(vl, vl, vh, ord[c], ord[c + 1]) || !choose_hi(vh, vl, vh, ord[c], ord[c + 1])) {
        x_safe = 0.0;  // degenerate pair: keep the exact scan
        break;
      }
      uint64_t klo = dkey(vl), khi = dkey(vh);
      while (khi - klo > 1) {
        const uint64_t mid = klo + (khi - klo) / 2;
        if (choose_hi(dfromkey(mid), vl, vh, ord[c], ord[c + 1])) khi = mid;
        else klo = mid;
      }
      t[c] = dfromkey(khi);
    }
    // uniform buckets over [t_0, t_{N-2}]; the fewest (multiple of N) that keep
    // one threshold per bucket, else at most two (then a rare one-step walk)
    uint32_t nb = 1;
    double lo = 0.0, inv_w = 0.0;
    if (npts > 2 && x_safe > 0.0) {
      lo = t[0];
      const double span = t[npts - 2] - t[0];
      uint32_t pick2 = 0;
      for (uint32_t m = 1; m <= 8; ++m) {
        const uint32_t cand = static_cast<uint32_t>(m * npts);
        const double iw = static_cast<double>(cand) / span;
        if (!std::isfinite(iw) || !(iw > 0.0)) break;
        uint32_t prev = 0xFFFFFFFFu, run = 0, worst = 0;
        for (uint64_t c = 0; c + 1 < npts; ++c) {
          const uint32_t b = qt::bucket_of(t[c], lo, iw, static_cast<double>(cand), cand);
          run = b == prev ? run + 1 : 1;
          prev = b;
          worst = std::max(worst, run);
        }
        if (worst <= 2 && !pick2) pick2 = cand;
        if (worst <= 1 && m <= 6) {
          nb = cand;
          break;
        }
        if (m == 8) nb = pick2 ? pick2 : cand;
      }
      if (nb > 1) inv_w = static_cast<double>(nb) / span;
      else nb = 1;
    }
    h.lo = lo;
    h.inv_w = inv_w;
    h.cert_c = 0.0f;     // set on the x-tables (make_plan), which know layer k-1
    h.cert_xmax = 0.0f;
    h.x_safe = x_safe;
    h.nb = nb;
    h.nb_d = static_cast<double>(nb);
    h.off_start = round16(h.off_rec + 16ull * (npts + 1));
    h.bytes = round16(h.off_start + 2ull * nb);
    out.hot.assign(h.bytes, 0);
    qt::Thr* T = reinterpret_cast<qt::Thr*>(out.hot.data() + h.off_rec);
    const float ninf = -std::numeric_limits<float>::infinity();
    for (uint64_t c = 0; c < npts; ++c) T[c] = qt::Thr{t[c], ord[c], c ? f32_up(t[c - 1]) : ninf};
    T[npts] = qt::Thr{std::numeric_limits<double>::infinity(), ord[npts - 1],
                      f32_up(t[npts - 1])};
    uint16_t* start = reinterpret_cast<uint16_t*>(out.hot.data() + h.off_start);
    uint64_t c = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      while (c + 1 < npts && qt::bucket_of(t[c], lo, inv_w, h.nb_d, nb) < b) ++c;
      start[b] = static_cast<uint16_t>(std::min<uint64_t>(c, 65535));
    }
    if ((kind == QT_CHAIN_BROWNIAN_1D || kind == QT_CHAIN_OU_1D) && npts <= 65535 &&
        fast_enabled())
      out.fast = build_fast_table(kind, t, ord, x_safe, step, joff);
    out.cold.assign(16ull * npts, 0);
    Rec1* R = reinterpret_cast<Rec1*>(out.cold.data());
    for (uint64_t s = 0; s < npts; ++s) R[s] = Rec1{v[s], ord[s], 0};
  } else {
    h.bytes = round16(h.off_rec + 8ull * dim * npts);
    out.hot.assign(h.bytes, 0);
    std::memcpy(out.hot.data() + h.off_rec, pts, 8ull * dim * npts);
  }
  std::memcpy(out.hot.data(), &h, sizeof h);
  return out;
}

void set_cold_off(std::vector<uint8_t>& hot_table, uint64_t cold_off) {
  LayerTable h;
  std::memcpy(&h, hot_table.data(), sizeof h);
  h.cold_off = cold_off;
  std::memcpy(hot_table.data(), &h, sizeof h);
}

constexpr uint32_t kMaxTableBytes = 110u * 1024u;  // two must fit in 227 KB of smem
constexpr uint32_t kStageBudget = 48u * 1024u;     // shared-memory ring per k_paths CTA
constexpr uint32_t kResidentBudget = 96u * 1024u;

}  // namespace

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct qt_plan {
  int device = 0;
  int kind = 0, dim = 1, nps = 1, n = 0;
  std::vector<uint64_t> sizes, voff, joff;
  uint64_t nvis = 0, njoint = 0, max_cols = 0, max_rows = 0, max_elems = 0;
  std::vector<uint32_t> tab_off, tab_bytes;
  uint32_t max_tab = 0, total_tab = 0, stages = 2;
  bool gmem = false;  // some exact table exceeds kMaxTableBytes
  int sm_count = 148;
  uint8_t* d_tables = nullptr;
  uint32_t* d_tab_off = nullptr;
  uint32_t* d_tab_bytes = nullptr;
  uint64_t* d_fin = nullptr;  // rows, cols, joff, voff_row, voff_col (5 x n)
  std::vector<uint8_t> host_tables;
  // fast 1-D path: replay list + counters (FastArgs::stats), paths sent to it
  qt::AmbEntry* d_amb = nullptr;
  unsigned long long* d_stats = nullptr;
  uint8_t* d_stables = nullptr;  // FP32 scan tables (d >= 2), concatenated
  qt::CellHdr* d_chdr = nullptr;  // cell-list index (d >= 2, qt_cell.cu): headers [n],
  uint32_t* d_cstart = nullptr;   // bucket starts over all layers, and
  uint16_t* d_clist = nullptr;    // the candidate lists
  uint4* d_crec = nullptr;        // bucket records (short lists inline)
  uint32_t* d_stab_off = nullptr;
  uint32_t* d_stab_bytes = nullptr;
  uint32_t max_stab = 0, total_stab = 0;
  uint8_t* d_ftables = nullptr;  // fast-path tables (d == 1), concatenated
  uint32_t* d_ftab_off = nullptr;
  uint32_t* d_ftab_bytes = nullptr;
  uint32_t max_ftab = 0, total_ftab = 0;
  std::vector<uint32_t> ftab_off_h, ftab_bytes_h;
  uint64_t amb_cap = 0, fast_paths = 0;
  // d = 1: k_paths_x tables (threshold pairs), sorted -> original cell index per
  // layer (indexed by voff), and the sorted-cell count scratch (njoint, lazy)
  uint8_t* d_xtables = nullptr;
  uint32_t* d_orig = nullptr;
  unsigned long long* d_sjoint = nullptr;
  // one-call estimate buffers (joint, visits, pi), allocated on first use and
  // kept with the (cached) plan
  uint64_t* d_ojoint = nullptr;
  uint64_t* d_ovis = nullptr;
  double* d_opi = nullptr;

  ~qt_plan() {
    cudaSetDevice(device);
    cudaFree(d_ojoint);
    cudaFree(d_ovis);
    cudaFree(d_opi);
    cudaFree(d_xtables);
    cudaFree(d_orig);
    cudaFree(d_sjoint);
    if (d_stats) {
      unsigned long long st[3] = {0, 0, 0};
      if (cudaMemcpy(st, d_stats, sizeof st, cudaMemcpyDeviceToHost) == cudaSuccess) {
        g_fast_replayed.fetch_add(st[1]);
        g_fast_inline.fetch_add(st[2]);
      }
      g_fast_paths.fetch_add(fast_paths);
    }
    cudaFree(d_amb);
    cudaFree(d_stats);
    cudaFree(d_ftables);
    cudaFree(d_stables);
    cudaFree(d_chdr);
    cudaFree(d_cstart);
    cudaFree(d_clist);
    cudaFree(d_crec);
    cudaFree(d_stab_off);
    cudaFree(d_stab_bytes);
    cudaFree(d_ftab_off);
    cudaFree(d_ftab_bytes);
    cudaFree(d_tables);
    cudaFree(d_tab_off);
    cudaFree(d_tab_bytes);
    cudaFree(d_fin);
  }
};

namespace {

void check_inputs(const qt_chain* chain, const qt_grids* grids) {
  if (!chain || !grids || !grids->sizes || !grids->points || !chain->step || !chain->marginal)
    raise(QT_ERR_INVALID_ARGUMENT, "estimate: null argument");
  const int dim = chain_dim(chain->kind);
  if (grids->layers != chain->layers || chain->layers < 1)
    raise(QT_ERR_INVALID_ARGUMENT, "estimate: need one grid per layer 1..n");
  if (grids->dim != dim) raise(QT_ERR_INVALID_ARGUMENT, "estimate: grid dimension mismatch");
  if (grids->sizes[0] != 1) raise(QT_ERR_INVALID_ARGUMENT, "estimate: layer 0 must be {x0}");
}

qt_plan* make_plan(const qt_chain* chain, const qt_grids* grids, int device) {
  check_inputs(chain, grids);
  auto p = std::make_unique<qt_plan>();
  p->device = device;
  p->kind = chain->kind;
  p->dim = chain_dim(chain->kind);
  p->nps = p->dim;
  p->n = chain->layers;
  const int n = p->n;
  p->sizes.assign(grids->sizes, grids->sizes + n + 1);
  p->voff.assign(n + 2, 0);
  p->joff.assign(n + 1, 0);
  for (int k = 0; k <= n; ++k) p->voff[k + 1] = p->voff[k] + p->sizes[k];
  for (int t = 0; t < n; ++t) {
    p->joff[t + 1] = p->joff[t] + p->sizes[t] * p->sizes[t + 1];
    p->max_cols = std::max(p->max_cols, p->sizes[t + 1]);
    p->max_rows = std::max(p->max_rows, p->sizes[t]);
    p->max_elems = std::max(p->max_elems, p->sizes[t] * p->sizes[t + 1]);
  }
  p->nvis = p->voff[n + 1];
  p->njoint = p->joff[n];
  // tables
  const double* pts = grids->points;
  std::vector<TableBlob> blobs;
  for (int k = 1; k <= n; ++k) {
    const uint64_t N = p->sizes[k];
    if (N == 0 || N > 0xFFFFFFF0ull)
      raise(QT_ERR_NUMERIC, "grid: point data size is not a positive multiple of dim");
    check_grid(p->dim, N, pts, k);
    blobs.push_back(build_table(p->kind, p->dim, N, pts, chain->step + 6 * (k - 1),
                                chain->marginal + 6 * (k - 1), p->joff[k - 1], p->sizes[k - 1],
                                static_cast<uint32_t>(k)));
    const auto& t = blobs.back().hot;
    if (t.size() > kMaxTableBytes) p->gmem = true;  // too big to stage: global-memory kernels
    p->tab_off.push_back(static_cast<uint32_t>(p->host_tables.size()));
    p->tab_bytes.push_back(static_cast<uint32_t>(t.size()));
    p->max_tab = std::max<uint32_t>(p->max_tab, static_cast<uint32_t>(t.size()));
    p->host_tables.insert(p->host_tables.end(), t.begin(), t.end());
    pts += N * p->dim;
  }
  p->total_tab = static_cast<uint32_t>(p->host_tables.size());
  // fast-path tables (every layer must have one)
  std::vector<uint8_t> ftables;
  std::vector<uint32_t> foff, fbytes;
  bool have_fast = true;
  for (const TableBlob& b : blobs) have_fast = have_fast && !b.fast.empty();
  if (have_fast) {
    for (const TableBlob& b : blobs) {
      foff.push_back(static_cast<uint32_t>(ftables.size()));
      fbytes.push_back(static_cast<uint32_t>(b.fast.size()));
      p->max_ftab = std::max<uint32_t>(p->max_ftab, static_cast<uint32_t>(b.fast.size()));
      ftables.insert(ftables.end(), b.fast.begin(), b.fast.end());
    }
    p->total_ftab = static_cast<uint32_t>(ftables.size());
    p->ftab_off_h = foff;
    p->ftab_bytes_h = fbytes;
    if (std::getenv("QT_DEBUG"))
      std::fprintf(stderr, "qtree: fast tables max %u B, total %u B\n", p->max_ftab, p->total_ftab);
  }
  // cold blocks after all hot tables; patch each header's cold_off
  for (int k = 1; k <= n; ++k) {
    TableBlob& b = blobs[k - 1];
    if (b.cold.empty()) continue;
    const uint64_t at = p->host_tables.size();
    std::vector<uint8_t> hot(p->host_tables.begin() + p->tab_off[k - 1],
                             p->host_tables.begin() + p->tab_off[k - 1] + p->tab_bytes[k - 1]);
    set_cold_off(hot, at);
    std::copy(hot.begin(), hot.end(), p->host_tables.begin() + p->tab_off[k - 1]);
    p->host_tables.insert(p->host_tables.end(), b.cold.begin(), b.cold.end());
  }
  p->stages = std::max<uint32_t>(2, std::min<uint32_t>(8, kStageBudget / std::max(p->max_tab, 1u)));
  // d = 1: the k_paths_x copy of the hot tables, Thr[c] -> {t_c, t_c+1}, and the
  // original index of every sorted cell (layer 0 = the singleton {x0})
  std::vector<uint8_t> xtables;
  std::vector<uint32_t> orig;
  if (p->dim == 1) {
    xtables.assign(p->host_tables.begin(), p->host_tables.begin() + p->total_tab);
    orig.assign(p->nvis, 0);
    for (int k = 1; k <= n; ++k) {
      uint8_t* tb = xtables.data() + p->tab_off[k - 1];
      const qt::LayerTable& h = *reinterpret_cast<const qt::LayerTable*>(tb);
      const qt::Thr* T = reinterpret_cast<const qt::Thr*>(
          p->host_tables.data() + p->tab_off[k - 1] + h.off_rec);
      double* PT = reinterpret_cast<double*>(tb + h.off_rec);
      const uint64_t N = p->sizes[k];
      for (uint64_t c = 0; c < N; ++c) {
        orig[p->voff[k] + c] = T[c].orig;
        PT[2 * c] = T[c].t;
        PT[2 * c + 1] = T[c + 1].t;
      }
      PT[2 * N] = PT[2 * N + 1] = std::numeric_limits<double>::infinity();
    }
    // the certified kernel's per-layer state range X_k and rounding term (LayerTable)
    double xprev = 0.0;  // layer 0: the origin
    for (int k = 1; k <= n; ++k) {
      uint8_t* tb = xtables.data() + p->tab_off[k - 1];
      qt::LayerTable& h = *reinterpret_cast<qt::LayerTable*>(tb);
      const double* PT = reinterpret_cast<const double*>(tb + h.off_rec);
      const uint64_t N = p->sizes[k];
      double X = 1e6;  // a single cell takes every state
      if (N >= 2) X = 8.0 * std::max(std::fabs(PT[0]), std::fabs(PT[2 * (N - 2)]));
      X = std::min(X, h.x_safe);
      float xmax = static_cast<float>(X);
      if (static_cast<double>(xmax) > X) xmax = std::nextafter(xmax, 0.0f);
      h.cert_xmax = xmax > 0.0f ? xmax : 0.0f;
      const double mag = static_cast<double>(h.fa) * xprev + static_cast<double>(h.fs) * 6.7 + X;
      h.cert_c = f32_up(mag * 0x1p-50 * (1.0 + 0x1p-30));
      xprev = static_cast<double>(h.cert_xmax);
    }
  }
  // FP32 scan tables (d >= 2)
  std::vector<uint8_t> stables;
  std::vector<uint32_t> soff, sbytes;
  if (p->dim >= 2) {
    const double* sp = grids->points;
    for (int k = 1; k <= n; ++k) {
      const uint64_t N = p->sizes[k];
      auto t = build_scan_table(p->dim, N, sp, chain->step + 6 * (k - 1), p->joff[k - 1],
                                p->tab_off[k - 1]);
      soff.push_back(static_cast<uint32_t>(stables.size()));
      sbytes.push_back(static_cast<uint32_t>(t.size()));
      p->max_stab = std::max<uint32_t>(p->max_stab, static_cast<uint32_t>(t.size()));
      stables.insert(stables.end(), t.begin(), t.end());
      sp += N * p->dim;
    }
    p->total_stab = static_cast<uint32_t>(stables.size());
  }
  // cell-list geometry (d >= 2); the lists are built on the device below
  std::vector<qt::CellHdr> chdr;
  if (p->dim >= 2 && cell_enabled()) {
    const double* sp = grids->points;
    uint64_t off = 0;
    for (int k = 1; k <= n; ++k) {
      qt::CellHdr h = cell_geometry(p->dim, p->sizes[k], sp);
      h.start_off = off;
      off += static_cast<uint64_t>(h.g[0]) * h.g[1] * h.g[2];
      chdr.push_back(h);
      sp += p->sizes[k] * p->dim;
    }
  }
  QT_CUDA(cudaSetDevice(device));
  QT_CUDA(cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, device));
  QT_CUDA(cudaMalloc(&p->d_tables, p->host_tables.size()));
  QT_CUDA(cudaMemcpy(p->d_tables, p->host_tables.data(), p->host_tables.size(),
                     cudaMemcpyHostToDevice));
  if (!stables.empty() && p->max_stab <= kMaxTableBytes) {
    QT_CUDA(cudaMalloc(&p->d_stables, stables.size()));
    QT_CUDA(cudaMemcpy(p->d_stables, stables.data(), stables.size(), cudaMemcpyHostToDevice));
    QT_CUDA(cudaMalloc(&p->d_stab_off, n * sizeof(uint32_t)));
    QT_CUDA(cudaMalloc(&p->d_stab_bytes, n * sizeof(uint32_t)));
    QT_CUDA(cudaMemcpy(p->d_stab_off, soff.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    QT_CUDA(cudaMemcpy(p->d_stab_bytes, sbytes.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
  }
  if (have_fast && p->max_ftab <= kMaxTableBytes) {
    QT_CUDA(cudaMalloc(&p->d_ftables, ftables.size()));
    QT_CUDA(cudaMemcpy(p->d_ftables, ftables.data(), ftables.size(), cudaMemcpyHostToDevice));
    QT_CUDA(cudaMalloc(&p->d_ftab_off, n * sizeof(uint32_t)));
    QT_CUDA(cudaMalloc(&p->d_ftab_bytes, n * sizeof(uint32_t)));
    QT_CUDA(cudaMemcpy(p->d_ftab_off, foff.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    QT_CUDA(cudaMemcpy(p->d_ftab_bytes, fbytes.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
  }
  if (!xtables.empty()) {
    QT_CUDA(cudaMalloc(&p->d_xtables, xtables.size()));
    QT_CUDA(cudaMemcpy(p->d_xtables, xtables.data(), xtables.size(), cudaMemcpyHostToDevice));
    QT_CUDA(cudaMalloc(&p->d_orig, orig.size() * sizeof(uint32_t)));
    QT_CUDA(cudaMemcpy(p->d_orig, orig.data(), orig.size() * sizeof(uint32_t),
                       cudaMemcpyHostToDevice));
  }
  QT_CUDA(cudaMalloc(&p->d_tab_off, n * sizeof(uint32_t)));
  QT_CUDA(cudaMalloc(&p->d_tab_bytes, n * sizeof(uint32_t)));
  QT_CUDA(cudaMemcpy(p->d_tab_off, p->tab_off.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
  QT_CUDA(cudaMemcpy(p->d_tab_bytes, p->tab_bytes.data(), n * sizeof(uint32_t),
                     cudaMemcpyHostToDevice));
  if (!chdr.empty()) {
    std::vector<uint64_t> pts_off(n);
    for (int k = 1; k <= n; ++k) {
      const qt::LayerTable& lt =
          *reinterpret_cast<const qt::LayerTable*>(p->host_tables.data() + p->tab_off[k - 1]);
      pts_off[k - 1] = p->tab_off[k - 1] + lt.off_rec;
    }
    uint64_t total = 0;
    // inline bucket records: d = 2 lists are short (C4: <= 6 candidates) and the
    // record saves one dependent load (C4 3.0e10 vs 2.33e10); d = 3 lists mostly
    // overflow the 7 slots (C5 5.37e9 vs 5.55e9 without). QT_CELL_REC=0/1 overrides.
    bool recs = p->dim == 2;
    if (const char* e = std::getenv("QT_CELL_REC")) recs = e[0] != '0';
    QT_CUDA(qt::build_cell_lists(p->dim, n, chdr.data(), p->sizes.data() + 1, p->d_tables,
                                 pts_off.data(), &p->d_chdr, &p->d_cstart, &p->d_clist,
                                 recs ? &p->d_crec : nullptr, &total));
    g_launches.fetch_add(2ull * n + 1);
  }
  std::vector<uint64_t> fin(5 * n);
  for (int t = 0; t < n; ++t) {
    fin[t] = p->sizes[t];
    fin[n + t] = p->sizes[t + 1];
    fin[2 * n + t] = p->joff[t];
    fin[3 * n + t] = p->voff[t];
    fin[4 * n + t] = p->voff[t + 1];
  }
  QT_CUDA(cudaMalloc(&p->d_fin, fin.size() * sizeof(uint64_t)));
  QT_CUDA(cudaMemcpy(p->d_fin, fin.data(), fin.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  device_tables(device);
  return p.release();
}

// Plans of recent one-call estimates, keyed by every input make_plan reads
// (chain kind and coefficients, grid sizes and points, device), so a repeated qt_estimate on the same grids skips the host table
// build and uploads. A call takes its plan out of the cache (exclusive use:
// the sorted-cell scratch is per plan) and returns it afterwards; at most
// kPlanCacheSize plans are kept. Leaked at exit on purpose (no CUDA calls from
// static destructors).
constexpr size_t kPlanCacheSize = 2;
struct PlanCache {
  std::mutex mu;
  std::vector<std::pair<std::vector<uint8_t>, std::unique_ptr<qt_plan>>> items;
};
PlanCache& plan_cache() {
  static PlanCache* c = new PlanCache;
  return *c;
}
std::vector<uint8_t> plan_key(const qt_chain* chain, const qt_grids* grids, int device) {
  std::vector<uint8_t> k;
  auto put = [&](const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    k.insert(k.end(), b, b + n);
  };
  const int32_t hdr[6] = {chain->kind, chain->layers, grids->dim, device, mode1d(),
                          cell_enabled() ? 1 : 0};
  put(hdr, sizeof hdr);
  const size_t n = static_cast<size_t>(chain->layers);
  put(chain->step, 6 * n * sizeof(double));
  put(chain->marginal, 6 * n * sizeof(double));
  put(grids->sizes, (n + 1) * sizeof(uint64_t));
  uint64_t pts = 0;
  for (size_t i = 1; i <= n; ++i) pts += grids->sizes[i];
  put(grids->points, pts * static_cast<size_t>(grids->dim) * sizeof(double));
  return k;
}
std::unique_ptr<qt_plan> take_plan(const std::vector<uint8_t>& key, const qt_chain* chain,
                                   const qt_grids* grids, int device) {
  {
    PlanCache& c = plan_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    for (size_t i = 0; i < c.items.size(); ++i)
      if (c.items[i].first == key) {
        std::unique_ptr<qt_plan> p = std::move(c.items[i].second);
        c.items.erase(c.items.begin() + static_cast<std::ptrdiff_t>(i));
        return p;
      }
  }
  return std::unique_ptr<qt_plan>(make_plan(chain, grids, device));
}
void give_plan(std::vector<uint8_t> key, std::unique_ptr<qt_plan> p, size_t keep) {
  if (const char* e = std::getenv("QT_PLAN_CACHE"); e && e[0] == '0') return;
  PlanCache& c = plan_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.items.emplace_back(std::move(key), std::move(p));
  while (c.items.size() > std::max(kPlanCacheSize, keep)) c.items.erase(c.items.begin());
}

int source_of(int engine, bool normals_in) {
  if (normals_in) return 3;
  if (engine < 0 || engine > 2) raise(QT_ERR_INVALID_ARGUMENT, "unknown engine kind");
  return engine;
}

// Enqueue the count kernel(s) for units [first, first+count).
int plan_count(qt_plan* p, int alg, int engine, uint64_t seed, uint64_t first, uint64_t count,
               uint64_t total, const double* d_normals, uint64_t* d_joint, cudaStream_t st) {
  if (alg < QT_ALG_I || alg > QT_ALG_III)
    raise(QT_ERR_INVALID_ARGUMENT, "estimate: unknown estimator kind");
  if (count == 0) return 0;
  QT_CUDA(cudaSetDevice(p->device));
  const int src = source_of(engine, d_normals != nullptr);
  int extra = 0;  // launches besides the count kernel
  if (alg != QT_ALG_III) {
    const uint64_t normals = static_cast<uint64_t>(p->n) * p->nps;
    qt::PathArgs a{};
    a.src = make_src(p->device, engine, seed, 2 * ((normals + 1) / 2),
                     static_cast<uint32_t>(normals), d_normals, first);
    a.tables = p->d_tables;
    a.tab_off = p->d_tab_off;
    a.tab_bytes = p->d_tab_bytes;
    a.joint = reinterpret_cast<unsigned long long*>(d_joint);
    a.first = first;
    a.n = static_cast<uint32_t>(p->n);
    a.buf_bytes = p->max_tab;
    a.resident_bytes = p->total_tab;
    a.stages = p->stages;
    a.layers_per_stage = 1;
    const bool resident = p->total_tab <= kResidentBudget;
    const size_t smem = resident ? p->total_tab : static_cast<size_t>(p->stages) * p->max_tab;
    const bool fast = fast_enabled() && src == QT_ENGINE_MRG32K3A && p->d_ftables && p->d_orig &&
                      (p->kind == QT_CHAIN_BROWNIAN_1D || p->kind == QT_CHAIN_OU_1D) &&
                      p->n < 65536 && first + count <= (1ull << 48);
    if (fast) {
      // replay list: room for 1/8 of the window (ambiguous paths are a few %;
      // an overflow is still exact, replayed inline by the path kernel)
      uint64_t want = std::max<uint64_t>(1u << 16, count / 8 + 1);
      if (const char* cap = std::getenv("QT_FAST_REPLAY_CAP"))  // test hook: force overflow
        want = std::max<uint64_t>(1, std::strtoull(cap, nullptr, 10));
      if (!p->d_stats) {
        QT_CUDA(cudaMalloc(&p->d_stats, 3 * sizeof(unsigned long long)));
        QT_CUDA(cudaMemset(p->d_stats, 0, 3 * sizeof(unsigned long long)));
      }
      if (p->amb_cap < want || std::getenv("QT_FAST_REPLAY_CAP")) {
        QT_CUDA(cudaFree(p->d_amb));
        p->d_amb = nullptr;
        p->amb_cap = 0;
        QT_CUDA(cudaMalloc(&p->d_amb, want * sizeof(qt::AmbEntry)));
        p->amb_cap = want;
      }
      int P = 4;  // paths in flight per thread (QT_FAST_P = 1 / 2 / 4)
      if (const char* e = std::getenv("QT_FAST_P")) P = std::atoi(e) == 1 ? 1 : std::atoi(e) == 2 ? 2 : 4;
      // fast tables: all resident when they fit, else prefetched S layers ahead
      const bool fres = p->total_ftab <= kResidentBudget;
      // stages of one or two layers (two: the pair of one Box-Muller draw); one
      // measured faster at C2 (1.187e11 vs 1.119e11, profiles/r02_c2_variant_sweeps.txt)
      uint32_t fl = 1;
      if (const char* e = std::getenv("QT_FAST_L")) fl = std::atoi(e) == 1 ? 1u : 2u;
      uint32_t fbuf = p->max_ftab;
      if (fl == 2)
        for (int k = 0; k < p->n; k += 2) {
          const int k1 = std::min(k + 1, p->n - 1);
          fbuf = std::max<uint32_t>(fbuf, p->ftab_off_h[k1] + p->ftab_bytes_h[k1] - p->ftab_off_h[k]);
        }
      uint32_t st_n = 2;
      if (const char* e = std::getenv("QT_FAST_STAGES")) st_n = std::max(2, std::min(8, std::atoi(e)));
      const size_t fsmem = fres ? p->total_ftab : static_cast<size_t>(st_n) * fbuf;
      qt::PathArgs fa_args = a;
      const int bps = qt::paths_fast_blocks_per_sm(p->kind, fres, P, fsmem);
      uint64_t blocks = static_cast<uint64_t>(p->sm_count) * bps;
      const uint64_t slots_per_block = static_cast<uint64_t>(qt::kPathConsumers) * P;
      const uint64_t need = (count + slots_per_block - 1) / slots_per_block;
      if (need < blocks) blocks = need;
      const uint64_t T = blocks * slots_per_block;
      fa_args.q = count / T;
      fa_args.rem = count % T;
      if (!p->d_sjoint) QT_CUDA(cudaMalloc(&p->d_sjoint, p->njoint * sizeof(uint64_t)));
      QT_CUDA(cudaMemsetAsync(p->d_sjoint, 0, p->njoint * sizeof(uint64_t), st));
      qt::FastArgs fa{fa_args, p->d_amb, p->d_stats, std::min(p->amb_cap, want),
                      p->d_ftables, p->d_ftab_off, p->d_ftab_bytes, fbuf, p->total_ftab,
                      st_n, {}, std::getenv("QT_PROBE_NORED") ? 1u : 0u, p->d_sjoint, fl};
      mrg_back_jump(2 * ((static_cast<uint64_t>(p->n) + 1) / 2), fa.back);
      QT_CUDA(cudaMemsetAsync(p->d_stats, 0, sizeof(unsigned long long), st));
      QT_CUDA(qt::launch_paths_fast(p->kind, fres, P, fa, static_cast<uint32_t>(blocks), fsmem,
                                    static_cast<uint32_t>(p->sm_count) * 4u, st));
      QT_CUDA(qt::launch_permute_add(p->d_sjoint, reinterpret_cast<unsigned long long*>(d_joint),
                                     p->d_fin, p->d_orig, static_cast<uint32_t>(p->n),
                                     p->max_elems, st));
      p->fast_paths += count;
      g_launches.fetch_add(3);
      return 3;
    }
    if (src == QT_ENGINE_MRG32K3A && (p->kind == QT_CHAIN_BROWNIAN_1D || p->kind == QT_CHAIN_OU_1D) &&
        xkernel_enabled() && !p->gmem && p->d_xtables) {  // 1-D MRG32k3a: the lockstep exact kernel
      // counts go to the plan's sorted-cell scratch, then are permute-added into
      // d_joint (calls on one plan are ordered by their streams: one scratch)
      if (!p->d_sjoint) QT_CUDA(cudaMalloc(&p->d_sjoint, p->njoint * sizeof(uint64_t)));
      QT_CUDA(cudaMemsetAsync(p->d_sjoint, 0, p->njoint * sizeof(uint64_t), st));
      // paths in flight per thread: 2 (C2 1.33e11 vs 1.06e11 with 1); 1 when every
      // thread slot would run only a few paths (C1, 7 rounds: 1.05e11 vs 9.9e10 with 2)
      int P = count < static_cast<uint64_t>(p->sm_count) * 2 * qt::kXThreads * 2 * 64 ? 1 : 2;
      if (const char* e = std::getenv("QT_X_P")) P = std::atoi(e) == 1 ? 1 : std::atoi(e) == 4 ? 4 : 2;
      qt::PathArgs xa = a;
      // layers per pipeline stage (1 or 2)
      uint32_t Lp = 2;
      if (const char* e = std::getenv("QT_X_L")) Lp = std::atoi(e) == 1 ? 1u : 2u;
      uint32_t buf = p->max_tab;
      if (Lp == 2)
        for (int k = 0; k < p->n; k += 2) {
          const int k1 = std::min(k + 1, p->n - 1);
          buf = std::max<uint32_t>(buf, p->tab_off[k1] + p->tab_bytes[k1] - p->tab_off[k]);
        }
      if (Lp == 2 && 2ull * buf > 200u * 1024u) {  // two-layer stages do not fit: one layer
        Lp = 1;
        buf = p->max_tab;
      }
      xa.layers_per_stage = Lp;
      xa.buf_bytes = buf;
      xa.stages = Lp == 2 ? 2u : (3u * p->max_tab <= 150u * 1024u ? 3u : 2u);
      if (const char* e = std::getenv("QT_X_S")) xa.stages = std::max(2, std::min(8, std::atoi(e)));
      xa.probe_nored = std::getenv("QT_PROBE_NORED") ? 1u : 0u;
      const bool cert = cert_enabled() && first + count <= (1ull << 48) && p->n < 65536;
      if (cert) {  // the replay list: a certified path is rarely ambiguous (~1e-9)
        const uint64_t want = std::max<uint64_t>(1u << 16, count / 1024 + 1);
        if (!p->d_stats) {
          QT_CUDA(cudaMalloc(&p->d_stats, 3 * sizeof(unsigned long long)));
          QT_CUDA(cudaMemset(p->d_stats, 0, 3 * sizeof(unsigned long long)));
        }
        if (p->amb_cap < want) {
          QT_CUDA(cudaFree(p->d_amb));
          p->d_amb = nullptr;
          p->amb_cap = 0;
          QT_CUDA(cudaMalloc(&p->d_amb, want * sizeof(qt::AmbEntry)));
          p->amb_cap = want;
        }
        QT_CUDA(cudaMemsetAsync(p->d_stats, 0, sizeof(unsigned long long), st));
        xa.amb = p->d_amb;
        xa.stats = p->d_stats;
        xa.amb_cap = p->amb_cap;
        xa.ojoint = reinterpret_cast<unsigned long long*>(d_joint);
        mrg_back_jump(2 * ((static_cast<uint64_t>(p->n) + 1) / 2), xa.back);
      }
      size_t xsmem = resident ? p->total_tab : static_cast<size_t>(xa.stages) * buf;
      // the first transition's single row (x0 -> N_1 cells: every path hits it) is
      // counted per CTA in shared memory: at C1 the row takes 1e6 REDs on 7 L2 lines
      xa.n1 = 0;
      const char* h1 = std::getenv("QT_X_HIST1");
      if (!(h1 && h1[0] == '0') && p->sizes[1] <= 16384) {
        xa.hist1_off = static_cast<uint32_t>((xsmem + 15) & ~size_t(15));
        xa.n1 = static_cast<uint32_t>(p->sizes[1]);
        xsmem = xa.hist1_off + 4ull * xa.n1;
      }
      int xbps = 1;
      QT_CUDA(qt::launch_paths_x(p->kind, resident, P, cert, xa, 0, xsmem, st, &xbps));
      uint64_t xblocks = static_cast<uint64_t>(p->sm_count) * xbps;
      const uint64_t per_block = static_cast<uint64_t>(qt::kXThreads) * P;
      const uint64_t xneed = (count + per_block - 1) / per_block;
      if (xneed < xblocks) xblocks = xneed;
      const uint64_t T = xblocks * per_block;
      xa.q = count / T;
      xa.rem = count % T;
      if ((xa.q + 1) * per_block >= (1ull << 31)) xa.n1 = 0;  // u32 per-CTA counters
      xa.joint = p->d_sjoint;
      xa.xtables = p->d_xtables;
      QT_CUDA(qt::launch_paths_x(p->kind, resident, P, cert, xa, static_cast<uint32_t>(xblocks),
                                 xsmem, st, nullptr));
      QT_CUDA(qt::launch_permute_add(p->d_sjoint, reinterpret_cast<unsigned long long*>(d_joint),
                                     p->d_fin, p->d_orig, static_cast<uint32_t>(p->n),
                                     p->max_elems, st));
      if (cert) {  // the exact replay of the uncertified paths, into the original-index counts
        qt::FastArgs fr{};
        fr.p = xa;
        fr.p.joint = reinterpret_cast<unsigned long long*>(d_joint);
        fr.amb = p->d_amb;
        fr.stats = p->d_stats;
        fr.cap = p->amb_cap;
        QT_CUDA(qt::launch_replay(p->kind, fr, static_cast<uint32_t>(p->sm_count) * 4u, st));
        p->fast_paths += count;
        g_launches.fetch_add(3);
        return 3;
      }
      g_launches.fetch_add(2);
      return 2;
    }
    if (p->d_chdr && cell_enabled()) {  // d >= 2: exact cell-list search (qt_cell.cu)
      // paths per thread: 2 for d = 2 (C4 2.36e10 vs 2.17e10), 1 for d = 3 (C5 5.55e9 vs 4.43e9)
      int P = p->dim == 3 ? 1 : 2;
      if (const char* e = std::getenv("QT_CELL_P")) P = std::atoi(e) == 1 ? 1 : 2;
      const int cbps = qt::paths_cell_blocks_per_sm(p->kind, src, P);
      uint64_t cblocks = static_cast<uint64_t>(p->sm_count) * cbps;
      const uint64_t per_block = 256ull * P;  // kCellThreads
      const uint64_t cneed = (count + per_block - 1) / per_block;
      if (cneed < cblocks) cblocks = cneed;
      const uint64_t T = cblocks * per_block;
      qt::CellArgs ca{a, p->d_chdr, p->d_cstart, p->d_clist, p->d_crec};
      ca.p.q = count / T;
      ca.p.rem = count % T;
      QT_CUDA(qt::launch_paths_cell(p->kind, src, P, ca, static_cast<uint32_t>(cblocks), st));
      g_launches.fetch_add(1);
      return 1;
    }
    if (p->d_stables && scan_enabled()) {  // d >= 2: FP32 scan + exact FP64 decision
      // queries per thread: d = 2 keeps two CTAs per SM at P = 2; d = 3 is one
      // CTA per SM anyway (64 KB tables), where P = 4 gives the ILP
      // queries per thread: 2 (d = 2: three 256-thread CTAs per SM; d = 3: one
      // 512-thread CTA per SM, the 64 KB tables allow no more)
      int P = 2;
      if (const char* e = std::getenv("QT_SCAN_P")) P = std::atoi(e) == 1 ? 1 : std::atoi(e) == 2 ? 2 : 4;
      const uint64_t nt = p->dim == 3 ? 512 : 256;  // scan_threads<K>() in qt_scan.cu
      const bool sres = p->total_stab <= kResidentBudget;
      const uint32_t S = 3u * p->max_stab <= 200u * 1024u ? 3u : 2u;
      const size_t ssmem = sres ? p->total_stab : static_cast<size_t>(S) * p->max_stab;
      const int sbps = qt::paths_scan_blocks_per_sm(p->kind, src, sres, P, ssmem);
      uint64_t sblocks = static_cast<uint64_t>(p->sm_count) * sbps;
      const uint64_t per_block = nt * P;
      const uint64_t sneed = (count + per_block - 1) / per_block;
      if (sneed < sblocks) sblocks = sneed;
      const uint64_t T = sblocks * per_block;
      qt::ScanArgs sa{a, p->d_stables, p->d_stab_off, p->d_stab_bytes, p->max_stab, p->total_stab, S};
      sa.p.q = count / T;
      sa.p.rem = count % T;
      QT_CUDA(qt::launch_paths_scan(p->kind, src, sres, P, sa, static_cast<uint32_t>(sblocks), ssmem, st));
      g_launches.fetch_add(1);
      return 1;
    }
    if (p->gmem) {  // tables too large to stage: read them from global memory
      uint64_t gblocks = static_cast<uint64_t>(p->sm_count) * 8;
      const uint64_t gneed = (count + 255) / 256;
      if (gneed < gblocks) gblocks = gneed;
      const uint64_t T = gblocks * 256;
      a.q = count / T;
      a.rem = count % T;
      QT_CUDA(qt::launch_gmem(p->kind, src, false, a, qt::Alg3Args{}, static_cast<uint32_t>(gblocks), st));
      g_launches.fetch_add(1);
      return 1;
    }
    const int bps = qt::paths_blocks_per_sm(p->kind, src, resident, smem);
    uint64_t blocks = static_cast<uint64_t>(p->sm_count) * bps;
    const uint64_t need = (count + qt::kPathConsumers - 1) / qt::kPathConsumers;
    if (need < blocks) blocks = need;
    const uint64_t T = blocks * qt::kPathConsumers;
    a.q = count / T;
    a.rem = count % T;
    QT_CUDA(qt::launch_paths(p->kind, src, resident, a, static_cast<uint32_t>(blocks), smem, st));
  } else {
    if (total % p->n != 0) raise(QT_ERR_INVALID_ARGUMENT, "Alg III: total must be n * M");
    const uint64_t M = total / p->n;
    qt::Alg3Args a{};
    const uint64_t normals = static_cast<uint64_t>(p->dim) + p->nps;
    a.src = make_src(p->device, engine, seed, 2 * ((normals + 1) / 2),
                     static_cast<uint32_t>(normals), d_normals, first);
    a.tables = p->d_tables;
    a.tab_off = p->d_tab_off;
    a.tab_bytes = p->d_tab_bytes;
    a.joint = reinterpret_cast<unsigned long long*>(d_joint);
    a.M = M;
    a.first = first;
    a.count = count;
    a.n = static_cast<uint32_t>(p->n);
    a.buf_bytes = p->max_tab;
    a.probe_nored = std::getenv("QT_PROBE_NORED") ? 1u : 0u;
    const size_t smem = 2ull * p->max_tab;
    // slices per layer: ~8 waves of resident CTAs overall, >= 64 samples per thread
    uint64_t slices = std::max<uint64_t>(1, (static_cast<uint64_t>(p->sm_count) * 32) / p->n);
    const uint64_t cap = std::max<uint64_t>(1, M / (256 * 64));
    slices = std::min(slices, cap);
    slices = std::min<uint64_t>(slices, 1u << 30);
    if (src == QT_ENGINE_MRG32K3A && (p->kind == QT_CHAIN_BROWNIAN_1D || p->kind == QT_CHAIN_OU_1D) &&
        xkernel_enabled() && !p->gmem && p->d_xtables) {
      int P = 1;  // measured best for C3 (exact: P = 1; certified: P = 1 8.24e10 vs P = 2 7.93e10)
      if (const char* e = std::getenv("QT_X_P")) P = std::atoi(e) == 2 ? 2 : std::atoi(e) == 4 ? 4 : 1;
      // sorted-cell counts into the plan's scratch, then permute-added (as k_paths_x)
      if (!p->d_sjoint) QT_CUDA(cudaMalloc(&p->d_sjoint, p->njoint * sizeof(uint64_t)));
      QT_CUDA(cudaMemsetAsync(p->d_sjoint, 0, p->njoint * sizeof(uint64_t), st));
      a.joint = p->d_sjoint;
      a.xtables = p->d_xtables;
      const bool cert = cert_enabled() && first + count <= (1ull << 48) && p->n < 65536;
      if (cert) {  // uncertified samples -> k_replay3 (none expected at C3)
        const uint64_t want = std::max<uint64_t>(1u << 16, count / 1024 + 1);
        if (!p->d_stats) {
          QT_CUDA(cudaMalloc(&p->d_stats, 3 * sizeof(unsigned long long)));
          QT_CUDA(cudaMemset(p->d_stats, 0, 3 * sizeof(unsigned long long)));
        }
        if (p->amb_cap < want) {
          QT_CUDA(cudaFree(p->d_amb));
          p->d_amb = nullptr;
          p->amb_cap = 0;
          QT_CUDA(cudaMalloc(&p->d_amb, want * sizeof(qt::AmbEntry)));
          p->amb_cap = want;
        }
        QT_CUDA(cudaMemsetAsync(p->d_stats, 0, sizeof(unsigned long long), st));
        a.amb = p->d_amb;
        a.stats = p->d_stats;
        a.amb_cap = p->amb_cap;
        a.ojoint = reinterpret_cast<unsigned long long*>(d_joint);
        mrg_back_jump(2, a.back2);
        if (P == 4) P = 2;
      }
      // the layer's counts privatised in a shared-memory tile when it fits
      // (QT_A3_PRIV=0: one L2 RED per sample instead; C3 8.47e10 vs 8.24e10 samples/s).
      // One 1024-thread CTA per SM; slices per layer chosen so the n * slices CTAs fill
      // whole waves (C3: 2 slices = 730 CTAs = 4.93 waves of 148)
      size_t xsmem = smem;
      const char* pe = std::getenv("QT_A3_PRIV");
      if (!(pe && std::atoi(pe) == 0)) {
        uint64_t tile = 0;
        for (size_t k = 1; k < p->sizes.size(); ++k) tile = std::max<uint64_t>(tile, p->sizes[k - 1] * p->sizes[k] * 4);
        const double sm = static_cast<double>(p->sm_count);
        uint64_t ps = 1;
        double best = 1e300;
        for (uint64_t s = 1; s <= 8; ++s) {
          const double w = static_cast<double>(s * p->n) / sm;
          const double loss = std::ceil(w) / w;
          if (loss < best - 1e-3) best = loss, ps = s;
        }
        if (const char* e2 = std::getenv("QT_A3_SLICES")) ps = std::max<uint64_t>(1, std::atoll(e2));
        ps = std::min<uint64_t>(ps, std::max<uint64_t>(1, M / (1024 * 64)));
        if (smem + tile <= 200 * 1024 && M / ps < (1ull << 31)) {
          a.priv_bytes = static_cast<uint32_t>(tile);
          xsmem = smem + tile;
          slices = ps;
        }
      }
      QT_CUDA(qt::launch_alg3_x(p->kind, P, cert, a, static_cast<uint32_t>(slices), xsmem, st));
      QT_CUDA(qt::launch_permute_add(p->d_sjoint, reinterpret_cast<unsigned long long*>(d_joint),
                                     p->d_fin, p->d_orig, static_cast<uint32_t>(p->n),
                                     p->max_elems, st));
      g_launches.fetch_add(1);
      extra = 1;
      if (cert) {
        QT_CUDA(qt::launch_replay3(p->kind, a, static_cast<uint32_t>(p->sm_count) * 4u, st));
        g_launches.fetch_add(1);
        extra = 2;
      }
    } else if (p->d_chdr && cell_enabled()) {  // d >= 2: exact cell-list search
      qt::Alg3CellArgs ca{a, p->d_chdr, p->d_cstart, p->d_clist, p->d_crec};
      QT_CUDA(qt::launch_alg3_cell(p->kind, src, ca, static_cast<uint32_t>(slices), st));
    } else if (p->d_stables && scan_enabled() && 2ull * p->max_stab <= 200u * 1024u) {
      qt::Alg3ScanArgs sa{a, p->d_stables, p->d_stab_off, p->d_stab_bytes, p->max_stab};
      QT_CUDA(qt::launch_alg3_scan(p->kind, src, sa, static_cast<uint32_t>(slices),
                                   2ull * p->max_stab, st));
    } else if (p->gmem) {  // tables too large to stage: read them from global memory
      const uint64_t gneed = (count + 255) / 256;
      const uint64_t gblocks = std::min<uint64_t>(gneed, static_cast<uint64_t>(p->sm_count) * 8);
      QT_CUDA(qt::launch_gmem(p->kind, src, true, qt::PathArgs{}, a, static_cast<uint32_t>(gblocks), st));
    } else {
      QT_CUDA(qt::launch_alg3(p->kind, src, a, static_cast<uint32_t>(slices), smem, st));
    }
  }
  g_launches.fetch_add(1);
  return 1 + extra;
}

int plan_finalize(qt_plan* p, int alg, uint64_t samples, const uint64_t* d_joint, uint64_t* d_visits,
                  double* d_pi, cudaStream_t st) {
  QT_CUDA(cudaSetDevice(p->device));
  const int n = p->n;
  qt::FinalizeArgs f{p->d_fin, p->d_fin + n, p->d_fin + 2 * n, p->d_fin + 3 * n, p->d_fin + 4 * n};
  int l = 0;
  QT_CUDA(qt::launch_finalize(alg == QT_ALG_III, reinterpret_cast<const unsigned long long*>(d_joint),
                              reinterpret_cast<unsigned long long*>(d_visits), d_pi, samples, f,
                              static_cast<uint32_t>(n), p->max_cols, p->max_rows, p->max_elems, st,
                              &l));
  g_launches.fetch_add(static_cast<uint64_t>(l));
  return l;
}

// ---------------------------------------------------------------------------
// NCCL, loaded on demand (only multi-device calls need it)
// ---------------------------------------------------------------------------
struct Nccl {
  typedef int (*InitAll)(void** comms, int ndev, const int* devlist);
  typedef int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*Group)();
  typedef int (*Destroy)(void*);
  typedef const char* (*ErrStr)(int);
  InitAll init_all = nullptr;
  AllReduce all_reduce = nullptr;
  Group group_start = nullptr, group_end = nullptr;
  Destroy destroy = nullptr;
  ErrStr err = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.init_all = reinterpret_cast<Nccl::InitAll>(dlsym(h, "ncclCommInitAll"));
    n.all_reduce = reinterpret_cast<Nccl::AllReduce>(dlsym(h, "ncclAllReduce"));
    n.group_start = reinterpret_cast<Nccl::Group>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<Nccl::Group>(dlsym(h, "ncclGroupEnd"));
    n.destroy = reinterpret_cast<Nccl::Destroy>(dlsym(h, "ncclCommDestroy"));
    n.err = reinterpret_cast<Nccl::ErrStr>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.init_all && n.all_reduce && n.group_start && n.group_end && n.destroy;
  });
  return n;
}
// One communicator clique per device range (first device, count), created on
// first use and kept (ncclCommInitAll costs far more than a C2-sized
// all-reduce); calls that use the same clique are serialised by its mutex. A
// clique whose collective failed is destroyed and re-created by the next call.
// Never destroyed otherwise (process exit).
struct NcclClique {
  std::mutex mu;
  std::vector<void*> comms;
};
NcclClique& nccl_clique(int base, int G) {
  static std::mutex m;
  static std::map<std::pair<int, int>, std::unique_ptr<NcclClique>>* cliques =
      new std::map<std::pair<int, int>, std::unique_ptr<NcclClique>>;
  std::lock_guard<std::mutex> lk(m);
  auto& c = (*cliques)[{base, G}];
  if (!c) c = std::make_unique<NcclClique>();
  return *c;
}
constexpr int kNcclUint64 = 5;  // ncclUint64
constexpr int kNcclSum = 0;     // ncclSum

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Map the pages of host output buffers while the GPU computes: fresh arrays
// (calloc / np.zeros) are lazily mapped, and faulting 100s of MB in during the
// device->host copy costs more than the copy. MADV_POPULATE_WRITE (Linux 5.14)
// maps without changing the contents; without it, one byte per page is
// rewritten with its own value (the buffers are pure outputs of the call).
class Prefault {
 public:
  void add(void* p, size_t bytes) {
    if (p && bytes >= (1u << 20)) spans_.push_back({static_cast<char*>(p), bytes});
  }
  void start() {
    size_t total = 0;
    for (const auto& s : spans_) total += s.second;
    if (total == 0) return;
    const int nt = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, total >> 24)));
    for (int t = 0; t < nt; ++t)
      threads_.emplace_back([this, t, nt] {
        const size_t pg = static_cast<size_t>(sysconf(_SC_PAGESIZE));
        for (const auto& s : spans_) {
          const uintptr_t b = reinterpret_cast<uintptr_t>(s.first);
          const uintptr_t lo = (b + pg - 1) / pg * pg, hi = (b + s.second) / pg * pg;
          if (hi <= lo) continue;
          const size_t pages = (hi - lo) / pg;
          const uintptr_t a = lo + pages * t / nt * pg, e = lo + pages * (t + 1) / nt * pg;
          if (e <= a) continue;
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
          if (madvise(reinterpret_cast<void*>(a), e - a, MADV_POPULATE_WRITE) == 0) continue;
          for (uintptr_t q = a; q < e; q += pg) {
            volatile char* c = reinterpret_cast<volatile char*>(q);
            *c = *c;
          }
        }
      });
  }
  void join() {
    for (auto& t : threads_) t.join();
    threads_.clear();
  }
  ~Prefault() { join(); }

 private:
  std::vector<std::pair<char*, size_t>> spans_;
  std::vector<std::thread> threads_;
};

void d2h_pinned(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  QT_CUDA(qt::staged_copy(dst, src, bytes, false, st));
}

}  // namespace

// An estimated tree kept on the device (qt_estimate_device): counts, visits
// and pi in the layouts of qt_estimate, on `device`; the pricers read them in
// place (bdp.hpp:20-23 keeps a non-owning tree pointer the same way).
struct qt_dtree {
  int device = 0;
  int layers = 0;
  int dim = 0;
  uint64_t samples = 0;
  std::vector<uint64_t> sizes;
  uint64_t nvis = 0, njoint = 0;
  uint64_t* d_visits = nullptr;
  uint64_t* d_joint = nullptr;
  double* d_pi = nullptr;
  ~qt_dtree() {
    qt::DeviceRestore keep_device;
    cudaSetDevice(device);
    cudaFree(d_visits);
    cudaFree(d_joint);
    cudaFree(d_pi);
  }
};

namespace {

template <class F>
void with_bdp_errors(F&& f) {
  try {
    f();
  } catch (const qt::BdpError& e) {
    raise(static_cast<qt_status>(e.code), e.msg);
  }
}

// Shared body of qt_estimate / qt_estimate_normals / qt_accumulate_paths.
void run_estimate(int alg, const qt_chain* chain, const qt_grids* grids, uint64_t samples,
                  int engine, uint64_t seed, int devices, const double* h_normals,
                  uint64_t win_first, uint64_t win_count, uint64_t win_total, bool accumulate,
                  uint64_t* visits, uint64_t* joint, double* pi, double* phases,
                  qt_dtree** keep = nullptr) {
  const auto t0 = std::chrono::steady_clock::now();
  if (alg < QT_ALG_I || alg > QT_ALG_III)
    raise(QT_ERR_INVALID_ARGUMENT, "estimate: unknown estimator kind");
  if (samples == 0) raise(QT_ERR_INVALID_ARGUMENT, "estimate: need at least one path");
  if (devices < 1) raise(QT_ERR_INVALID_ARGUMENT, "estimate: devices must be >= 1");
  int avail = 0;
  if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
    raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the estimator has no CPU path)");
  // devices base .. base + G - 1, base = the caller's current device (a torchrun
  // rank that did set_device(local_rank) estimates on its own GPU)
  const int base = qt::current_device();
  if (base + devices > avail)
    raise(QT_ERR_INVALID_ARGUMENT, "estimate: requested " + std::to_string(devices) +
                                       " devices from device " + std::to_string(base) + ", " +
                                       std::to_string(avail) + " present");
  if (h_normals && devices != 1) raise(QT_ERR_INVALID_ARGUMENT, "normals mode is single-device");
  check_inputs(chain, grids);
  const int n = chain->layers;
  const uint64_t units_total = alg == QT_ALG_III ? static_cast<uint64_t>(n) * samples : samples;
  const uint64_t first = accumulate ? win_first : 0;
  const uint64_t count = accumulate ? win_count : units_total;
  const uint64_t total = accumulate ? win_total : units_total;
  const int G = devices;
  std::vector<std::unique_ptr<qt_plan>> plans(G);
  std::vector<std::vector<uint8_t>> keys(G);
  std::vector<uint64_t*> dj(G, nullptr);
  std::vector<cudaStream_t> streams(G, nullptr);
  std::vector<cudaEvent_t> ev(4 * G, nullptr);
  double* d_normals = nullptr;
  uint64_t* d_vis = nullptr;
  double* d_pi = nullptr;
  auto cleanup = [&] {
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(base + g);
      if (streams[g]) cudaStreamDestroy(streams[g]);
      for (int e = 0; e < 4; ++e)
        if (ev[4 * g + e]) cudaEventDestroy(ev[4 * g + e]);
    }
    cudaSetDevice(base);
    cudaFree(d_normals);
  };
  const bool dbg = std::getenv("QT_DEBUG") != nullptr;
  auto mark = [&](const char* what) {
    if (dbg) std::fprintf(stderr, "qtree: %-12s %9.2f ms\n", what, ms_since(t0));
  };
  try {
    for (int g = 0; g < G; ++g) keys[g] = plan_key(chain, grids, base + g);
    for (int g = 0; g < G; ++g) {
      plans[g] = take_plan(keys[g], chain, grids, base + g);
      mark("plan");
      QT_CUDA(cudaSetDevice(base + g));
      QT_CUDA(cudaStreamCreateWithFlags(&streams[g], cudaStreamNonBlocking));
      for (int e = 0; e < 4; ++e) QT_CUDA(cudaEventCreate(&ev[4 * g + e]));
      if (!plans[g]->d_ojoint)
        QT_CUDA(cudaMalloc(&plans[g]->d_ojoint, plans[g]->njoint * sizeof(uint64_t)));
      dj[g] = plans[g]->d_ojoint;
      QT_CUDA(cudaMemsetAsync(dj[g], 0, plans[g]->njoint * sizeof(uint64_t), streams[g]));
    }
    if (h_normals) {
      const uint64_t per = alg == QT_ALG_III ? static_cast<uint64_t>(plans[0]->dim + plans[0]->nps)
                                             : static_cast<uint64_t>(n) * plans[0]->nps;
      QT_CUDA(cudaSetDevice(base));
      QT_CUDA(cudaMalloc(&d_normals, count * per * sizeof(double)));
      QT_CUDA(cudaMemcpyAsync(d_normals, h_normals, count * per * sizeof(double),
                              cudaMemcpyHostToDevice, streams[0]));
    }
    mark("alloc");
    // shard g: units [first + count g / G, first + count (g+1) / G)  (estimate.hpp:180-181)
    for (int g = 0; g < G; ++g) {
      const uint64_t b = first + static_cast<uint64_t>(static_cast<u128>(count) * g / G);
      const uint64_t e = first + static_cast<uint64_t>(static_cast<u128>(count) * (g + 1) / G);
      QT_CUDA(cudaSetDevice(base + g));
      QT_CUDA(cudaEventRecord(ev[4 * g], streams[g]));
      plan_count(plans[g].get(), alg, engine, seed, b, e - b, total, d_normals, dj[g], streams[g]);
      QT_CUDA(cudaEventRecord(ev[4 * g + 1], streams[g]));
    }
    Prefault prefault;  // host output pages, mapped while the counts run
    if (!accumulate && !keep) {
      prefault.add(visits, plans[0]->nvis * 8);
      prefault.add(joint, plans[0]->njoint * 8);
      prefault.add(pi, plans[0]->njoint * 8);
      prefault.start();
    }
    if (G > 1) {
      const Nccl& nc = nccl();
      if (!nc.ok) raise(QT_ERR_DEVICE, "nccl: libnccl.so.2 not loadable for devices > 1");
      if (G > 64) raise(QT_ERR_INVALID_ARGUMENT, "estimate: at most 64 devices");
      NcclClique& cq = nccl_clique(base, G);
      std::lock_guard<std::mutex> clk(cq.mu);
      int rc = 0;
      if (cq.comms.empty()) {
        std::vector<void*> comms(G);
        std::vector<int> devs(G);
        std::iota(devs.begin(), devs.end(), base);
        rc = nc.init_all(comms.data(), G, devs.data());
        if (rc) raise(QT_ERR_DEVICE, std::string("nccl: ") + (nc.err ? nc.err(rc) : "init failed"));
        cq.comms = comms;
      }
      rc = nc.group_start();
      int rc_ar = 0;
      for (int g = 0; g < G && rc == 0; ++g) {
        cudaSetDevice(base + g);
        const int r = nc.all_reduce(dj[g], dj[g], plans[g]->njoint, kNcclUint64, kNcclSum,
                                    cq.comms[g], streams[g]);
        if (r && !rc_ar) rc_ar = r;
      }
      if (rc == 0) rc = nc.group_end();
      if (rc == 0) rc = rc_ar;
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(base + g);
        cudaEventRecord(ev[4 * g + 2], streams[g]);
        cudaStreamSynchronize(streams[g]);
      }
      if (rc) {  // a communicator that saw an error is not reused
        for (void* c : cq.comms)
          if (c) nc.destroy(c);
        cq.comms.clear();
      }
      if (rc) raise(QT_ERR_DEVICE, std::string("nccl: ") + (nc.err ? nc.err(rc) : "all-reduce failed"));
    } else {
      QT_CUDA(cudaEventRecord(ev[2], streams[0]));
    }
    QT_CUDA(cudaSetDevice(base));
    qt_plan* p0 = plans[0].get();
    if (!p0->d_ovis) QT_CUDA(cudaMalloc(&p0->d_ovis, p0->nvis * sizeof(uint64_t)));
    if (!p0->d_opi) QT_CUDA(cudaMalloc(&p0->d_opi, p0->njoint * sizeof(double)));
    d_vis = p0->d_ovis;
    d_pi = p0->d_opi;
    const uint64_t M_for_visits = accumulate ? count : samples;
    plan_finalize(p0, alg, M_for_visits, dj[0], d_vis, d_pi, streams[0]);
    QT_CUDA(cudaEventRecord(ev[3], streams[0]));
    std::vector<uint64_t> hv, hj;
    if (keep) {  // the tree stays on the device: the handle takes the plan's result buffers
      auto t = std::make_unique<qt_dtree>();
      t->device = base;
      t->layers = n;
      t->dim = grids->dim;
      t->samples = samples;
      t->sizes.assign(grids->sizes, grids->sizes + n + 1);
      t->nvis = p0->nvis;
      t->njoint = p0->njoint;
      t->d_joint = dj[0];
      t->d_visits = d_vis;
      t->d_pi = d_pi;
      p0->d_ojoint = nullptr;
      p0->d_ovis = nullptr;
      p0->d_opi = nullptr;
      *keep = t.release();
    } else if (accumulate) {
      hv.resize(p0->nvis);
      hj.resize(p0->njoint);
      QT_CUDA(cudaMemcpyAsync(hv.data(), d_vis, p0->nvis * 8, cudaMemcpyDeviceToHost, streams[0]));
      QT_CUDA(cudaMemcpyAsync(hj.data(), dj[0], p0->njoint * 8, cudaMemcpyDeviceToHost, streams[0]));
    } else if (!keep) {
      if (dbg) {
        QT_CUDA(cudaStreamSynchronize(streams[0]));
        mark("kernels done");
      }
      prefault.join();
      mark("prefaulted");
      d2h_pinned(visits, d_vis, p0->nvis * 8, streams[0]);
      d2h_pinned(joint, dj[0], p0->njoint * 8, streams[0]);
      mark("joint d2h");
      if (pi) d2h_pinned(pi, d_pi, p0->njoint * 8, streams[0]);
    }
    QT_CUDA(cudaStreamSynchronize(streams[0]));
    mark("d2h done");
    if (accumulate) {
      for (uint64_t i = 0; i < p0->nvis; ++i) visits[i] += hv[i];
      for (uint64_t i = 0; i < p0->njoint; ++i) joint[i] += hj[i];
    }
    if (phases) {
      float count_ms = 0, merge_ms = 0, norm_ms = 0;
      for (int g = 0; g < G; ++g) {
        float c = 0;
        cudaSetDevice(base + g);
        cudaEventElapsedTime(&c, ev[4 * g], ev[4 * g + 1]);
        count_ms = std::max(count_ms, c);
      }
      cudaSetDevice(base);
      cudaEventElapsedTime(&merge_ms, ev[1], ev[2]);
      cudaEventElapsedTime(&norm_ms, ev[2], ev[3]);
      phases[0] = 0.0;       // simulate: fused into the path kernel, reported under nn
      phases[1] = count_ms;  // fused path kernel (busiest device)
      phases[2] = merge_ms;  // NCCL all-reduce
      phases[3] = norm_ms;   // visits + normalize
      phases[4] = ms_since(t0);
    }
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  for (int g = 0; g < G; ++g)
    if (plans[g]) give_plan(std::move(keys[g]), std::move(plans[g]), static_cast<size_t>(G));
}

}  // namespace

namespace qt {
void note_error(const std::string& msg) { g_error = msg; }
void note_launches(uint64_t n) { g_launches.fetch_add(n); }

// Pageable host <-> device copy through a pinned double buffer: the DMA of one
// 32 MB chunk overlaps the (8-thread) memcpy of the next/previous chunk between
// the caller's buffer and pinned memory. A plain cudaMemcpy on pageable memory
// runs at a few GB/s (driver staging + page faults on fresh arrays); this keeps
// the host link busy. The two pinned buffers are shared and serialised.
cudaError_t staged_copy(void* dst, const void* src, size_t bytes, bool to_device,
                        cudaStream_t st) {
  constexpr size_t kChunk = 32u << 20;
  static std::mutex mu;
  static uint8_t* pin[2] = {nullptr, nullptr};
  std::lock_guard<std::mutex> lk(mu);
  const cudaMemcpyKind kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  cudaError_t e = cudaSuccess;
  if (bytes < (4u << 20)) {  // small: direct
    if ((e = cudaMemcpyAsync(dst, src, bytes, kind, st)) != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
  }
  for (auto*& b : pin)
    if (!b && (e = cudaHostAlloc(reinterpret_cast<void**>(&b), kChunk, cudaHostAllocDefault)))
      return e;
  auto par_copy = [](uint8_t* d, const uint8_t* s, size_t n) {
    constexpr int kT = 8;
    std::vector<std::thread> th;
    const size_t per = (n + kT - 1) / kT;
    for (int t = 1; t < kT; ++t) {
      const size_t b = per * t, en = std::min(n, b + per);
      if (b < en) th.emplace_back([=] { std::memcpy(d + b, s + b, en - b); });
    }
    std::memcpy(d, s, std::min(n, per));
    for (auto& x : th) x.join();
  };
  cudaEvent_t ev[2];
  if ((e = cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming))) return e;
  if ((e = cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming))) {
    cudaEventDestroy(ev[0]);
    return e;
  }
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  auto* d8 = static_cast<uint8_t*>(dst);
  auto* s8 = static_cast<const uint8_t*>(src);
  auto len = [&](size_t c) { return std::min(kChunk, bytes - c * kChunk); };
  if (to_device) {
    // chunk c: wait until buffer c&1 is free (DMA of c-2 done), fill it, DMA it
    for (size_t c = 0; c < nchunks && !e; ++c) {
      if (c >= 2 && (e = cudaEventSynchronize(ev[c & 1]))) break;
      par_copy(pin[c & 1], s8 + c * kChunk, len(c));
      if ((e = cudaMemcpyAsync(d8 + c * kChunk, pin[c & 1], len(c), kind, st))) break;
      e = cudaEventRecord(ev[c & 1], st);
    }
    if (!e) e = cudaStreamSynchronize(st);
  } else {
    auto issue = [&](size_t c) {
      cudaError_t r = cudaMemcpyAsync(pin[c & 1], s8 + c * kChunk, len(c), kind, st);
      return r ? r : cudaEventRecord(ev[c & 1], st);
    };
    e = issue(0);
    for (size_t c = 0; c < nchunks && !e; ++c) {
      if (c + 1 < nchunks && (e = issue(c + 1))) break;
      if ((e = cudaEventSynchronize(ev[c & 1]))) break;
      par_copy(d8 + c * kChunk, pin[c & 1], len(c));
    }
  }
  if (e) cudaStreamSynchronize(st);  // never leave a DMA in flight on the shared buffers
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  return e;
}
}  // namespace qt

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

QT_API qt_status qt_chain_coefficients(int32_t kind, const qt_model_params* params, double* step,
                                       double* marginal) {
  return guarded([&] {
    if (!params || !step || !marginal) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    chain_coefficients(kind, *params, step, marginal);
  });
}

// ---- obstacles (pipeline.hpp:120-170, two_factor.hpp:144-176) ------------------
// The reference builds std::function payoffs and the pricer evaluates them per
// node; here the same expressions are tabulated once per tree on the host, in
// the reference's evaluation order (no FMA contraction on x86-64 baseline), so
// phi is bit-identical. std::max(a, b) is (a < b) ? b : a.
namespace {
double rmax(double a, double b) { return (a < b) ? b : a; }

// model::spot (two_factor.hpp:144-152)
double spot_of(const qt_model_params& p, double t, double x1, double x2) {
  double c[3];
  ou_cov(t, p.alpha1, p.alpha2, p.rho, c);
  const double comp = p.sigma1 * p.sigma1 * c[0] + 2.0 * p.sigma1 * p.sigma2 * c[1] +
                      p.sigma2 * p.sigma2 * c[2];
  return p.s0 * std::exp(p.sigma1 * x1 + p.sigma2 * x2 - 0.5 * comp);
}

// one node's discounted obstacle; x has the chain's dimension
double payoff_at(int payoff, int chain_kind, const qt_model_params& p, const double* gsig, int k,
                 const double* x) {
  const double dt = p.horizon / p.steps;
  const double t = k * dt;
  if (chain_kind == QT_CHAIN_GBM_3D || payoff == QT_PAYOFF_MAX_CALL) {
    // config 5 (new): e^{-rt} max(max_a S_a - K, 0), S_a = s0 e^{(r - s_a^2/2) t + s_a x_a}
    double best = -std::numeric_limits<double>::infinity();
    for (int a = 0; a < 3; ++a) {
      const double sa = p.s0 * std::exp((p.r - 0.5 * gsig[a] * gsig[a]) * t + gsig[a] * x[a]);
      best = rmax(best, sa);
    }
    return std::exp(-p.r * t) * rmax(best - p.strike, 0.0);
  }
  if (chain_kind == QT_CHAIN_OU_1D) {
    // config 3 (new): the 2-factor spot with sigma2 = 0 on the OU factor-1 state
    qt_model_params q = p;
    q.sigma2 = 0.0;
    const double sp = spot_of(q, t, x[0], 0.0);
    if (payoff == QT_PAYOFF_SWING) return std::exp(-q.r * t) * (sp - q.strike);
    if (payoff == QT_PAYOFF_PUT) return std::exp(-q.r * t) * rmax(q.strike - sp, 0.0);
    return std::exp(-q.r * t) * rmax(sp - q.strike, 0.0);
  }
  if (chain_kind == QT_CHAIN_BROWNIAN_1D) {
    // make_*_payoff(cfg, 1): lognormal benchmark on the Brownian state
    // (amer_payoff / amer_put_payoff two_factor.hpp:158-170, pipeline.hpp:160-164)
    const double sp = p.s0 * std::exp((p.r - 0.5 * p.sigma1 * p.sigma1) * t + p.sigma1 * x[0]);
    if (payoff == QT_PAYOFF_PUT) return std::exp(-p.r * t) * rmax(p.strike - sp, 0.0);
    if (payoff == QT_PAYOFF_CALL) return std::exp(-p.r * t) * rmax(sp - p.strike, 0.0);
    return std::exp(-p.r * t) * (sp - p.strike);
  }
  // make_*_payoff(cfg, 2): the 2-factor spot (pipeline.hpp:131-134,146-149,166-169)
  const double sp = spot_of(p, t, x[0], x[1]);
  if (payoff == QT_PAYOFF_PUT) return std::exp(-p.r * t) * rmax(p.strike - sp, 0.0);
  if (payoff == QT_PAYOFF_CALL) return std::exp(-p.r * t) * rmax(sp - p.strike, 0.0);
  return std::exp(-p.r * t) * (sp - p.strike);
}
}  // namespace

QT_API qt_status qt_payoff_table(int32_t payoff, int32_t chain_kind, const qt_model_params* params,
                                 const double* gbm_sigma, int32_t layers, const uint64_t* sizes,
                                 const double* points_all, double* phi) {
  return guarded([&] {
    if (!params || !sizes || !points_all || !phi) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    if (payoff < QT_PAYOFF_PUT || payoff > QT_PAYOFF_MAX_CALL)
      raise(QT_ERR_INVALID_ARGUMENT, "payoff: unknown kind");
    const int dim = chain_dim(chain_kind);
    const bool maxcall = chain_kind == QT_CHAIN_GBM_3D || payoff == QT_PAYOFF_MAX_CALL;
    if (maxcall && (dim != 3 || !gbm_sigma))
      raise(QT_ERR_INVALID_ARGUMENT, "payoff: max-call needs the 3-D chain and gbm_sigma[3]");
    if (layers < 1 || layers != params->steps)
      raise(QT_ERR_INVALID_ARGUMENT, "payoff: layers must equal params->steps");
    uint64_t o = 0;
    for (int k = 0; k <= layers; ++k)
      for (uint64_t i = 0; i < sizes[k]; ++i, ++o)
        phi[o] = payoff_at(payoff, chain_kind, *params, gbm_sigma, k, points_all + o * dim);
  });
}

QT_API qt_status qt_estimate(int32_t estimator, const qt_chain* chain, const qt_grids* grids,
                             uint64_t samples, int32_t engine, uint64_t seed, int32_t devices,
                             uint64_t* visits, uint64_t* joint, double* pi, double* phases_ms) {
  return guarded([&] {
    if (!visits || !joint) raise(QT_ERR_INVALID_ARGUMENT, "estimate: null output");
    source_of(engine, false);
    run_estimate(estimator, chain, grids, samples, engine, seed, devices, nullptr, 0, 0, 0, false,
                 visits, joint, pi, phases_ms);
  });
}

// ---- estimate -> price on the device ----------------------------------------
QT_API qt_status qt_estimate_device(int32_t estimator, const qt_chain* chain,
                                    const qt_grids* grids, uint64_t samples, int32_t engine,
                                    uint64_t seed, int32_t devices, qt_dtree** tree,
                                    double* phases_ms) {
  return guarded([&] {
    if (!tree) raise(QT_ERR_INVALID_ARGUMENT, "estimate: null output");
    *tree = nullptr;
    source_of(engine, false);
    run_estimate(estimator, chain, grids, samples, engine, seed, devices, nullptr, 0, 0, 0, false,
                 nullptr, nullptr, nullptr, phases_ms, tree);
  });
}

QT_API qt_status qt_dtree_destroy(qt_dtree* tree) {
  return guarded([&] { delete tree; });
}

QT_API qt_status qt_dtree_info(const qt_dtree* tree, int32_t* layers, int32_t* dim,
                               uint64_t* samples, uint64_t* sizes, uint64_t sizes_cap,
                               int32_t* device) {
  return guarded([&] {
    if (!tree) raise(QT_ERR_INVALID_ARGUMENT, "dtree: null tree");
    if (layers) *layers = tree->layers;
    if (dim) *dim = tree->dim;
    if (samples) *samples = tree->samples;
    if (device) *device = tree->device;
    if (sizes && sizes_cap >= tree->sizes.size())
      std::copy(tree->sizes.begin(), tree->sizes.end(), sizes);
  });
}

QT_API qt_status qt_dtree_device_arrays(const qt_dtree* tree, const uint64_t** visits,
                                        const uint64_t** joint, const double** pi) {
  return guarded([&] {
    if (!tree) raise(QT_ERR_INVALID_ARGUMENT, "dtree: null tree");
    if (visits) *visits = tree->d_visits;
    if (joint) *joint = tree->d_joint;
    if (pi) *pi = tree->d_pi;
  });
}

QT_API qt_status qt_dtree_download(const qt_dtree* tree, uint64_t* visits, uint64_t* joint,
                                   double* pi) {
  return guarded([&] {
    if (!tree) raise(QT_ERR_INVALID_ARGUMENT, "dtree: null tree");
    QT_CUDA(cudaSetDevice(tree->device));
    if (visits) QT_CUDA(qt::staged_copy(visits, tree->d_visits, tree->nvis * 8, false, 0));
    if (joint) QT_CUDA(qt::staged_copy(joint, tree->d_joint, tree->njoint * 8, false, 0));
    if (pi) QT_CUDA(qt::staged_copy(pi, tree->d_pi, tree->njoint * 8, false, 0));
  });
}

QT_API qt_status qt_dtree_stopping(const qt_dtree* tree, const double* phi, double* value,
                                   uint8_t* exercise, double* price) {
  return guarded([&] {
    if (!tree) raise(QT_ERR_INVALID_ARGUMENT, "solve_stopping: incomplete problem");
    QT_CUDA(cudaSetDevice(tree->device));
    with_bdp_errors([&] {
      qt::bdp_stopping_device(tree->layers, tree->sizes.data(), tree->d_visits, tree->d_pi, phi,
                              value, exercise, price);
    });
  });
}

QT_API qt_status qt_dtree_swing(const qt_dtree* tree, const double* phi, int32_t qmin,
                                int32_t qmax, double* price, double* value_all,
                                uint8_t* take_all) {
  return guarded([&] {
    if (!tree) raise(QT_ERR_INVALID_ARGUMENT, "solve_swing: incomplete problem");
    QT_CUDA(cudaSetDevice(tree->device));
    with_bdp_errors([&] {
      qt::bdp_swing_device(tree->layers, tree->sizes.data(), tree->d_visits, tree->d_pi, phi, qmin,
                           qmax, price, value_all, take_all);
    });
  });
}

QT_API qt_status qt_estimate_normals(int32_t estimator, const qt_chain* chain,
                                     const qt_grids* grids, uint64_t samples,
                                     const double* normals, uint64_t* visits, uint64_t* joint,
                                     double* pi) {
  return guarded([&] {
    if (!visits || !joint || !normals) raise(QT_ERR_INVALID_ARGUMENT, "estimate: null argument");
    run_estimate(estimator, chain, grids, samples, QT_ENGINE_MRG32K3A, 0, 1, normals, 0, 0, 0,
                 false, visits, joint, pi, nullptr);
  });
}

QT_API qt_status qt_accumulate_paths(const qt_chain* chain, const qt_grids* grids,
                                     int32_t engine, uint64_t seed, uint64_t first,
                                     uint64_t count, uint64_t total, uint64_t* visits,
                                     uint64_t* joint) {
  return guarded([&] {
    if (!visits || !joint) raise(QT_ERR_INVALID_ARGUMENT, "accumulate: null output");
    source_of(engine, false);
    if (count == 0) return;
    run_estimate(QT_ALG_I, chain, grids, total ? total : 1, engine, seed, 1, nullptr, first,
                 count, total, true, visits, joint, nullptr, nullptr);
  });
}

QT_API qt_status qt_plan_create(const qt_chain* chain, const qt_grids* grids, int32_t device,
                                qt_plan** out) {
  return guarded([&] {
    if (!out) raise(QT_ERR_INVALID_ARGUMENT, "plan: null output");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the estimator has no CPU path)");
    if (device < 0 || device >= avail) raise(QT_ERR_INVALID_ARGUMENT, "plan: bad device");
    *out = make_plan(chain, grids, device);
  });
}

QT_API qt_status qt_plan_destroy(qt_plan* plan) {
  return guarded([&] { delete plan; });
}

QT_API qt_status qt_plan_layout(const qt_plan* plan, uint64_t* n_visits, uint64_t* n_joint) {
  return guarded([&] {
    if (!plan) raise(QT_ERR_INVALID_ARGUMENT, "plan: null");
    if (n_visits) *n_visits = plan->nvis;
    if (n_joint) *n_joint = plan->njoint;
  });
}

QT_API qt_status qt_plan_count(qt_plan* plan, int32_t estimator, int32_t engine, uint64_t seed,
                               uint64_t first, uint64_t count, uint64_t total,
                               const double* d_normals, uint64_t* d_joint, void* stream,
                               int32_t* launches) {
  return guarded([&] {
    if (!plan || !d_joint) raise(QT_ERR_INVALID_ARGUMENT, "plan_count: null argument");
    if (total == 0 || first + count > total)
      raise(QT_ERR_INVALID_ARGUMENT, "plan_count: window outside [0, total)");
    const int l = plan_count(plan, estimator, engine, seed, first, count, total, d_normals, d_joint,
                             static_cast<cudaStream_t>(stream));
    if (launches) *launches = l;
  });
}

QT_API qt_status qt_plan_finalize(qt_plan* plan, int32_t estimator, uint64_t samples,
                                  const uint64_t* d_joint, uint64_t* d_visits, double* d_pi,
                                  void* stream, int32_t* launches) {
  return guarded([&] {
    if (!plan || !d_joint || !d_visits || !d_pi)
      raise(QT_ERR_INVALID_ARGUMENT, "plan_finalize: null argument");
    if (estimator < QT_ALG_I || estimator > QT_ALG_III)
      raise(QT_ERR_INVALID_ARGUMENT, "estimate: unknown estimator kind");
    const int l = plan_finalize(plan, estimator, samples, d_joint, d_visits, d_pi,
                                static_cast<cudaStream_t>(stream));
    if (launches) *launches = l;
  });
}

// Device tables of one grid for batch projection: the exact table (+ cold
// block) and, for d >= 2, the FP32 scan table behind it. Uploads into *buf
// (grown as needed) and enqueues the projection of nq device queries.
struct GridTables {
  std::vector<uint8_t> blob;  // exact hot | exact cold | scan (d >= 2)
  uint32_t hot_bytes = 0, scan_off = 0, scan_bytes = 0;
};
// d >= 2 grids this small are faster with the plain FP64 scan (k_nearest)
constexpr uint64_t kScanMinPoints = 192;

GridTables grid_tables(int dim, uint64_t n, const double* pts) {
  double zeros[6] = {0, 0, 0, 0, 0, 0};
  TableBlob tb = build_table(-1, dim, n, pts, zeros, zeros, 0, 1, 1);
  GridTables g;
  g.blob = tb.hot;
  g.hot_bytes = static_cast<uint32_t>(tb.hot.size());
  set_cold_off(g.blob, g.blob.size());
  g.blob.insert(g.blob.end(), tb.cold.begin(), tb.cold.end());
  if (dim >= 2 && n >= kScanMinPoints) {
    g.blob.resize(round16(g.blob.size()), 0);
    g.scan_off = static_cast<uint32_t>(g.blob.size());
    const auto sc = build_scan_table(dim, n, pts, zeros, 0, 0);
    g.scan_bytes = static_cast<uint32_t>(sc.size());
    g.blob.insert(g.blob.end(), sc.begin(), sc.end());
  }
  return g;
}
cudaError_t project_on_device(int dim, const GridTables& g, const uint8_t* d_blob, const double* dq,
                              uint64_t nq, unsigned long long* dout, cudaStream_t st) {
  if (dim >= 2 && g.scan_bytes && g.scan_bytes <= 200u * 1024u)
    return qt::launch_nearest_scan(dim, d_blob + g.scan_off, g.scan_bytes, d_blob, dq, nq, dout, st);
  return qt::launch_nearest(dim, d_blob, g.hot_bytes, dq, nq, dout, st);
}

// lloyd_build (lloyd.hpp:59-107) with the GaussianSampler on the serial
// MRG32k3a stream seeded `stream_seed` (the pipeline passes seed ^ 0x9E3779B9,
// pipeline.hpp:35,63). normals (nullable): the stream's normals supplied by the
// caller (parity mode), at least as many as the build consumes.
}  // extern "C"

namespace {

// The serial normal stream of lloyd_build / distortion: an optional cached
// Box-Muller mate of the caller's RngStream first (stream.hpp:97-103), then
// the stream's own normals from `src` (pair p from uniforms 2p, 2p+1), or the
// caller's normals (parity mode).
struct NormalStream {
  qt::SrcArgs src{};
  bool lead = false;        // a cached mate precedes the device normals
  double lead_value = 0.0;
  const double* normals = nullptr;  // parity mode
  uint64_t n_normals = 0;
};

// lloyd_build (lloyd.hpp:59-107) with the GaussianSampler; returns the number
// of normals consumed from the stream.
uint64_t lloyd_core(int32_t dim, uint64_t n_points, int32_t iterations, uint64_t samples_per_iter,
                    const NormalStream& ns, double* centers, double* distortion) {
  uint64_t used_total = 0;
  {
    if (n_points == 0) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: need at least one center");
    if (iterations < 0) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: iterations must be >= 0");
    if (dim < 1 || dim > 3) raise(QT_ERR_NUMERIC, "lloyd_build: sampler dimension mismatch");
    if (!centers) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: null output");
    if (samples_per_iter == 0 && iterations > 0)
      raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: samples_per_iter must be >= 1");
    if (samples_per_iter > 0x7fffffffull || n_points > 0x7fffffffull)
      raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: batch too large");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the build has no CPU path)");
    const uint64_t d = static_cast<uint64_t>(dim), N = n_points, M = samples_per_iter;
    const double* normals = ns.normals;
    const uint64_t n_normals = ns.n_normals;
    cudaStream_t st = nullptr;
    std::vector<void*> bufs;
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      QT_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
      bufs.push_back(p);
      return p;
    };
    auto cleanup = [&] {
      for (void* p : bufs) cudaFree(p);
      if (st) cudaStreamDestroy(st);
    };
    try {
      QT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      uint64_t consumed = 0;  // normals of the stream used so far
      auto fetch = [&](double* dst_dev, uint64_t count) {
        if (normals) {
          if (consumed + count > n_normals)
            raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: not enough normals supplied");
          QT_CUDA(cudaMemcpyAsync(dst_dev, normals + consumed, count * 8, cudaMemcpyHostToDevice, st));
        } else {
          uint64_t at = consumed, n = count;
          double* dst = dst_dev;
          if (ns.lead && at == 0 && n > 0) {  // the caller's cached mate comes first
            QT_CUDA(cudaMemcpyAsync(dst, &ns.lead_value, 8, cudaMemcpyHostToDevice, st));
            ++dst;
            --n;
            ++at;
          }
          if (n) {
            QT_CUDA(qt::launch_serial_normals(ns.src, at - (ns.lead ? 1 : 0), n, dst, st));
            g_launches.fetch_add(1);
          }
        }
        consumed += count;
      };
      // initial centers: distinct samples in stream order (lloyd.hpp:72-83)
      std::vector<double> c;
      c.reserve(N * d);
      {
        std::set<std::vector<double>> seen;
        uint64_t attempts = 0;
        const uint64_t batch = (N + 64) * d;
        double* dn = static_cast<double*>(dalloc(batch * 8));
        std::vector<double> h(batch);
        while (c.size() < N * d) {
          fetch(dn, batch);
          QT_CUDA(cudaMemcpyAsync(h.data(), dn, batch * 8, cudaMemcpyDeviceToHost, st));
          QT_CUDA(cudaStreamSynchronize(st));
          uint64_t used = 0;
          for (; used + d <= batch && c.size() < N * d; used += d) {
            std::vector<double> x(h.begin() + used, h.begin() + used + d);
            if (seen.insert(x).second) c.insert(c.end(), x.begin(), x.end());
            if (++attempts > 100 * N + 100)
              raise(QT_ERR_NUMERIC, "lloyd_build: sampler cannot produce enough distinct centers");
          }
          consumed -= batch - used;  // hand the unused normals back to the stream
        }
      }
      if (iterations > 0) {
        double* dX = static_cast<double*>(dalloc(M * d * 8));
        double* dC = static_cast<double*>(dalloc(N * d * 8));
        double* dd2 = static_cast<double*>(dalloc(M * 8));
        auto* dcell = static_cast<unsigned long long*>(dalloc(M * 8));
        auto* key = static_cast<uint32_t*>(dalloc(M * 4));
        auto* idx = static_cast<uint32_t*>(dalloc(M * 4));
        auto* key2 = static_cast<uint32_t*>(dalloc(M * 4));
        auto* idx2 = static_cast<uint32_t*>(dalloc(M * 4));
        auto* cnt = static_cast<uint32_t*>(dalloc(N * 4));
        auto* offs = static_cast<uint32_t*>(dalloc(N * 4));
        const size_t tmp_bytes = qt::lloyd_tmp_bytes(M, N);
        void* tmp = dalloc(tmp_bytes);
        uint8_t* dT = nullptr;
        size_t dT_bytes = 0;
        std::vector<double> hd2(M);
        QT_CUDA(cudaMemcpyAsync(dC, c.data(), N * d * 8, cudaMemcpyHostToDevice, st));
        for (int it = 0; it < iterations; ++it) {
          // snapshot grid (lloyd.hpp:88-89): the reference's QuantGrid checks
          check_grid(dim, N, c.data(), 0);
          const GridTables gt = grid_tables(dim, N, c.data());
          const std::vector<uint8_t>& t = gt.blob;
          if (t.size() > dT_bytes) {
            dT = static_cast<uint8_t*>(dalloc(t.size()));
            dT_bytes = t.size();
          }
          QT_CUDA(cudaMemcpyAsync(dT, t.data(), t.size(), cudaMemcpyHostToDevice, st));
          fetch(dX, M * d);
          QT_CUDA(project_on_device(dim, gt, dT, dX, M, dcell, st));
          QT_CUDA(qt::launch_lloyd_update(dX, dcell, M, N, dim, dC, dd2, key, idx, key2, idx2, cnt,
                                          offs, tmp, tmp_bytes, st));
          g_launches.fetch_add(4);
          QT_CUDA(cudaMemcpyAsync(hd2.data(), dd2, M * 8, cudaMemcpyDeviceToHost, st));
          QT_CUDA(cudaMemcpyAsync(c.data(), dC, N * d * 8, cudaMemcpyDeviceToHost, st));
          QT_CUDA(cudaStreamSynchronize(st));
          if (distortion) {  // dist_sum in sample order (lloyd.hpp:94-97)
            double sum = 0.0;
            for (uint64_t m = 0; m < M; ++m) sum += hd2[m];
            distortion[it] = sum / static_cast<double>(M);
          }
        }
      }
      check_grid(dim, N, c.data(), 0);  // result.grid = QuantGrid(dim, centers)
      std::memcpy(centers, c.data(), N * d * 8);
      QT_CUDA(cudaStreamSynchronize(st));
      used_total = consumed;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
  return used_total;
}

void lloyd_args(int32_t dim, uint64_t n_points, int32_t iterations, uint64_t samples_per_iter,
                const double* centers) {
  if (n_points == 0) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: need at least one center");
  if (iterations < 0) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: iterations must be >= 0");
  if (dim < 1 || dim > 3) raise(QT_ERR_NUMERIC, "lloyd_build: sampler dimension mismatch");
  if (!centers) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: null output");
  if (samples_per_iter == 0 && iterations > 0)
    raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: samples_per_iter must be >= 1");
  if (samples_per_iter > 0x7fffffffull || n_points > 0x7fffffffull)
    raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: batch too large");
  int avail = 0;
  if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
    raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the build has no CPU path)");
}

// The caller's RngStream state (s1[3], s2[3], cached mate) -> NormalStream.
NormalStream stream_of(const uint64_t* state6, int32_t has_spare, double spare) {
  NormalStream ns;
  ns.src = make_src(qt::current_device(), QT_ENGINE_MRG32K3A, 0, 1, 1, nullptr, 0);
  for (int i = 0; i < 6; ++i) {
    const uint64_t m = i < 3 ? kM1 : kM2;
    if (state6[i] >= m) raise(QT_ERR_INVALID_ARGUMENT, "rng: MRG32k3a state word out of range");
    ns.src.mrg_seed[i] = static_cast<uint32_t>(state6[i]);
  }
  ns.lead = has_spare != 0;
  ns.lead_value = spare;
  return ns;
}

// Leave the caller's stream where the reference's would be after `used`
// normals: the device normals consumed D = used - lead advance the state by
// 2 ceil(D / 2) uniforms, and an odd D leaves the last pair's mate cached.
void advance_stream(const NormalStream& ns, uint64_t used, uint64_t* state6, int32_t* has_spare,
                    double* spare) {
  if (used == 0) return;
  if (ns.lead && used == 1) {
    *has_spare = 0;
    return;
  }
  const uint64_t D = used - (ns.lead ? 1 : 0);
  const uint64_t pairs = (D + 1) / 2;
  if (D % 2 == 1) {  // the mate of pair D / 2 is normal D of the device stream
    double* dn = nullptr;
    QT_CUDA(cudaMalloc(&dn, 8));
    cudaError_t e = qt::launch_serial_normals(ns.src, D, 1, dn, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(spare, dn, 8, cudaMemcpyDeviceToHost);
    cudaFree(dn);
    QT_CUDA(e);
    g_launches.fetch_add(1);
    *has_spare = 1;
  } else {
    *has_spare = 0;
  }
  mrg_skip_host(state6, 2 * pairs);
}

}  // namespace

extern "C" {

QT_API qt_status qt_lloyd_build(int32_t dim, uint64_t n_points, int32_t iterations,
                                uint64_t samples_per_iter, uint64_t stream_seed,
                                const double* normals, uint64_t n_normals, double* centers,
                                double* distortion) {
  return guarded([&] {
    lloyd_args(dim, n_points, iterations, samples_per_iter, centers);
    NormalStream ns;
    ns.src = make_src(qt::current_device(), QT_ENGINE_MRG32K3A, stream_seed, 1, 1, nullptr, 0);
    ns.normals = normals;
    ns.n_normals = n_normals;
    lloyd_core(dim, n_points, iterations, samples_per_iter, ns, centers, distortion);
  });
}

QT_API qt_status qt_lloyd_build_stream(int32_t dim, uint64_t n_points, int32_t iterations,
                                       uint64_t samples_per_iter, uint64_t* state6,
                                       int32_t* has_spare, double* spare, double* centers,
                                       double* distortion) {
  return guarded([&] {
    // zero samples per iteration: the reference's iterations assign nothing, keep
    // every center and record 0 / 0 (lloyd.hpp:97-105)
    const bool empty = samples_per_iter == 0 && iterations > 0;
    lloyd_args(dim, n_points, empty ? 0 : iterations, samples_per_iter, centers);
    if (!state6 || !has_spare || !spare) raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: null stream");
    const NormalStream ns = stream_of(state6, *has_spare, *spare);
    const uint64_t used = lloyd_core(dim, n_points, empty ? 0 : iterations, samples_per_iter, ns,
                                     centers, distortion);
    if (empty && distortion) {
      volatile double zero = 0.0;  // the reference's dist_sum / 0 (lloyd.hpp:97), same NaN bits
      for (int it = 0; it < iterations; ++it) distortion[it] = zero / zero;
    }
    advance_stream(ns, used, state6, has_spare, spare);
  });
}

// One iteration of lloyd_build (lloyd.hpp:86-106) on caller-drawn samples X
// (M x dim, sample-major; any PointSampler): the snapshot's exact cells on the
// device, per-cell sums in sample order (stable sort, one thread per cell),
// empty cells keep their point; *distortion = the mean squared distance to the
// old centers, summed in sample order.
QT_API qt_status qt_lloyd_iterate(int32_t dim, uint64_t n_points, double* centers, uint64_t M,
                                  const double* X, double* distortion) {
  return guarded([&] {
    if (dim < 1 || dim > 3 || n_points == 0 || !centers || !X || M == 0 || !distortion)
      raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: bad iteration arguments");
    if (M > 0x7fffffffull || n_points > 0x7fffffffull)
      raise(QT_ERR_INVALID_ARGUMENT, "lloyd_build: batch too large");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the build has no CPU path)");
    check_grid(dim, n_points, centers, 0);  // QuantGrid snapshot(dim, centers)
    const uint64_t d = static_cast<uint64_t>(dim), N = n_points;
    std::vector<void*> bufs;
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      QT_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
      bufs.push_back(p);
      return p;
    };
    try {
      double* dX = static_cast<double*>(dalloc(M * d * 8));
      double* dC = static_cast<double*>(dalloc(N * d * 8));
      double* dd2 = static_cast<double*>(dalloc(M * 8));
      auto* dcell = static_cast<unsigned long long*>(dalloc(M * 8));
      auto* key = static_cast<uint32_t*>(dalloc(M * 4));
      auto* idx = static_cast<uint32_t*>(dalloc(M * 4));
      auto* key2 = static_cast<uint32_t*>(dalloc(M * 4));
      auto* idx2 = static_cast<uint32_t*>(dalloc(M * 4));
      auto* cnt = static_cast<uint32_t*>(dalloc(N * 4));
      auto* offs = static_cast<uint32_t*>(dalloc(N * 4));
      const size_t tmp_bytes = qt::lloyd_tmp_bytes(M, N);
      void* tmp = dalloc(tmp_bytes);
      const GridTables gt = grid_tables(dim, N, centers);
      uint8_t* dT = static_cast<uint8_t*>(dalloc(gt.blob.size()));
      QT_CUDA(cudaMemcpy(dT, gt.blob.data(), gt.blob.size(), cudaMemcpyHostToDevice));
      QT_CUDA(qt::staged_copy(dX, X, M * d * 8, true, 0));
      QT_CUDA(cudaMemcpy(dC, centers, N * d * 8, cudaMemcpyHostToDevice));
      QT_CUDA(project_on_device(dim, gt, dT, dX, M, dcell, nullptr));
      QT_CUDA(qt::launch_lloyd_update(dX, dcell, M, N, dim, dC, dd2, key, idx, key2, idx2, cnt, offs,
                                      tmp, tmp_bytes, nullptr));
      g_launches.fetch_add(5);
      std::vector<double> hd2(M);
      QT_CUDA(cudaMemcpy(hd2.data(), dd2, M * 8, cudaMemcpyDeviceToHost));
      QT_CUDA(cudaMemcpy(centers, dC, N * d * 8, cudaMemcpyDeviceToHost));
      double sum = 0.0;
      for (uint64_t m = 0; m < M; ++m) sum += hd2[m];
      *distortion = sum / static_cast<double>(M);
    } catch (...) {
      for (void* b : bufs) cudaFree(b);
      throw;
    }
    for (void* b : bufs) cudaFree(b);
  });
}

// distortion (lloyd.hpp:30-48) on caller-drawn samples X (M x dim): exact cells
// on the device, sum and sum of squares in sample order on the host.
QT_API qt_status qt_distortion_points(int32_t dim, uint64_t n_points, const double* centers,
                                      uint64_t M, const double* X, double* mean,
                                      double* std_error) {
  return guarded([&] {
    if (M == 0) raise(QT_ERR_INVALID_ARGUMENT, "distortion: samples must be >= 1");
    if (dim < 1 || dim > 3 || n_points == 0 || !centers || !X || !mean || !std_error)
      raise(QT_ERR_INVALID_ARGUMENT, "distortion: null argument");
    std::vector<uint64_t> cell(M);
    if (const qt_status rc = qt_nearest(dim, n_points, centers, M, X, cell.data()))
      raise(rc, std::string(g_error));
    const uint64_t d = static_cast<uint64_t>(dim);
    double sum = 0.0, sum_sq = 0.0;
    for (uint64_t m = 0; m < M; ++m) {
      const double* x = X + m * d;
      const double* c = centers + cell[m] * d;
      double d2 = 0.0;  // squared_distance (grid.hpp:65-72)
      for (uint64_t j = 0; j < d; ++j) {
        volatile double t = x[j] - c[j];
        volatile double tt = t * t;
        d2 = d2 + tt;
      }
      sum += d2;
      volatile double sq = d2 * d2;
      sum_sq += sq;
    }
    const double mu = sum / static_cast<double>(M);
    const double var = std::max(0.0, sum_sq / static_cast<double>(M) - mu * mu);
    *mean = mu;
    *std_error = std::sqrt(var / static_cast<double>(M));
  });
}

// distortion (lloyd.hpp:30-48): E min_i |X - x_i|^2 over `samples` GaussianSampler
// draws of the caller's stream; the cells by the exact projection, the sums in
// sample order on the host (sum, sum of squares; as the reference).
QT_API qt_status qt_distortion_stream(int32_t dim, uint64_t n_points, const double* centers,
                                      uint64_t samples, uint64_t* state6, int32_t* has_spare,
                                      double* spare, double* mean, double* std_error) {
  return guarded([&] {
    if (samples == 0) raise(QT_ERR_INVALID_ARGUMENT, "distortion: samples must be >= 1");
    if (dim < 1 || dim > 3 || n_points == 0 || !centers)
      raise(QT_ERR_NUMERIC, "distortion: sampler dimension mismatch");
    if (!state6 || !has_spare || !spare || !mean || !std_error)
      raise(QT_ERR_INVALID_ARGUMENT, "distortion: null argument");
    if (samples > 0x7fffffffull) raise(QT_ERR_INVALID_ARGUMENT, "distortion: batch too large");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the build has no CPU path)");
    check_grid(dim, n_points, centers, 0);
    const NormalStream ns = stream_of(state6, *has_spare, *spare);
    const uint64_t d = static_cast<uint64_t>(dim), total = samples * d;
    double* dX = nullptr;
    unsigned long long* dcell = nullptr;
    uint8_t* dT = nullptr;
    auto fin = [&] {
      cudaFree(dX);
      cudaFree(dcell);
      cudaFree(dT);
    };
    try {
      QT_CUDA(cudaMalloc(&dX, total * 8));
      QT_CUDA(cudaMalloc(&dcell, samples * 8));
      double* dst = dX;
      uint64_t n = total;
      if (ns.lead) {
        QT_CUDA(cudaMemcpy(dst, &ns.lead_value, 8, cudaMemcpyHostToDevice));
        ++dst;
        --n;
      }
      if (n) {
        QT_CUDA(qt::launch_serial_normals(ns.src, 0, n, dst, nullptr));
        g_launches.fetch_add(1);
      }
      const GridTables gt = grid_tables(dim, n_points, centers);
      QT_CUDA(cudaMalloc(&dT, gt.blob.size()));
      QT_CUDA(cudaMemcpy(dT, gt.blob.data(), gt.blob.size(), cudaMemcpyHostToDevice));
      QT_CUDA(project_on_device(dim, gt, dT, dX, samples, dcell, nullptr));
      std::vector<double> X(total);
      std::vector<unsigned long long> cell(samples);
      QT_CUDA(cudaMemcpy(X.data(), dX, total * 8, cudaMemcpyDeviceToHost));
      QT_CUDA(cudaMemcpy(cell.data(), dcell, samples * 8, cudaMemcpyDeviceToHost));
      double sum = 0.0, sum_sq = 0.0;
      for (uint64_t m = 0; m < samples; ++m) {
        const double* x = X.data() + m * d;
        const double* c = centers + cell[m] * d;
        double d2 = 0.0;  // squared_distance (grid.hpp:65-72), coordinate order from 0.0
        for (uint64_t j = 0; j < d; ++j) {
          volatile double t = x[j] - c[j];  // volatile: no contraction
          volatile double tt = t * t;
          d2 = d2 + tt;
        }
        sum += d2;
        volatile double sq = d2 * d2;
        sum_sq += sq;
      }
      const double mu = sum / static_cast<double>(samples);
      const double var = std::max(0.0, sum_sq / static_cast<double>(samples) - mu * mu);
      *mean = mu;
      *std_error = std::sqrt(var / static_cast<double>(samples));
    } catch (...) {
      fin();
      throw;
    }
    fin();
    advance_stream(ns, total, state6, has_spare, spare);
  });
}

// estimate_pi_partitioned (monte_carlo.hpp:51-77) on the GPU
QT_API qt_status qt_bench_pi(int32_t engine, uint64_t seed, uint64_t samples, uint64_t streams,
                             int32_t skip_ahead, uint64_t* inside, double* estimate,
                             double* std_error, double* ms) {
  return guarded([&] {
    if (engine < 0 || engine > 2) raise(QT_ERR_CONFIG, "bench-rng: unknown engine");
    if (streams == 0) raise(QT_ERR_INVALID_ARGUMENT, "estimate_pi_partitioned: streams must be >= 1");
    if (samples == 0 || samples % (2 * streams) != 0)
      raise(QT_ERR_INVALID_ARGUMENT,
            "estimate_pi_partitioned: sample count must be a positive multiple of 2*streams");
    if (engine == QT_ENGINE_XORWOW && skip_ahead && streams > 1)
      raise(QT_ERR_INVALID_ARGUMENT, "split_stream: skip-ahead is unsupported for xorwow");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    const int dev0 = qt::current_device();  // the caller's device
    const qt::SrcArgs a = make_src(dev0, engine, seed, 1, 1, nullptr, 0);
    unsigned long long* d = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto fin = [&] {
      cudaFree(d);
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
    };
    try {
      QT_CUDA(cudaMalloc(&d, 8));
      QT_CUDA(cudaMemset(d, 0, 8));
      QT_CUDA(cudaEventCreate(&e0));
      QT_CUDA(cudaEventCreate(&e1));
      QT_CUDA(cudaEventRecord(e0));
      QT_CUDA(qt::launch_pi(engine, skip_ahead, a, samples, streams, d, nullptr));
      QT_CUDA(cudaEventRecord(e1));
      g_launches.fetch_add(1);
      unsigned long long in = 0;
      QT_CUDA(cudaMemcpy(&in, d, 8, cudaMemcpyDeviceToHost));
      float t = 0;
      QT_CUDA(cudaEventElapsedTime(&t, e0, e1));
      const uint64_t points = samples / 2;  // pi_from_counts (monte_carlo.hpp:31-35)
      const double est = 4.0 * static_cast<double>(in) / static_cast<double>(points);
      if (inside) *inside = in;
      if (estimate) *estimate = est;
      if (std_error) *std_error = std::sqrt(est * (4.0 - est) / static_cast<double>(points));
      if (ms) *ms = t;
    } catch (...) {
      fin();
      throw;
    }
    fin();
  });
}

// `qtree bench-nn` (qtree_main.cpp:162-191): a 2-D grid of n standard-normal
// points and `queries` standard-normal queries from one MRG32k3a stream seeded
// `seed`, every query projected on the GPU; *sink = sum of the indices (the
// CLI prints sink % 7), *ms = device time of the searches only.
QT_API qt_status qt_bench_nn(uint64_t n, uint64_t queries, uint64_t seed, uint64_t* sink,
                             double* ms) {
  return guarded([&] {
    if (n == 0 || queries == 0) raise(QT_ERR_INVALID_ARGUMENT, "bench-nn: n and queries must be >= 1");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    const int dev0 = qt::current_device();  // the caller's device
    const qt::SrcArgs a = make_src(dev0, QT_ENGINE_MRG32K3A, seed, 1, 1, nullptr, 0);
    std::vector<void*> bufs;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto fin = [&] {
      for (void* p : bufs) cudaFree(p);
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
    };
    try {
      auto dalloc = [&](size_t b) {
        void* p = nullptr;
        QT_CUDA(cudaMalloc(&p, b));
        bufs.push_back(p);
        return p;
      };
      auto* dp = static_cast<double*>(dalloc(2 * n * 8));
      auto* dq = static_cast<double*>(dalloc(2 * queries * 8));
      auto* di = static_cast<unsigned long long*>(dalloc(queries * 8));
      auto* ds = static_cast<unsigned long long*>(dalloc(8));
      QT_CUDA(qt::launch_serial_normals(a, 0, 2 * n, dp, nullptr));
      QT_CUDA(qt::launch_serial_normals(a, 2 * n, 2 * queries, dq, nullptr));
      std::vector<double> hp(2 * n);
      QT_CUDA(cudaMemcpy(hp.data(), dp, 2 * n * 8, cudaMemcpyDeviceToHost));
      check_grid(2, n, hp.data(), 0);
      const GridTables gt = grid_tables(2, n, hp.data());
      auto* dt = static_cast<uint8_t*>(dalloc(gt.blob.size()));
      QT_CUDA(cudaMemcpy(dt, gt.blob.data(), gt.blob.size(), cudaMemcpyHostToDevice));
      QT_CUDA(cudaMemset(ds, 0, 8));
      QT_CUDA(cudaEventCreate(&e0));
      QT_CUDA(cudaEventCreate(&e1));
      QT_CUDA(cudaEventRecord(e0));
      QT_CUDA(project_on_device(2, gt, dt, dq, queries, di, nullptr));
      QT_CUDA(cudaEventRecord(e1));
      QT_CUDA(qt::launch_sum_u64(di, queries, ds, nullptr));
      g_launches.fetch_add(5);
      unsigned long long s = 0;
      QT_CUDA(cudaMemcpy(&s, ds, 8, cudaMemcpyDeviceToHost));
      float t = 0;
      QT_CUDA(cudaEventElapsedTime(&t, e0, e1));
      if (sink) *sink = s;
      if (ms) *ms = t;
    } catch (...) {
      fin();
      throw;
    }
    fin();
  });
}

QT_API qt_status qt_nearest(int32_t dim, uint64_t n_points, const double* points,
                            uint64_t n_queries, const double* queries, uint64_t* out) {
  return guarded([&] {
    if (dim < 1 || dim > 3) raise(QT_ERR_INVALID_ARGUMENT, "nearest: dimension must be 1..3");
    if (!points || (!queries && n_queries) || (!out && n_queries))
      raise(QT_ERR_INVALID_ARGUMENT, "nearest: null argument");
    check_grid(dim, n_points, points, 0);
    if (n_queries == 0) return;
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    const GridTables gt = grid_tables(dim, n_points, points);
    const std::vector<uint8_t>& t = gt.blob;
    uint8_t* d_t = nullptr;
    double* d_q = nullptr;
    unsigned long long* d_o = nullptr;
    auto fin = [&] {
      cudaFree(d_t);
      cudaFree(d_q);
      cudaFree(d_o);
    };
    try {
      QT_CUDA(cudaMalloc(&d_t, t.size()));
      QT_CUDA(cudaMalloc(&d_q, n_queries * dim * sizeof(double)));
      QT_CUDA(cudaMalloc(&d_o, n_queries * sizeof(uint64_t)));
      QT_CUDA(cudaMemcpy(d_t, t.data(), t.size(), cudaMemcpyHostToDevice));
      QT_CUDA(cudaMemcpy(d_q, queries, n_queries * dim * sizeof(double), cudaMemcpyHostToDevice));
      QT_CUDA(project_on_device(dim, gt, d_t, d_q, n_queries, d_o, nullptr));
      g_launches.fetch_add(1);
      QT_CUDA(cudaMemcpy(out, d_o, n_queries * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    } catch (...) {
      fin();
      throw;
    }
    fin();
  });
}

QT_API qt_status qt_path_normals(int32_t engine, uint64_t seed, uint64_t normals_per_path,
                                 uint64_t first, uint64_t count, double* out) {
  return guarded([&] {
    source_of(engine, false);
    if (count == 0) return;
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    const int dev0 = qt::current_device();  // the caller's device
    auto a = make_src(dev0, engine, seed, 2 * ((normals_per_path + 1) / 2),
                      static_cast<uint32_t>(normals_per_path), nullptr, 0);
    double* d = nullptr;
    QT_CUDA(cudaMalloc(&d, count * normals_per_path * sizeof(double)));
    cudaError_t e = qt::launch_path_normals(engine, a, first, count, d, nullptr);
    g_launches.fetch_add(1);
    if (e == cudaSuccess)
      e = cudaMemcpy(out, d, count * normals_per_path * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    QT_CUDA(e);
  });
}

QT_API qt_status qt_uniforms(int32_t engine, uint64_t seed, uint64_t offset, uint64_t count,
                             double* out) {
  return guarded([&] {
    if (engine != QT_ENGINE_MRG32K3A && engine != QT_ENGINE_LCG48)
      raise(QT_ERR_INVALID_ARGUMENT, "uniforms: jumpable engines only");
    if (count == 0) return;
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    const int dev0 = qt::current_device();  // the caller's device
    auto a = make_src(dev0, engine, seed, 1, 1, nullptr, 0);
    double* d = nullptr;
    QT_CUDA(cudaMalloc(&d, count * sizeof(double)));
    cudaError_t e = qt::launch_uniforms(engine, a, offset, count, d, nullptr);
    g_launches.fetch_add(1);
    if (e == cudaSuccess) e = cudaMemcpy(out, d, count * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    QT_CUDA(e);
  });
}

// 1-D kernel selection (mode1d): 0 exact, 1 FP32 fast path, 2 certified FP64 (default)
QT_API qt_status qt_set_fast_path(int32_t mode) {
  return guarded([&] {
    if (mode < 0 || mode > 2) raise(QT_ERR_INVALID_ARGUMENT, "set_fast_path: mode must be 0, 1 or 2");
    g_fast.store(mode);
  });
}

// Exhaustive bound check of the certified kernel's approximate Box-Muller
// (qt_math_fast.h) against the glibc-exact one: out[0..3] as k_apx_bounds_check,
// out[4..6] = the bounds the kernel uses (kApxRadRel, kApxAng, kApxZ).
QT_API qt_status qt_apx_bounds_check(double* out) {
  return guarded([&] {
    if (!out) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    unsigned long long* d = nullptr;
    QT_CUDA(cudaMalloc(&d, 4 * sizeof(unsigned long long)));
    cudaError_t e = cudaMemset(d, 0, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = qt::launch_apx_bounds_check(d, nullptr);
    unsigned long long h[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    QT_CUDA(e);
    g_launches.fetch_add(1);
    for (int i = 0; i < 4; ++i) std::memcpy(out + i, h + i, 8);
    out[4] = qt::apx::kApxRadRel;
    out[5] = qt::apx::kApxAng;
    out[6] = qt::apx::kApxZ;
  });
}

QT_API qt_status qt_fast_stats(uint64_t* out) {
  return guarded([&] {
    if (!out) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    out[0] = g_fast_paths.load();
    out[1] = g_fast_replayed.load();
    out[2] = g_fast_inline.load();
    // plus the plans still held by the one-call cache (destroyed plans add theirs above)
    PlanCache& c = plan_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    for (const auto& it : c.items) {
      const qt_plan* pl = it.second.get();
      if (!pl->d_stats) continue;
      unsigned long long st[3] = {0, 0, 0};
      QT_CUDA(cudaSetDevice(pl->device));
      QT_CUDA(cudaDeviceSynchronize());
      QT_CUDA(cudaMemcpy(st, pl->d_stats, sizeof st, cudaMemcpyDeviceToHost));
      out[0] += pl->fast_paths;
      out[1] += st[1];
      out[2] += st[2];
    }
  });
}

QT_API qt_status qt_plan_fast_stats(const qt_plan* plan, uint64_t* out) {
  return guarded([&] {
    if (!plan || !out) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    unsigned long long st[3] = {0, 0, 0};
    if (plan->d_stats) {
      QT_CUDA(cudaSetDevice(plan->device));
      QT_CUDA(cudaDeviceSynchronize());
      QT_CUDA(cudaMemcpy(st, plan->d_stats, sizeof st, cudaMemcpyDeviceToHost));
    }
    out[0] = plan->fast_paths;
    out[1] = st[1];
    out[2] = st[2];
  });
}

QT_API qt_status qt_fast_bounds_check(double* out) {
  return guarded([&] {
    if (!out) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    unsigned int* d = nullptr;
    QT_CUDA(cudaMalloc(&d, 4 * sizeof(unsigned int)));
    cudaError_t e = cudaMemset(d, 0, 4 * sizeof(unsigned int));
    if (e == cudaSuccess) e = qt::launch_fast_bounds_check(d, nullptr);
    unsigned int h[4] = {0, 0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    QT_CUDA(e);
    g_launches.fetch_add(1);
    for (int i = 0; i < 4; ++i) {
      float f;
      std::memcpy(&f, &h[i], 4);
      out[i] = f;
    }
  });
}

QT_API qt_status qt_math_checksum(int32_t domain, uint64_t* out) {
  return guarded([&] {
    if (!out) raise(QT_ERR_INVALID_ARGUMENT, "null argument");
    if (domain != 0 && domain != 1) raise(QT_ERR_INVALID_ARGUMENT, "domain must be 0 or 1");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
      raise(QT_ERR_DEVICE, "cuda: no CUDA device available");
    unsigned long long* d = nullptr;
    QT_CUDA(cudaMalloc(&d, 3 * sizeof(unsigned long long)));
    cudaError_t e = cudaMemset(d, 0, 3 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = qt::launch_math_checksum(domain, d, nullptr);
    unsigned long long h[3] = {0, 0, 0};
    if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(d);
    QT_CUDA(e);
    g_launches.fetch_add(1);
    for (int i = 0; i < 3; ++i) out[i] = h[i];
  });
}

// Frees every cached one-call plan (tables and the joint / visits / pi result
// buffers) on whatever device each lives on.
QT_API qt_status qt_plan_cache_clear(void) {
  return guarded([&] {
    std::vector<std::pair<std::vector<uint8_t>, std::unique_ptr<qt_plan>>> drop;
    {
      PlanCache& c = plan_cache();
      std::lock_guard<std::mutex> lk(c.mu);
      drop.swap(c.items);
    }
    drop.clear();
  });
}

QT_API const char* qt_last_error(void) { return g_error.c_str(); }

QT_API const char* qt_version(void) {
  return "qtree_cuda 0.1 sm_100a (fused MRG32k3a/LCG48/XORWOW path kernel, cp.async.bulk tables)";
}

QT_API uint64_t qt_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"
