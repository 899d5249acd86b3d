// qt_device.cuh -- device building blocks of the fused path kernel:
// the three reference RNG engines with O(log s) positioning, Box-Muller,
// the chain steps, the exact Voronoi projection and the async-copy helpers.
//
// Every floating-point expression that mirrors reference arithmetic uses the
// explicitly rounded intrinsics (__dadd_rn / __dsub_rn / __dmul_rn), which the
// compiler never contracts into FMA: the reference is built without FMA
// contraction (SURVEY.md §7 hard part 1), and bit-exact cell indices need every
// product and sum rounded exactly as it rounds there.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "qt_internal.h"
#include "qt_layout.h"
#include "qt_math.h"

namespace qt {

// ---------------------------------------------------------------------------
// MRG32k3a (rng/mrg32k3a.hpp:8-63). State words are residues < 2^32, kept in
// u32 registers; each recurrence is one 32x32->64 multiply-add pair plus a
// two-fold reduction by 2^32 = m + c, which yields the same residue as the
// reference's signed-64 `%` + fix-up.
// ---------------------------------------------------------------------------
constexpr uint32_t kM1 = 4294967087u;
constexpr uint32_t kM2 = 4294944443u;
constexpr uint32_t kC1 = 209u;    // 2^32 - m1
constexpr uint32_t kC2 = 22853u;  // 2^32 - m2
constexpr uint32_t kA12 = 1403580u, kA13n = 810728u, kA21 = 527612u, kA23n = 1370589u;
// (double)(m1 + 1): the uniform is (x + 1) / (m1 + 1), mrg32k3a.hpp:62
constexpr double kM1p1 = 4294967088.0;
constexpr double kInvM1p1 = 1.0 / 4294967088.0;

struct Mrg {
  uint32_t a0, a1, a2;  // s1 = (x_{n-3}, x_{n-2}, x_{n-1})
  uint32_t b0, b1, b2;  // s2
};

__device__ __forceinline__ uint64_t mulw(uint32_t a, uint32_t b) {
  return static_cast<uint64_t>(a) * static_cast<uint64_t>(b);
}

// t mod m1 for any t < 2^64
__device__ __forceinline__ uint32_t red_m1(uint64_t t) {
  uint64_t r = mulw(static_cast<uint32_t>(t >> 32), kC1) + (t & 0xffffffffull);
  r = mulw(static_cast<uint32_t>(r >> 32), kC1) + (r & 0xffffffffull);
  return static_cast<uint32_t>(r >= kM1 ? r - kM1 : r);
}
// t mod m2 for any t < 2^64
__device__ __forceinline__ uint32_t red_m2(uint64_t t) {
  uint64_t r = mulw(static_cast<uint32_t>(t >> 32), kC2) + (t & 0xffffffffull);
  r = mulw(static_cast<uint32_t>(r >> 32), kC2) + (r & 0xffffffffull);
  return static_cast<uint32_t>(r >= kM2 ? r - kM2 : r);
}

// One step of both recurrences; returns the combined integer x in [0, m1).
__device__ __forceinline__ uint32_t mrg_step(Mrg& s) {
  // p1 = (a12 s1[1] - a13n s1[0]) mod m1, made non-negative by + a13n m1
  const uint32_t p1 = red_m1(mulw(kA12, s.a1) + mulw(kA13n, kM1 - s.a0));
  s.a0 = s.a1;
  s.a1 = s.a2;
  s.a2 = p1;
  // p2 = (a21 s2[2] - a23n s2[0]) mod m2
  const uint32_t p2 = red_m2(mulw(kA21, s.b2) + mulw(kA23n, kM2 - s.b0));
  s.b0 = s.b1;
  s.b1 = s.b2;
  s.b2 = p2;
  return p1 >= p2 ? p1 - p2 : p1 - p2 + kM1;  // mod-2^32 wrap gives the exact value
}

// Two consecutive outputs (x1 then x2) with the residues reduced by
// min_u32(r, r - m): r - m wraps above r exactly when r < m.
__device__ __forceinline__ uint32_t fold_m1(uint64_t t) {  // t < 2^54
  const uint64_t r = mulw(static_cast<uint32_t>(t >> 32), kC1) + static_cast<uint32_t>(t);
  const uint32_t r2 = static_cast<uint32_t>(r) + static_cast<uint32_t>(r >> 32) * kC1;
  return min(r2, r2 - kM1);
}
__device__ __forceinline__ uint32_t fold_m2(uint64_t t) {  // t < 2^54
  const uint64_t r = mulw(static_cast<uint32_t>(t >> 32), kC2) + static_cast<uint32_t>(t);
  const uint64_t r2 = mulw(static_cast<uint32_t>(r >> 32), kC2) + static_cast<uint32_t>(r);
  const uint32_t r3 = static_cast<uint32_t>(r2) + static_cast<uint32_t>(r2 >> 32) * kC2;
  return min(r3, r3 - kM2);
}
__device__ __forceinline__ void mrg_step2(Mrg& s, uint32_t& x1, uint32_t& x2) {
  // component 1: x_n = a12 x_{n-2} - a13n x_{n-3}; the two new values are independent
  const uint32_t p1 = fold_m1(mulw(kA12, s.a1) + mulw(kA13n, kM1 - s.a0));
  const uint32_t q1 = fold_m1(mulw(kA12, s.a2) + mulw(kA13n, kM1 - s.a1));
  // component 2: x_n = a21 x_{n-1} - a23n x_{n-3}
  const uint32_t p2 = fold_m2(mulw(kA21, s.b2) + mulw(kA23n, kM2 - s.b0));
  const uint32_t q2 = fold_m2(mulw(kA21, p2) + mulw(kA23n, kM2 - s.b1));
  s.a0 = s.a2;
  s.a1 = p1;
  s.a2 = q1;
  s.b0 = s.b2;
  s.b1 = p2;
  s.b2 = q2;
  x1 = p1 >= p2 ? p1 - p2 : p1 - p2 + kM1;
  x2 = q1 >= q2 ? q1 - q2 : q1 - q2 + kM1;
}

// (x + 1) / (m1 + 1), correctly rounded. Division by the constant is done as
// q = RN(a R); r = a - q d (exact, FMA); RN(q + r R): tests/test_division.py
// proves it equals the IEEE quotient for all 2^32 possible numerators.
__device__ __forceinline__ double mrg_to_unit(uint32_t x) {
  const double a = __uint2double_rn(x + 1u);
#if defined(QT_PLAIN_DIVISION)
  return __ddiv_rn(a, kM1p1);
#else
  const double q = __dmul_rn(a, kInvM1p1);
  const double r = __fma_rn(-q, kM1p1, a);
  return __fma_rn(r, kInvM1p1, q);
#endif
}

// 3x3 matrix (mod m) times state; the jump table holds J^(2^b) for b = 0..63
// (rows of u32 residues, [b][component][3][3]).
__device__ __forceinline__ void mat_apply_m1(const uint32_t* J, uint32_t& x0, uint32_t& x1,
                                             uint32_t& x2) {
  uint32_t r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint64_t acc = static_cast<uint64_t>(red_m1(mulw(__ldg(J + 3 * i + 0), x0))) +
                         red_m1(mulw(__ldg(J + 3 * i + 1), x1)) +
                         red_m1(mulw(__ldg(J + 3 * i + 2), x2));
    r[i] = red_m1(acc);
  }
  x0 = r[0];
  x1 = r[1];
  x2 = r[2];
}
__device__ __forceinline__ void mat_apply_m2(const uint32_t* J, uint32_t& x0, uint32_t& x1,
                                             uint32_t& x2) {
  uint32_t r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint64_t acc = static_cast<uint64_t>(red_m2(mulw(__ldg(J + 3 * i + 0), x0))) +
                         red_m2(mulw(__ldg(J + 3 * i + 1), x1)) +
                         red_m2(mulw(__ldg(J + 3 * i + 2), x2));
    r[i] = red_m2(acc);
  }
  x0 = r[0];
  x1 = r[1];
  x2 = r[2];
}

// state <- J^e state (mrg32k3a_skip, mrg32k3a.hpp:124-146): one table entry
// J^(d 16^w) per non-zero hex digit d of e (the table is mrg_jump_table, qt_capi.cu)
__device__ __forceinline__ void mrg_jump(Mrg& s, uint64_t e, const uint32_t* table) {
  for (int w = 0; e != 0; ++w, e >>= 4) {
    const uint32_t d = static_cast<uint32_t>(e & 15u);
    if (d) {
      const uint32_t* J = table + (15u * w + d - 1u) * 18u;
      mat_apply_m1(J, s.a0, s.a1, s.a2);
      mat_apply_m2(J + 9, s.b0, s.b1, s.b2);
    }
  }
}

// ---------------------------------------------------------------------------
// LCG48 (rng/lcg48.hpp): x <- a x + c mod 2^48, u = x 2^-48. Jump table holds
// the affine maps of 2^b steps, [b] = (A, C).
// ---------------------------------------------------------------------------
constexpr uint64_t kLcgMask = (1ull << 48) - 1;
constexpr uint64_t kLcgA = 0x5DEECE66Dull;
constexpr uint64_t kLcgC = 0xBull;

__device__ __forceinline__ double lcg_uniform(uint64_t& x) {
  x = (kLcgA * x + kLcgC) & kLcgMask;
  return __ull2double_rn(x) * 0x1p-48;
}

__device__ __forceinline__ void lcg_jump(uint64_t& x, uint64_t e, const unsigned long long* table) {
  for (int b = 0; e != 0; ++b, e >>= 1)
    if (e & 1ull) x = (__ldg(table + 2 * b) * x + __ldg(table + 2 * b + 1)) & kLcgMask;
}

// ---------------------------------------------------------------------------
// XORWOW (rng/xorwow.hpp:16-47), re-seeded per path with 64 burn-in steps
// (stream.hpp:146-153,207-209).
// ---------------------------------------------------------------------------
struct Xorwow {
  uint32_t v, w, x, y, z, d;
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t& z) {
  z += 0x9E3779B97F4A7C15ull;
  uint64_t v = z;
  v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ull;
  v = (v ^ (v >> 27)) * 0x94D049BB133111EBull;
  return v ^ (v >> 31);
}

__device__ __forceinline__ uint32_t xorwow_step(Xorwow& s) {
  const uint32_t t = s.x ^ (s.x >> 2);
  s.x = s.y;
  s.y = s.z;
  s.z = s.w;
  s.w = s.v;
  s.v = (s.v ^ (s.v << 4)) ^ (t ^ (t << 1));
  s.d += 362437u;
  return s.v + s.d;
}

__device__ __forceinline__ Xorwow xorwow_stream(uint64_t seed, uint64_t stream) {
  uint64_t z = seed ^ (0x9E3779B97F4A7C15ull * (stream + 1));
  const uint64_t a = splitmix64(z), b = splitmix64(z), c = splitmix64(z);
  Xorwow s{static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32), static_cast<uint32_t>(b),
           static_cast<uint32_t>(b >> 32), static_cast<uint32_t>(c),
           static_cast<uint32_t>(c >> 32)};
  if ((s.v | s.w | s.x | s.y | s.z) == 0) s.v = 1;
  for (int i = 0; i < 64; ++i) xorwow_step(s);
  return s;
}

// ---------------------------------------------------------------------------
// Box-Muller (stream.hpp:57-62): r = sqrt(-2 log u1), a = 2 pi u2,
// (r cos a, r sin a); u1 <= 0 clamps to 2^-64. sqrt and the products are
// correctly rounded like the host's; log and sincos are qt_math.h's
// restatements of the glibc __log_fma / __sincos_fma the reference calls,
// bit-identical on every engine's uniforms (tests/tools/check_math.cpp:
// exhaustive over MRG32k3a and XORWOW, sampled over LCG48), so the normals --
// and with them the counts -- are the reference's by construction.
// ---------------------------------------------------------------------------
constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi, exact doubling

__device__ __forceinline__ void box_muller(double u1, double u2, double& z1, double& z2) {
  if (u1 <= 0.0) u1 = 0x1p-64;
  const double r = __dsqrt_rn(__dmul_rn(-2.0, qt_log_unit(u1)));
  const double a = __dmul_rn(kTwoPi, u2);
  double s, c;
  qt_sincos_2pi(a, &s, &c);
  z1 = __dmul_rn(r, c);
  z2 = __dmul_rn(r, s);
}

// box_muller() for P independent pairs, in sweeps: the log-table loads of
// every pair first, then sincos (independent of them), then the log table
// path. The 6 % of radii with u1 in [1 - 2^-4, 1) take glibc's separate
// near-1 polynomial; those are evaluated afterwards in a loop that runs once
// per near-1 pair of the lane (max over the warp, usually one pass) instead of
// once per pair index. Same operations, same bits as box_muller().
template <int P>
__device__ __forceinline__ void box_muller_batch(const double (&u1)[P], const double (&u2)[P],
                                                 double (&z1)[P], double (&z2)[P]) {
  LogPrep lp[P];
  double v[P], ang[P], sn[P], cs[P], lg[P];
  unsigned near = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    v[p] = u1[p] <= 0.0 ? 0x1p-64 : u1[p];
    lp[p] = qt_log_prep(v[p]);
    near |= qt_log_near1(v[p]) ? (1u << p) : 0u;
    ang[p] = __dmul_rn(kTwoPi, u2[p]);
  }
#pragma unroll
  for (int p = 0; p < P; ++p) qt_sincos_2pi(ang[p], &sn[p], &cs[p]);
#pragma unroll
  for (int p = 0; p < P; ++p) lg[p] = qt_log_finish(lp[p]);
  while (near) {
    const int q = __ffs(near) - 1;
    double x = v[0];
#pragma unroll
    for (int p = 1; p < P; ++p) x = q == p ? v[p] : x;
    const double l = qt_log_near1_eval(x);
#pragma unroll
    for (int p = 0; p < P; ++p) lg[p] = q == p ? l : lg[p];
    near &= near - 1;
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const double r = __dsqrt_rn(__dmul_rn(-2.0, lg[p]));
    z1[p] = __dmul_rn(r, cs[p]);
    z2[p] = __dmul_rn(r, sn[p]);
  }
}

// ---------------------------------------------------------------------------
// FP32 Box-Muller of the fast 1-D path (MRG32k3a only). It never decides a
// cell by itself: it yields z~ together with a rigorous bound
// |z~ - z| <= bz(r~) against the exact FP64 normal z of box_muller() above, and
// the path kernel only counts a transition whose FP64 state interval
// [x~ - e, x~ + e] lies strictly inside one cell. The bound constants below
// are verified over ALL 2^32 MRG32k3a outputs by k_fast_bounds_check
// (qt_fast_bounds_check, tests/test_gpu_parity.py), with the composition
// |r~c~ - rc| <= |r~-r| |c~| + r |c~-c| + 2^-24 |z~| done analytically.
// Every FP32 operation is an explicitly rounded intrinsic or an .approx
// instruction (deterministic MUFU), so the kernel and the checker compute the
// same bits.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float mufu_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_sin(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_cos(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// radius bound |r~ - r| <= kRadA + kRadB r~ ; angle bound |c~ - c|, |s~ - s| <= kAng
constexpr float kRadA = 2.2e-7f;
constexpr float kRadB = 1.6e-7f;
constexpr float kAng = 5.5e-7f;
// bz = kBzA + kBzB r~ >= kRadA (1 + kAng) + r~ ((kRadB (1 + kAng) + kAng + 2^-23)
// (rounded up generously; |c~| <= 1 is also checked exhaustively)
constexpr float kBzA = 2.21e-7f;
constexpr float kBzB = 7.75e-7f;

// r~ = sqrt(-2 ln u), u = (x + 1) / (m1 + 1), from the MRG32k3a integer x
__device__ __forceinline__ float fast_radius(uint32_t x) {
  const uint32_t v = kM1 - x;  // (m1 + 1) (1 - u), in (0, m1]
  const float uf = __fmul_rn(__uint2float_rn(x + 1u), 0x1p-32f);
  const float wf = __fmul_rn(__uint2float_rn(v), 0x1p-32f);
  const bool lower = x < 2147483544u;  // u < 1/2: log of u itself
  const float t = __fsub_rn(1.0f, wf);
  const float L = mufu_lg2(lower ? uf : t);
  // u < 1/2: -2 ln2 (log2(x+1) - 32 + log2(2^32 / (m1 + 1)))
  const float RA = __fmaf_rn(L, -1.3862943611198906f, -9.6853e-8f);
  // 1/8 < w <= 1/2: log1p(-w) = ln(t) w / (1 - t) corrects the rounding of t
  const float RB = __fmul_rn(__fmul_rn(L, -1.3862943611198906f), __fmul_rn(wf, mufu_rcp(__fsub_rn(1.0f, t))));
  // w <= 1/8: -2 ln(1 - w) = 2 w (1 + w/2 + ... + w^6/7)
  float P = __fmaf_rn(wf, 0.14285714285714285f, 0.16666666666666666f);
  P = __fmaf_rn(wf, P, 0.2f);
  P = __fmaf_rn(wf, P, 0.25f);
  P = __fmaf_rn(wf, P, 0.3333333333333333f);
  P = __fmaf_rn(wf, P, 0.5f);
  P = __fmaf_rn(wf, P, 1.0f);
  const float RS = __fmul_rn(__fmul_rn(2.0f, wf), P);
  return mufu_sqrt(lower ? RA : (wf <= 0.125f ? RS : RB));
}

// (c~, s~) = (cos, sin)(2 pi u) as -(cos, sin)(2 pi (u - 1/2))
__device__ __forceinline__ void fast_angle(uint32_t x, float& c, float& s) {
  const int d = static_cast<int>(x + 1u - 2147483544u);  // (m1 + 1)(u - 1/2), exact
  const float a = __fmul_rn(__int2float_rn(d), 1.4629180792671596e-09f);  // 2 pi / (m1 + 1)
  c = -mufu_cos(a);
  s = -mufu_sin(a);
}

// ---------------------------------------------------------------------------
// Normal sources: one per engine plus the parity-mode reader. Each models a
// PathStreamer positioned at a path (or Alg III sample) and hands out that
// unit's normals in order, Box-Muller mate cached (stream.hpp:97-108) and
// dropped at the unit boundary.
// ---------------------------------------------------------------------------
enum : int { kSrcLcg48 = 0, kSrcMrg = 1, kSrcXorwow = 2, kSrcNormalsIn = 3 };

// SrcArgs (engine seeds, jump tables, parity-mode normals) lives in qt_internal.h.


template <int SRC>
struct Source;

template <>
struct Source<kSrcMrg> {
  Mrg s;
  double spare;
  bool has;
  // Position at the first draw of `unit` (unit * draws serial draws in).
  __device__ __forceinline__ void start(const SrcArgs& a, uint64_t unit) {
    s = Mrg{a.mrg_seed[0], a.mrg_seed[1], a.mrg_seed[2], a.mrg_seed[3], a.mrg_seed[4], a.mrg_seed[5]};
    mrg_jump(s, unit * a.draws, a.mrg_table);
    has = false;
  }
  // Units are contiguous blocks of the serial stream, so after a unit has
  // consumed its `draws` uniforms the state already sits on the next unit.
  __device__ __forceinline__ void next_unit(const SrcArgs&, uint64_t) { has = false; }
  __device__ __forceinline__ double uniform() { return mrg_to_unit(mrg_step(s)); }
  __device__ __forceinline__ double normal() {
    if (has) {
      has = false;
      return spare;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    double z1;
    box_muller(u1, u2, z1, spare);
    has = true;
    return z1;
  }
};

template <>
struct Source<kSrcLcg48> {
  uint64_t x;
  double spare;
  bool has;
  __device__ __forceinline__ void start(const SrcArgs& a, uint64_t unit) {
    x = a.lcg_seed;
    lcg_jump(x, unit * a.draws, a.lcg_table);
    has = false;
  }
  __device__ __forceinline__ void next_unit(const SrcArgs&, uint64_t) { has = false; }
  __device__ __forceinline__ double uniform() { return lcg_uniform(x); }
  __device__ __forceinline__ double normal() {
    if (has) {
      has = false;
      return spare;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    double z1;
    box_muller(u1, u2, z1, spare);
    has = true;
    return z1;
  }
};

template <>
struct Source<kSrcXorwow> {
  Xorwow s;
  double spare;
  bool has;
  __device__ __forceinline__ void start(const SrcArgs& a, uint64_t unit) {
    s = xorwow_stream(a.seed, unit);
    has = false;
  }
  __device__ __forceinline__ void next_unit(const SrcArgs& a, uint64_t unit) { start(a, unit); }
  __device__ __forceinline__ double uniform() {
    return __uint2double_rn(xorwow_step(s)) * 0x1p-32;
  }
  __device__ __forceinline__ double normal() {
    if (has) {
      has = false;
      return spare;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    double z1;
    box_muller(u1, u2, z1, spare);
    has = true;
    return z1;
  }
};

template <>
struct Source<kSrcNormalsIn> {
  const double* p;
  __device__ __forceinline__ void start(const SrcArgs& a, uint64_t unit) {
    p = a.normals + (unit - a.normals_first) * a.per_unit;
  }
  __device__ __forceinline__ void next_unit(const SrcArgs& a, uint64_t unit) { start(a, unit); }
  __device__ __forceinline__ double normal() { return __ldg(p++); }
};

// ---------------------------------------------------------------------------
// Chains (model/chains.hpp). K = qt_chain_kind.
// ---------------------------------------------------------------------------
template <int K>
struct Chain;

template <>
struct Chain<0> {  // BrownianChain1d: x + sqrt(dt) eps (chains.hpp:83-86)
  static constexpr int D = 1, NPS = 1;
  __device__ __forceinline__ static void step(const double* c, const double* x, double* o,
                                              const double* e) {
    o[0] = __dadd_rn(x[0], __dmul_rn(c[0], e[0]));
  }
  __device__ __forceinline__ static void marginal(const double* m, bool origin, double* o,
                                                  const double* e) {
    o[0] = origin ? 0.0 : __dmul_rn(m[0], e[0]);  // k == 0 -> exactly 0 (chains.hpp:89)
  }
};

template <>
struct Chain<1> {  // TwoFactorChain (chains.hpp:48-59)
  static constexpr int D = 2, NPS = 2;
  __device__ __forceinline__ static void step(const double* c, const double* x, double* o,
                                              const double* e) {
    o[0] = __dadd_rn(__dmul_rn(c[0], x[0]), __dmul_rn(c[2], e[0]));
    o[1] = __dadd_rn(__dadd_rn(__dmul_rn(c[1], x[1]), __dmul_rn(c[3], e[0])),
                     __dmul_rn(c[4], e[1]));
  }
  __device__ __forceinline__ static void marginal(const double* m, bool, double* o,
                                                  const double* e) {
    o[0] = __dmul_rn(m[0], e[0]);
    o[1] = __dadd_rn(__dmul_rn(m[1], e[0]), __dmul_rn(m[2], e[1]));
  }
};

template <>
struct Chain<2> {  // OU 1-D = factor 1 of TwoFactorChain
  static constexpr int D = 1, NPS = 1;
  __device__ __forceinline__ static void step(const double* c, const double* x, double* o,
                                              const double* e) {
    o[0] = __dadd_rn(__dmul_rn(c[0], x[0]), __dmul_rn(c[2], e[0]));
  }
  __device__ __forceinline__ static void marginal(const double* m, bool, double* o,
                                                  const double* e) {
    o[0] = __dmul_rn(m[0], e[0]);
  }
};

template <>
struct Chain<3> {  // GBM 3-D basket log-state
  static constexpr int D = 3, NPS = 3;
  __device__ __forceinline__ static void step(const double* c, const double* x, double* o,
                                              const double* e) {
    o[0] = __dadd_rn(x[0], __dmul_rn(c[0], e[0]));
    o[1] = __dadd_rn(x[1], __dadd_rn(__dmul_rn(c[1], e[0]), __dmul_rn(c[2], e[1])));
    o[2] = __dadd_rn(x[2], __dadd_rn(__dadd_rn(__dmul_rn(c[3], e[0]), __dmul_rn(c[4], e[1])),
                                     __dmul_rn(c[5], e[2])));
  }
  __device__ __forceinline__ static void marginal(const double* m, bool, double* o,
                                                  const double* e) {
    o[0] = __dmul_rn(m[0], e[0]);
    o[1] = __dadd_rn(__dmul_rn(m[1], e[0]), __dmul_rn(m[2], e[1]));
    o[2] = __dadd_rn(__dadd_rn(__dmul_rn(m[3], e[0]), __dmul_rn(m[4], e[1])),
                     __dmul_rn(m[5], e[2]));
  }
};

// ---------------------------------------------------------------------------
// Voronoi projection (nearest_brute, nn.hpp:18-46): exact argmin of the
// reference's d2, smallest original index on ties.
// ---------------------------------------------------------------------------

// Exact scan over the sorted records (cold block, global memory) with
// (d2, original index) ordering: identical result to the reference's
// ascending strict-< scan for every x, including NaN / +-inf / overflow.
static __device__ __noinline__ uint32_t nearest_1d_scan(const Rec1* R, uint32_t n, double x) {
  uint32_t best = 0;
  double bd = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (uint32_t s = 0; s < n; ++s) {
    const Rec1 r = R[s];
    const double d = __dsub_rn(x, r.v);
    const double d2 = __dmul_rn(d, d);
    if (d2 < bd || (d2 == bd && r.orig < best)) {
      bd = d2;
      best = r.orig;
    }
  }
  return best;
}

// d == 1. The reference's argmin of fl(fl(x - v)^2) over a sorted grid is
// decided by the two values bracketing x, and that pairwise choice (with the
// smallest-index tie rule) flips exactly once on [v_c, v_c+1]: at the FP64
// decision threshold t_c the host finds by bisection over the doubles. So the
// cell is the number of thresholds <= x: one bucket lookup, one 16-byte
// shared-memory record pair, two FP64 compares. Exact whenever |x| < x_safe
// (no same-side d2 ties possible); otherwise (and for NaN/inf)
// the exact scan over the cold block.
__device__ __forceinline__ uint32_t nearest_1d(const LayerTable& h, const uint8_t* base, double x,
                                               const uint8_t* gtables) {
  if (!(fabs(x) < h.x_safe))
    return nearest_1d_scan(reinterpret_cast<const Rec1*>(gtables + h.cold_off), h.n_pts, x);
  const Thr* T = reinterpret_cast<const Thr*>(base + h.off_rec);
  const uint16_t* start = reinterpret_cast<const uint16_t*>(base + h.off_start);
  uint32_t c = start[bucket_of(x, h.lo, h.inv_w, h.nb_d, h.nb)];  // all t_{<c} < x
  const Thr r0 = T[c], r1 = T[c + 1];
  if (x < r0.t) return r0.orig;
  if (x < r1.t) return r1.orig;
  c += 2;
  while (!(x < T[c].t)) ++c;  // t_{N-1} = +inf stops the walk
  return T[c].orig;
}

// d == 2: the reference's fast path dx*dx + dy*dy (nn.hpp:25-37), strict <.
__device__ __forceinline__ uint32_t nearest_2d(const LayerTable& h, const uint8_t* base,
                                               const double* q) {
  const double2* P = reinterpret_cast<const double2*>(base + h.off_rec);
  uint32_t best = 0;
  double bd = __longlong_as_double(0x7ff0000000000000ll);
  const uint32_t n = h.n_pts;
  for (uint32_t i = 0; i < n; ++i) {
    const double2 p = P[i];
    const double dx = __dsub_rn(q[0], p.x);
    const double dy = __dsub_rn(q[1], p.y);
    const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    if (d2 < bd) {
      bd = d2;
      best = i;
    }
  }
  return best;
}

// d == 3: squared_distance accumulated from 0.0 in coordinate order
// (grid.hpp:65-72), strict < (nn.hpp:38-45).
__device__ __forceinline__ uint32_t nearest_3d(const LayerTable& h, const uint8_t* base,
                                               const double* q) {
  const double* P = reinterpret_cast<const double*>(base + h.off_rec);
  uint32_t best = 0;
  double bd = __longlong_as_double(0x7ff0000000000000ll);
  const uint32_t n = h.n_pts;
  for (uint32_t i = 0; i < n; ++i) {
    const double d0 = __dsub_rn(q[0], P[3 * i]);
    const double d1 = __dsub_rn(q[1], P[3 * i + 1]);
    const double d2_ = __dsub_rn(q[2], P[3 * i + 2]);
    double acc = __dadd_rn(0.0, __dmul_rn(d0, d0));
    acc = __dadd_rn(acc, __dmul_rn(d1, d1));
    acc = __dadd_rn(acc, __dmul_rn(d2_, d2_));
    if (acc < bd) {
      bd = acc;
      best = i;
    }
  }
  return best;
}

template <int D>
__device__ __forceinline__ uint32_t nearest(const LayerTable& h, const uint8_t* base,
                                            const double* q, const uint8_t* gtables) {
  if constexpr (D == 1) return nearest_1d(h, base, q[0], gtables);
  else if constexpr (D == 2) return nearest_2d(h, base, q);
  else return nearest_3d(h, base, q);
}

// ---------------------------------------------------------------------------
// Async bulk copy global -> shared with mbarrier completion (TMA bulk path,
// SASS UBLKCP), and the mbarrier primitives.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x100000u)  // suspend (not spin) up to ~1 ms
        : "memory");
  } while (!done);
}

// The same on a precomputed shared-window address (no per-call cvta).
__device__ __forceinline__ void mbar_wait_u32(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x100000u)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// bar.sync on a named barrier among `count` threads (a multiple of 32)
__device__ __forceinline__ void named_barrier_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// bytes must be a multiple of 16, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// No-return 64-bit atomic add (SASS RED.E.ADD.64): the count tally
// `joint[t][i*N_k+j] += 1` (estimate.hpp:118). No "memory" clobber: nothing in
// a path kernel reads the counts, so the compiler may move the next layer's
// shared-memory loads above the RED (the count array is only read after the
// kernel, by later launches).
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v));
}

}  // namespace qt
