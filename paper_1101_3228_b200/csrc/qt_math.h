// qt_math.h -- the Box-Muller transcendentals, bit-identical to the glibc the
// reference calls.
//
// The reference's box_muller (rng/stream.hpp:57-62) computes
//   r = std::sqrt(-2.0 * std::log(u1)),  a = 2 pi u2,  (r cos a, r sin a)
// and g++ -O3 turns the cos/sin pair into ONE sincos() call (objdump of the
// reference build: `call log@plt`, `call sincos@plt`). On x86-64 hosts with
// AVX2 + FMA (this image's CPUs) glibc 2.39 resolves those to __log_fma and
// __sincos_fma: glibc's own C sources (sysdeps/ieee754/dbl-64/e_log.c,
// s_sincos.c with the do_sin/do_cos/reduce_sincos of s_sin.c) compiled with
// -mfma, where GCC fused many `a*b + c` into FMAs. This file restates those
// two functions operation for operation -- the order of every add and which
// products are fused were read off the disassembly of that libm build -- with
// explicitly rounded operations only, so the host build (checked against the
// live libm by tests/tools/check_math.cpp over ALL 2^32 - 209 MRG32k3a
// uniforms) and the device build produce the same bits. Data tables and
// constants: qt_glibc_tab.h (generated from that libm by tools/gen_glibc_tab.c).
//
//   qt_log_unit(x)      == glibc log(x)     for positive normal x (x <= 1 here)
//   qt_sincos_2pi(x,..) == glibc sincos(x)  for |x| < 105414350 (2 pi u2 here)
#pragma once

#if defined(__CUDA_ARCH__)
#define QT_HD __host__ __device__ __forceinline__
#define QT_FMA(a, b, c) __fma_rn((a), (b), (c))
#define QT_MUL(a, b) __dmul_rn((a), (b))
#define QT_ADD(a, b) __dadd_rn((a), (b))
#define QT_SUB(a, b) __dsub_rn((a), (b))
#else
#include <cmath>
#if defined(__CUDACC__)
#define QT_HD __host__ __device__ inline
#else
#define QT_HD inline
#endif
#define QT_FMA(a, b, c) std::fma((a), (b), (c))
#define QT_MUL(a, b) ((a) * (b))
#define QT_ADD(a, b) ((a) + (b))
#define QT_SUB(a, b) ((a) - (b))
#endif

#include <stdint.h>
#include <string.h>

#include "qt_glibc_tab.h"

namespace qt {

#if defined(__CUDACC__)
static __device__ const double2 kGlibcLogTabDev[128] = {QT_GLIBC_LOG_TAB};
// row i = {sn, ssn} at [2i], {cs, ccs} at [2i + 1]
static __device__ const double2 kGlibcSincosTabDev[220] = {QT_GLIBC_SINCOS_TAB};
#endif
// The scalar constants again, as a __constant__ struct on the device: an FP64
// operand read from the constant bank costs no instruction, where a 64-bit
// immediate is first materialised into a uniform register pair (two UMOVs per
// use in the unrolled loops). Same values, same bits.
struct GlibcConst {
  double kLn2Hi, kLn2Lo, kA0, kA1, kA2, kA3, kA4, kB0, kB1, kB2, kB3, kB4, kB5, kB6, kB7, kB8, kB9, kB10, kBig, kSn3, kSn5, kCs2, kCs4, kCs6, kS1, kS2, kS3, kS4, kS5, kHp0, kHp1, kTaylorMax, kToint, kHpinv, kMp1, kMp2, kPp3, kPp4;
};
#if defined(__CUDACC__)
static __constant__ GlibcConst kGlibcConstDev = {glibc::kLn2Hi, glibc::kLn2Lo, glibc::kA0, glibc::kA1, glibc::kA2, glibc::kA3, glibc::kA4, glibc::kB0, glibc::kB1, glibc::kB2, glibc::kB3, glibc::kB4, glibc::kB5, glibc::kB6, glibc::kB7, glibc::kB8, glibc::kB9, glibc::kB10, glibc::kBig, glibc::kSn3, glibc::kSn5, glibc::kCs2, glibc::kCs4, glibc::kCs6, glibc::kS1, glibc::kS2, glibc::kS3, glibc::kS4, glibc::kS5, glibc::kHp0, glibc::kHp1, glibc::kTaylorMax, glibc::kToint, glibc::kHpinv, glibc::kMp1, glibc::kMp2, glibc::kPp3, glibc::kPp4};
#endif
#if defined(__CUDA_ARCH__)
#define QT_GK(n) (::qt::kGlibcConstDev.n)
#else
#define QT_GK(n) (::qt::glibc::n)
#endif
struct GlibcLogEnt {
  double invc, logc;
};
static const GlibcLogEnt kGlibcLogTabHost[128] = {QT_GLIBC_LOG_TAB};
static const double kGlibcSincosTabHost[440] = {QT_GLIBC_SINCOS_TAB};

#if defined(__CUDA_ARCH__)
QT_HD uint64_t qt_bits(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }
QT_HD double qt_from_bits(uint64_t b) { return __longlong_as_double(static_cast<long long>(b)); }
QT_HD void glibc_log_tab(int i, double* invc, double* logc) {
  const double2 e = __ldg(&kGlibcLogTabDev[i]);
  *invc = e.x;
  *logc = e.y;
}
QT_HD void glibc_sincos_tab(int i, double* sn, double* ssn, double* cs, double* ccs) {
  const double2 e0 = __ldg(&kGlibcSincosTabDev[2 * i]);
  const double2 e1 = __ldg(&kGlibcSincosTabDev[2 * i + 1]);
  *sn = e0.x;
  *ssn = e0.y;
  *cs = e1.x;
  *ccs = e1.y;
}
QT_HD double qt_copysign(double x, double s) { return copysign(x, s); }
QT_HD double qt_fabs(double x) { return fabs(x); }
#else
QT_HD uint64_t qt_bits(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  return b;
}
QT_HD double qt_from_bits(uint64_t b) {
  double x;
  memcpy(&x, &b, 8);
  return x;
}
QT_HD void glibc_log_tab(int i, double* invc, double* logc) {
  *invc = kGlibcLogTabHost[i].invc;
  *logc = kGlibcLogTabHost[i].logc;
}
QT_HD void glibc_sincos_tab(int i, double* sn, double* ssn, double* cs, double* ccs) {
  *sn = kGlibcSincosTabHost[4 * i];
  *ssn = kGlibcSincosTabHost[4 * i + 1];
  *cs = kGlibcSincosTabHost[4 * i + 2];
  *ccs = kGlibcSincosTabHost[4 * i + 3];
}
QT_HD double qt_copysign(double x, double s) { return std::copysign(x, s); }
QT_HD double qt_fabs(double x) { return std::fabs(x); }
#endif

// ---------------------------------------------------------------------------
// log (e_log.c, __FP_FAST_FMA build). Inputs here are positive normals; the
// subnormal / zero / negative / inf / NaN path of glibc is not restated.
// ---------------------------------------------------------------------------
constexpr uint64_t kLogLo = 0x3FEE000000000000ull;      // asuint64(1.0 - 0x1p-4)
constexpr uint64_t kLogHiMinusLo = 0x0003090000000000ull;  // asuint64(1.0 + 0x1.09p-4) - LO
constexpr uint64_t kLogOff = 0x3fe6000000000000ull;

QT_HD bool qt_log_near1(double x) { return qt_bits(x) - kLogLo < kLogHiMinusLo; }

// x in [1 - 2^-4, 1 + 0x1.09p-4): log1p(r), r = x - 1, by the degree-11
// polynomial plus the exact-ish head r - r^2/2 (e_log.c "close to 1.0").
QT_HD double qt_log_near1_eval(double x) {
  if (qt_bits(x) == 0x3ff0000000000000ull) return 0.0;
  const double r = QT_SUB(x, 1.0);
  const double r2 = QT_MUL(r, r);
  const double r3 = QT_MUL(r, r2);
  double t7 = QT_FMA(r, QT_GK(kB8), QT_GK(kB7));
  t7 = QT_FMA(r2, QT_GK(kB9), t7);
  t7 = QT_FMA(r3, QT_GK(kB10), t7);
  double t4 = QT_FMA(r, QT_GK(kB5), QT_GK(kB4));
  t4 = QT_FMA(r2, QT_GK(kB6), t4);
  t4 = QT_FMA(t7, r3, t4);
  double t1 = QT_FMA(r, QT_GK(kB2), QT_GK(kB1));
  t1 = QT_FMA(r2, QT_GK(kB3), t1);
  const double p = QT_FMA(t4, r3, t1);
  const double rhi = QT_FMA(-r, 0x1p27, QT_FMA(r, 0x1p27, r));  // (r + w) - w, w = r 2^27
  const double rlo = QT_SUB(r, rhi);
  const double rh2 = QT_MUL(rhi, rhi);
  const double hi = QT_FMA(rh2, QT_GK(kB0), r);
  double lo = QT_FMA(rh2, QT_GK(kB0), QT_SUB(r, hi));
  lo = QT_FMA(QT_MUL(QT_GK(kB0), rlo), QT_ADD(r, rhi), lo);
  return QT_ADD(hi, QT_FMA(p, r3, lo));
}

// Table path, split so a caller can issue the table loads of several logs
// before the arithmetic of the first: x = 2^k z, z in [OFF, 2 OFF),
// r = z invc_i - 1 by one FMA, log x = k ln2 + logc_i + log1p(r).
struct LogPrep {
  double z, invc, logc, kd;
};
QT_HD LogPrep qt_log_prep(double x) {
  const uint64_t ix = qt_bits(x);
  const uint64_t tmp = ix - kLogOff;
  const int i = static_cast<int>((tmp >> 45) & 127u);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  LogPrep q;
  q.z = qt_from_bits(ix - (tmp & (0xfffull << 52)));
  q.kd = static_cast<double>(k);
  glibc_log_tab(i, &q.invc, &q.logc);
  return q;
}
QT_HD double qt_log_finish(const LogPrep& q) {
  const double r = QT_FMA(q.z, q.invc, -1.0);
  const double w = QT_FMA(q.kd, QT_GK(kLn2Hi), q.logc);
  const double hi = QT_ADD(w, r);
  const double lo = QT_FMA(q.kd, QT_GK(kLn2Lo), QT_ADD(QT_SUB(w, hi), r));
  const double r2 = QT_MUL(r, r);
  const double p = QT_FMA(r2, QT_FMA(r, QT_GK(kA4), QT_GK(kA3)), QT_FMA(r, QT_GK(kA2), QT_GK(kA1)));
  const double y = QT_FMA(QT_MUL(r, r2), p, QT_FMA(r2, QT_GK(kA0), lo));
  return QT_ADD(y, hi);
}
QT_HD double qt_log_unit(double x) {
  return qt_log_near1(x) ? qt_log_near1_eval(x) : qt_log_finish(qt_log_prep(x));
}

// ---------------------------------------------------------------------------
// sincos (s_sincos.c with s_sin.c's do_sin / do_cos / reduce_sincos):
//   |x| < 2^-27          sin = x, cos = 1
//   |x| < 0.85546875     sin = do_sin(x, 0),              cos = do_cos(x, 0)
//   |x| < 2.426265       a + da = pi/2 - |x|:  sin = copysign(do_cos(a, da), x),
//                                              cos = do_sin(a, da)
//   |x| < 105414350      a + da = x - n pi/2:  sin = do_sincos(a, da, n),
//                                              cos = do_sincos(a, da, n + 1)
// Every range evaluates one do_sin and one do_cos of the same (a, da), so the
// restatement computes the range's (a, da, n) branch-free, then both kernels
// (sharing their table row), then routes and signs the two results.
// ---------------------------------------------------------------------------
struct SincosArg {
  double a, da;
  int route;  // 0: (sin, cos) = (S, C); 1: (C, S); bit 2: negate sin; bit 3: negate cos
  bool tiny;
};
QT_HD SincosArg qt_sincos_arg(double x) {
  const uint32_t k = static_cast<uint32_t>(qt_bits(x) >> 32) & 0x7fffffffu;
  SincosArg g;
  g.tiny = k < 0x3e400000u;
  if (k < 0x3feb6000u) {
    g.a = x;
    g.da = 0.0;
    g.route = 0;
  } else if (k < 0x400368fdu) {
    const double y = QT_SUB(QT_GK(kHp0), qt_fabs(x));
    g.a = QT_ADD(y, QT_GK(kHp1));
    g.da = QT_ADD(QT_SUB(y, g.a), QT_GK(kHp1));
    g.route = 1 | 16;  // bit 4: sin takes the sign of x
  } else {
    const double t = QT_FMA(x, QT_GK(kHpinv), QT_GK(kToint));
    const double xn = QT_SUB(t, QT_GK(kToint));
    const int n = static_cast<int>(qt_bits(t) & 3u);
    const double y = QT_FMA(-xn, QT_GK(kMp2), QT_FMA(-xn, QT_GK(kMp1), x));
    const double t2 = QT_FMA(-xn, QT_GK(kPp3), y);
    const double db = QT_FMA(-xn, QT_GK(kPp3), QT_SUB(y, t2));
    const double b = QT_FMA(-xn, QT_GK(kPp4), t2);
    g.a = b;
    g.da = QT_ADD(db, QT_FMA(-xn, QT_GK(kPp4), QT_SUB(t2, b)));
    g.route = (n & 1) | ((n & 2) ? 4 : 0) | (((n + 1) & 2) ? 8 : 0);
  }
  return g;
}

QT_HD void qt_sincos_eval(double x, const SincosArg& g, double* s_out, double* c_out) {
  const double a = g.a, da = g.da;
  const double ab = qt_fabs(a);
  const double u = QT_ADD(ab, QT_GK(kBig));
  const int row = static_cast<int>(static_cast<uint32_t>(qt_bits(u)));
  double sn, ssn, cs, ccs;
  glibc_sincos_tab(row, &sn, &ssn, &cs, &ccs);
  const double xr = QT_SUB(ab, QT_SUB(u, QT_GK(kBig)));
  // do_sin(a, da)
  double S;
  if (ab < QT_GK(kTaylorMax)) {
    const double xx = QT_MUL(a, a);
    const double p = QT_FMA(QT_FMA(QT_FMA(QT_FMA(QT_GK(kS5), xx, QT_GK(kS4)), xx, QT_GK(kS3)), xx, QT_GK(kS2)), xx, QT_GK(kS1));
    S = QT_ADD(a, QT_FMA(xx, QT_FMA(p, a, -QT_MUL(0.5, da)), da));
  } else {
    const double d = a <= 0.0 ? -da : da;
    const double xx = QT_MUL(xr, xr);
    const double s = QT_ADD(QT_FMA(QT_MUL(xr, xx), QT_FMA(xx, QT_GK(kSn5), QT_GK(kSn3)), d), xr);
    const double c = QT_FMA(d, xr, QT_MUL(xx, QT_FMA(QT_FMA(xx, QT_GK(kCs6), QT_GK(kCs4)), xx, QT_GK(kCs2))));
    const double cor = QT_FMA(s, cs, QT_FMA(-c, sn, QT_FMA(s, ccs, ssn)));
    S = qt_copysign(QT_ADD(cor, sn), a);
  }
  // do_cos(a, da)
  double C;
  {
    const double d = a < 0.0 ? -da : da;
    const double xc = QT_ADD(xr, d);
    const double xx = QT_MUL(xc, xc);
    const double s = QT_FMA(QT_MUL(xc, xx), QT_FMA(xx, QT_GK(kSn5), QT_GK(kSn3)), xc);
    const double c = QT_MUL(xx, QT_FMA(QT_FMA(xx, QT_GK(kCs6), QT_GK(kCs4)), xx, QT_GK(kCs2)));
    const double cor = QT_FMA(-s, sn, QT_FMA(-c, cs, QT_FMA(-s, ssn, ccs)));
    C = QT_ADD(cs, cor);
  }
  double sv = (g.route & 1) ? C : S;
  double cv = (g.route & 1) ? S : C;
  if (g.route & 4) sv = -sv;
  if (g.route & 8) cv = -cv;
  if (g.route & 16) sv = qt_copysign(sv, x);
  *s_out = g.tiny ? x : sv;
  *c_out = g.tiny ? 1.0 : cv;
}

QT_HD void qt_sincos_2pi(double x, double* s_out, double* c_out) {
  qt_sincos_eval(x, qt_sincos_arg(x), s_out, c_out);
}

}  // namespace qt
