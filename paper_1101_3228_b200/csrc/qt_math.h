// qt_math.h -- the Box-Muller transcendental kernels, specialised to their
// input domains and written with explicitly rounded operations only, so the
// host build (tests/tools/check_math.cpp, checked against glibc) and the
// device build produce the same bits.
//
//   qt_sincos_2pi(a): sin and cos of the Box-Muller angle a = 2 pi u2 in
//   [0, 2 pi]. Cody-Waite reduction by q pi/2 with pi/2 = HI + MID + LO
//   (HI has 3 trailing zero bits, so q HI is exact for q <= 4 and a - q HI is
//   exact by Sterbenz), then the fdlibm-form kernels on |r| <= pi/4 with the
//   reduction tail folded in (< 1 ulp). No table loads, no large-argument path.
#pragma once

#if defined(__CUDA_ARCH__)
#define QT_HD __host__ __device__ __forceinline__
#define QT_FMA(a, b, c) __fma_rn((a), (b), (c))
#define QT_MUL(a, b) __dmul_rn((a), (b))
#define QT_ADD(a, b) __dadd_rn((a), (b))
#define QT_SUB(a, b) __dsub_rn((a), (b))
#define QT_RINT(a) rint(a)
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
#define QT_RINT(a) std::nearbyint(a)
#endif

#include <stdint.h>
#include <string.h>

#include "qt_logtab.h"

namespace qt {

// The FP64 constants of both kernels. On the device they live in the constant
// bank, so every DFMA takes them as a c[][] operand instead of rebuilding each
// 64-bit literal with two uniform moves per use (ncu: UMOV was 12 % of the
// path kernel's instructions); the host build reads the same values.
#define QT_MATH_K_LIST                                                                  \
  /* 0 */ 0x1.2492492492492p-3, -0x1.5555555555555p-3, 0x1.999999999999ap-3,          \
  /* 3 */ 0x1.5555555555555p-2, kLn2Hi, kLn2Lo,                                        \
  /* 6 */ -1.66666666666666324348e-01, 8.33333333332248946124e-03,                     \
  /* 8 */ -1.98412698298579493134e-04, 2.75573137070700676789e-06,                     \
  /* 10 */ -2.50507602534068634195e-08, 1.58969099521155010221e-10,                    \
  /* 12 */ 4.16666666666666019037e-02, -1.38888888888741095749e-03,                    \
  /* 14 */ 2.48015872894767294178e-05, -2.75573143513906633035e-07,                    \
  /* 16 */ 2.08757232129817482790e-09, -1.13596475577881948265e-11,                    \
  /* 18 */ 0x1.45f306dc9c883p-1, 0x1.921fb54442d18p+0, 0x1.1a62633145c07p-54,          \
  /* 21 */ -0x1.f1976b7ed8fbcp-110, -0.125, -0.25, -0.5, 0.5, 1.0
#if defined(__CUDACC__)
static __device__ const LogEntry kLogTabDev[128] = {QT_LOGTAB_ENTRIES};
static __constant__ double kMathKDev[] = {QT_MATH_K_LIST};
#endif
static const double kMathKHost[] = {QT_MATH_K_LIST};
#if defined(__CUDA_ARCH__)
#define QTK(i) (kMathKDev[i])
#else
#define QTK(i) (kMathKHost[i])
#endif
#if defined(__CUDA_ARCH__)
QT_HD int64_t qt_bits(double x) { return __double_as_longlong(x); }
QT_HD double qt_from_bits(int64_t b) { return __longlong_as_double(b); }
QT_HD void qt_logtab(int i, double* invc, double* lhi, double* llo) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(&kLogTabDev[i]));
  *invc = a.x;
  *lhi = a.y;
  *llo = __ldg(&kLogTabDev[i].llo);
}
#else
static const LogEntry kLogTabHost[128] = {QT_LOGTAB_ENTRIES};
QT_HD int64_t qt_bits(double x) {
  int64_t b;
  memcpy(&b, &x, 8);
  return b;
}
QT_HD double qt_from_bits(int64_t b) {
  double x;
  memcpy(&x, &b, 8);
  return x;
}
QT_HD void qt_logtab(int i, double* invc, double* lhi, double* llo) {
  *invc = kLogTabHost[i].invc;
  *lhi = kLogTabHost[i].lhi;
  *llo = kLogTabHost[i].llo;
}
#endif

// log(u) for a positive normal u <= 1 (the Box-Muller radius argument:
// MRG32k3a gives u in [2^-32, 1), LCG48/XORWOW clamp 0 to 2^-64). u = 2^e m,
// m in [1, 2); cell i = round(128 (m - 1)) (the top cell folds to m/2 next to
// 1, so around u = 1 the reduced argument r = m - 1 is exact); r = m invc_i - 1
// by one FMA, |r| <= 2^-8; log u = e ln2 + (-log invc_i) + log1p(r) with the
// constants as hi + lo pairs and a degree-8 Taylor tail (< 1 ulp).
// Split form: qt_log_prep does the reduction and the table loads, qt_log_finish
// the arithmetic, so a caller can issue the loads of several logs (and other
// independent work) before the first use. qt_log_unit = finish(prep(u)).
struct LogPrep {
  double m, invc, lhi, llo;
  int e;
};
QT_HD LogPrep qt_log_prep(double u) {
  const int64_t b = qt_bits(u);
  LogPrep q;
  q.e = static_cast<int>(b >> 52) - 1023;
  const int64_t mant = b & ((int64_t(1) << 52) - 1);
  int i = static_cast<int>((mant + (int64_t(1) << 44)) >> 45);
  q.m = qt_from_bits(mant | (int64_t(1023) << 52));
  if (i == 128) {  // m in [2 - 2^-8, 2): use m/2 in [1 - 2^-9, 1), cell 0
    i = 0;
    q.e += 1;
    q.m = QT_MUL(q.m, 0.5);
  }
  qt_logtab(i, &q.invc, &q.lhi, &q.llo);
  return q;
}
QT_HD double qt_log_finish(const LogPrep& q) {
  const double m = q.m, invc = q.invc, lhi = q.lhi, llo = q.llo;
  const double r = QT_FMA(m, invc, -1.0);
  const double kd = static_cast<double>(q.e);
  const double t1 = QT_MUL(kd, QTK(4));               // exact (41-bit ln2 hi)
  const double hi = QT_ADD(t1, lhi);
  const double lo_a = QT_ADD(QT_SUB(t1, hi), lhi);    // Fast2Sum (|t1| >= |lhi| or t1 = 0)
  const double hi2 = QT_ADD(hi, r);
  const double lo_b = QT_ADD(QT_SUB(hi, hi2), r);     // Fast2Sum (|hi| >= |r| or hi = 0)
  // log1p(r) - r = r^2 (-1/2 + r (1/3 + r (-1/4 + r (1/5 + r (-1/6 + r (1/7 - r/8))))))
  const double p7 = QT_FMA(r, QTK(22), QTK(0));
  const double p6 = QT_FMA(r, p7, QTK(1));
  const double p5 = QT_FMA(r, p6, QTK(2));
  const double p4 = QT_FMA(r, p5, -0.25);
  const double p3 = QT_FMA(r, p4, QTK(3));
  const double p2 = QT_FMA(r, p3, -0.5);
  const double tail = QT_MUL(QT_MUL(r, r), p2);
  const double lo = QT_ADD(QT_ADD(QT_FMA(kd, QTK(5), llo), QT_ADD(lo_a, lo_b)), tail);
  return QT_ADD(hi2, lo);
}
QT_HD double qt_log_unit(double u) { return qt_log_finish(qt_log_prep(u)); }

QT_HD void qt_sincos_2pi(double a, double* s_out, double* c_out) {
  // fdlibm __kernel_sin / __kernel_cos coefficients (|x| <= pi/4)
  const double S1 = QTK(6), S2 = QTK(7), S3 = QTK(8), S4 = QTK(9), S5 = QTK(10), S6 = QTK(11);
  const double C1 = QTK(12), C2 = QTK(13), C3 = QTK(14), C4 = QTK(15), C5 = QTK(16),
               C6 = QTK(17);
  const double q = QT_RINT(QT_MUL(a, QTK(18)));  // round(a * 2/pi)
  const double t = QT_FMA(-q, QTK(19), a);       // exact
  const double r = QT_FMA(-q, QTK(20), t);
  // tail: (t - r) - q MID - q LO
  const double y = QT_FMA(-q, QTK(21), QT_FMA(-q, QTK(20), QT_SUB(t, r)));
  const double z = QT_MUL(r, r);
  const double v = QT_MUL(z, r);
  // sin(r + y) = r - ((z (y/2 - v P) - y) - v S1)
  const double ps = QT_FMA(z, QT_FMA(z, QT_FMA(z, QT_FMA(z, S6, S5), S4), S3), S2);
  const double sn =
      QT_SUB(r, QT_SUB(QT_SUB(QT_MUL(z, QT_FMA(-v, ps, QT_MUL(0.5, y))), y), QT_MUL(v, S1)));
  // cos(r + y) = w + (((1 - w) - z/2) + (z Q - r y)), w = 1 - z/2
  const double pc =
      QT_MUL(z, QT_FMA(z, QT_FMA(z, QT_FMA(z, QT_FMA(z, QT_FMA(z, C6, C5), C4), C3), C2), C1));
  const double hz = QT_MUL(0.5, z);
  const double w = QT_SUB(1.0, hz);
  const double cs =
      QT_ADD(w, QT_ADD(QT_SUB(QT_SUB(1.0, w), hz), QT_FMA(z, pc, -QT_MUL(r, y))));
  const int quad = static_cast<int>(q) & 3;
  const double s1 = (quad & 1) ? cs : sn;
  const double c1 = (quad & 1) ? sn : cs;
  *s_out = (quad & 2) ? -s1 : s1;
  *c_out = ((quad + 1) & 2) ? -c1 : c1;
}

}  // namespace qt
