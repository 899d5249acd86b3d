// check_math.cpp -- the device Box-Muller kernels (csrc/qt_math.h, built here
// with the same explicitly rounded operations) against glibc, which the
// reference's Box-Muller calls (stream.hpp:57-62). Inputs are the exact
// Box-Muller angles 2 pi u for MRG32k3a-shaped uniforms u = (x + 1) / (m1 + 1).
// Prints one JSON line: samples, bit-identical fraction and max ulp distance.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../paper_1101_3228_b200/csrc/qt_math.h"

static int64_t bits(double x) {
  int64_t b;
  std::memcpy(&b, &x, 8);
  return b;
}
static uint64_t ulp_dist(double a, double b) {
  int64_t x = bits(a), y = bits(b);
  if (x < 0) x = INT64_MIN - x;
  if (y < 0) y = INT64_MIN - y;
  return static_cast<uint64_t>(x > y ? x - y : y - x);
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 20000000ull;
  uint64_t z = 0x9E3779B97F4A7C15ull, same_s = 0, same_c = 0, max_s = 0, max_c = 0;
  uint64_t same_l = 0, max_l = 0;
  const double m1p1 = 4294967088.0;
  for (uint64_t i = 0; i < n; ++i) {
    z = z * 6364136223846793005ull + 1442695040888963407ull;
    const uint64_t x = (z >> 32) % 4294967087ull;
    const double u = static_cast<double>(x + 1) / m1p1;
    const double a = 2.0 * 3.14159265358979323846 * u;
    double s, c;
    qt::qt_sincos_2pi(a, &s, &c);
    const double rs = std::sin(a), rc = std::cos(a);
    const uint64_t ds = ulp_dist(s, rs), dc = ulp_dist(c, rc);
    const uint64_t dl = ulp_dist(qt::qt_log_unit(u), std::log(u));
    same_l += dl == 0;
    if (dl > max_l) max_l = dl;
    same_s += ds == 0;
    same_c += dc == 0;
    if (ds > max_s) max_s = ds;
    if (dc > max_c) max_c = dc;
  }
  std::printf("{\"samples\": %llu, \"sin_identical\": %.6f, \"cos_identical\": %.6f, "
              "\"sin_max_ulp\": %llu, \"cos_max_ulp\": %llu, \"log_identical\": %.6f, "
              "\"log_max_ulp\": %llu}\n",
              (unsigned long long)n, double(same_s) / n, double(same_c) / n,
              (unsigned long long)max_s, (unsigned long long)max_c, double(same_l) / n,
              (unsigned long long)max_l);
  return (max_s > 1 || max_c > 1 || max_l > 1) ? 1 : 0;
}
