/* Exhaustive proof that the device's constant division in mrg_to_unit
 * (paper_1101_3228_b200/csrc/qt_device.cuh) equals the IEEE quotient the
 * reference computes, static_cast<double>(x + 1) / static_cast<double>(m1 + 1)
 * (rng/mrg32k3a.hpp:62), for every possible numerator a = x + 1 in [1, m1].
 * Device: q = RN(a R); r = RN(a - q d) via fma; RN(q + r R) via fma, with
 * R = RN(1 / d). fma() here is the IEEE fused multiply-add (-mfma), the same
 * operation as the device's DFMA. Prints the mismatch count (expected 0). */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define M1 4294967087ull
static const double D = 4294967088.0;
static double R;
static int NT = 8;
static uint64_t bad[64];

static void* run(void* arg) {
  const uint64_t t = (uint64_t)(uintptr_t)arg;
  const uint64_t lo = 1 + M1 * t / NT, hi = 1 + M1 * (t + 1) / NT;
  uint64_t b = 0;
  for (uint64_t x = lo; x < hi; ++x) {
    const double a = (double)x;
    volatile double ref = a / D;
    const double q = a * R;
    const double r = fma(-q, D, a);
    const double z = fma(r, R, q);
    b += z != ref;
  }
  bad[t] = b;
  return NULL;
}

int main(int argc, char** argv) {
  if (argc > 1) NT = atoi(argv[1]);
  volatile double one = 1.0;
  R = one / D;
  pthread_t th[64];
  for (int t = 0; t < NT; ++t) pthread_create(&th[t], NULL, run, (void*)(uintptr_t)t);
  uint64_t total = 0;
  for (int t = 0; t < NT; ++t) {
    pthread_join(th[t], NULL);
    total += bad[t];
  }
  printf("%llu\n", (unsigned long long)total);
  return total != 0;
}
