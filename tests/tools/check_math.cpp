// check_math.cpp -- csrc/qt_math.h (the device's Box-Muller log and sincos,
// built here for the host with the same explicitly rounded operations) against
// the live glibc libm the reference's box_muller calls (stream.hpp:57-62:
// std::log, and the cos/sin pair g++ fuses into one sincos call).
//
// Domains, each the exact set of doubles an engine feeds Box-Muller:
//   mrg     u = (x + 1) / (m1 + 1), x = 0 .. m1 - 1       (mrg32k3a.hpp:62)  EXHAUSTIVE
//   xorwow  u = v * 2^-32,          v = 0 .. 2^32 - 1     (xorwow.hpp:46)    EXHAUSTIVE
//   lcg48   u = x * 2^-48,          x sampled + edges     (lcg48.hpp:30)
// For every u: log(u1) with u1 = u (u <= 0 clamps to 2^-64 like box_muller),
// and sincos(2 pi u). Prints one JSON line with the number of inputs and of
// bit mismatches; exit 1 on any mismatch.
//
//   g++ -O2 -std=c++17 -fno-builtin -ffp-contract=off -pthread check_math.cpp -lm
//   ./a.out [mrg|xorwow|lcg48|all] [lcg48_samples] [threads] [stride]
//   (stride > 1 checks every stride-th input of the two exhaustive domains)
//   ./a.out checksum [threads]   -> glibc's checksums for qt_math_checksum (domains 0, 1)
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../paper_1101_3228_b200/csrc/qt_math.h"

extern "C" void sincos(double, double*, double*);

static uint64_t bits(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
}

struct Tally {
  std::atomic<uint64_t> n{0}, bad_log{0}, bad_sin{0}, bad_cos{0};
  std::atomic<uint64_t> first_bad{~0ull};
};

static void check_one(double u, Tally& t, uint64_t tag, uint64_t& bl, uint64_t& bs, uint64_t& bc) {
  const double u1 = u <= 0.0 ? 0x1p-64 : u;
  volatile double vu1 = u1;
  const double gl = std::log(vu1);
  const double ml = qt::qt_log_unit(u1);
  const double a = 2.0 * 3.141592653589793 * u;
  double gs, gc, ms, mc;
  volatile double va = a;
  sincos(va, &gs, &gc);
  qt::qt_sincos_2pi(a, &ms, &mc);
  const bool b1 = bits(gl) != bits(ml), b2 = bits(gs) != bits(ms), b3 = bits(gc) != bits(mc);
  bl += b1;
  bs += b2;
  bc += b3;
  if (b1 || b2 || b3) {
    uint64_t cur = t.first_bad.load();
    while (tag < cur && !t.first_bad.compare_exchange_weak(cur, tag)) {
    }
  }
}

static uint64_t g_stride = 1;

template <class F>
static void run_range(uint64_t count, int threads, Tally& t, F&& uniform, bool strided = true) {
  const uint64_t st = strided ? g_stride : 1;
  std::vector<std::thread> th;
  for (int w = 0; w < threads; ++w) {
    th.emplace_back([&, w] {
      uint64_t bl = 0, bs = 0, bc = 0;
      const uint64_t lo = count * w / threads, hi = count * (w + 1) / threads;
      uint64_t cnt = 0;
      for (uint64_t i = (lo + st - 1) / st * st; i < hi; i += st, ++cnt)
        check_one(uniform(i), t, i, bl, bs, bc);
      t.n += cnt;
      t.bad_log += bl;
      t.bad_sin += bs;
      t.bad_cos += bc;
    });
  }
  for (auto& x : th) x.join();
}

// the order-independent checksum of k_math_checksum (csrc/qt_kernels.cu)
static uint64_t mix_checksum(uint64_t i, double v) {
  uint64_t z = bits(v) + 0x9E3779B97F4A7C15ull * (i + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int checksums(int threads) {
  std::printf("{");
  for (int domain = 0; domain < 2; ++domain) {
    const uint64_t n = domain == 0 ? 4294967087ull : (1ull << 32);
    std::atomic<uint64_t> sl{0}, ss{0}, sc{0};
    std::vector<std::thread> th;
    for (int w = 0; w < threads; ++w) {
      th.emplace_back([&, w] {
        uint64_t a = 0, b = 0, c = 0;
        for (uint64_t i = n * w / threads; i < n * (w + 1) / threads; ++i) {
          const double u = domain == 0 ? static_cast<double>(i + 1) / 4294967088.0
                                       : static_cast<double>(i) * 0x1p-32;
          volatile double u1 = u <= 0.0 ? 0x1p-64 : u;
          a += mix_checksum(i, std::log(u1));
          double s, co;
          volatile double ang = 2.0 * 3.141592653589793 * u;
          sincos(ang, &s, &co);
          b += mix_checksum(i, s);
          c += mix_checksum(i, co);
        }
        sl += a;
        ss += b;
        sc += c;
      });
    }
    for (auto& x : th) x.join();
    std::printf("%s\"%s\": [\"%llu\", \"%llu\", \"%llu\"]", domain ? ", " : "",
                domain == 0 ? "mrg32k3a" : "xorwow", (unsigned long long)sl.load(),
                (unsigned long long)ss.load(), (unsigned long long)sc.load());
    std::fflush(stdout);
  }
  std::printf("}\n");
  return 0;
}

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "all";
  if (which == "checksum")
    return checksums(argc > 2 ? std::atoi(argv[2]) : int(std::thread::hardware_concurrency()));
  const uint64_t lcg_samples = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 200000000ull;
  const int threads = argc > 3 ? std::atoi(argv[3]) : int(std::thread::hardware_concurrency());
  g_stride = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 1;
  std::printf("{");
  bool first = true, ok = true;
  auto report = [&](const char* name, Tally& t) {
    std::printf("%s\"%s\": {\"inputs\": %llu, \"log_mismatch\": %llu, \"sin_mismatch\": %llu, "
                "\"cos_mismatch\": %llu, \"first_bad_index\": %lld}",
                first ? "" : ", ", name, (unsigned long long)t.n.load(),
                (unsigned long long)t.bad_log.load(), (unsigned long long)t.bad_sin.load(),
                (unsigned long long)t.bad_cos.load(),
                t.first_bad.load() == ~0ull ? -1LL : (long long)t.first_bad.load());
    first = false;
    ok = ok && t.bad_log == 0 && t.bad_sin == 0 && t.bad_cos == 0;
    std::fflush(stdout);
  };
  if (which == "mrg" || which == "all") {
    Tally t;
    const uint64_t m1 = 4294967087ull;
    run_range(m1, threads, t, [](uint64_t x) {
      return static_cast<double>(x + 1) / static_cast<double>(4294967087ull + 1);
    });
    report("mrg32k3a", t);
  }
  if (which == "xorwow" || which == "all") {
    Tally t;
    run_range(1ull << 32, threads, t, [](uint64_t v) { return static_cast<double>(v) * 0x1p-32; });
    report("xorwow", t);
  }
  if (which == "lcg48" || which == "all") {
    Tally t;
    // edges: the 2^20 smallest and largest 48-bit states, then splitmix-spread samples
    run_range(lcg_samples + (1ull << 21), threads, t, [](uint64_t i) {
      uint64_t x;
      if (i < (1ull << 20)) {
        x = i;
      } else if (i < (1ull << 21)) {
        x = (1ull << 48) - 1 - (i - (1ull << 20));
      } else {
        uint64_t z = i * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        x = (z ^ (z >> 31)) >> 16;
      }
      return static_cast<double>(x) * 0x1p-48;
    }, false);
    report("lcg48", t);
  }
  std::printf("}\n");
  return ok ? 0 : 1;
}
