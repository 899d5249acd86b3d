// A minimal Catch2-v3-compatible test shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <catch2/catch_amalgamated.hpp>, which this container does not have
// (SURVEY.md §4). This header implements the subset they use -- TEST_CASE,
// SECTION (Catch's re-entry semantics: one leaf section per run), REQUIRE,
// CHECK, CHECK_THROWS_AS, FAIL and Catch::Approx (margin / epsilon) -- so
// those files compile UNMODIFIED against the drop-in headers in include/ and
// run on the device path. Written from Catch2's documented behaviour; no
// Catch2 source is involved.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct RequireFailed {};

struct TestCase {
  std::string name, tags;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* tags, void (*fn)()) {
    registry().push_back({name, tags, fn});
  }
};

// Section bookkeeping of one test case across its runs.
struct Tracker {
  std::set<std::string> done;           // fully explored section paths
  std::vector<std::string> stack;       // entered sections of the current run
  std::vector<bool> entered_at_level;   // a section was entered at this depth this run
  std::vector<bool> pending_at_level;   // an unexplored sibling was skipped at this depth
  int failures = 0;
  int assertions = 0;
  std::string test_name;
  std::set<std::string> skip;  // "test case/section path" entries to skip

  std::string path(const std::string& leaf) const {
    std::string p;
    for (const auto& s : stack) p += s + "/";
    return p + leaf;
  }
  void start_run() {
    stack.clear();
    entered_at_level.assign(1, false);
    pending_at_level.assign(1, false);
  }
};

inline Tracker*& tracker() {
  static Tracker* t = nullptr;
  return t;
}

class Section {
 public:
  explicit Section(const char* name) {
    Tracker& t = *tracker();
    const std::size_t level = t.stack.size();
    if (t.entered_at_level.size() <= level + 1) {
      t.entered_at_level.resize(level + 2, false);
      t.pending_at_level.resize(level + 2, false);
    }
    full_ = t.path(name);
    if (t.done.count(full_)) return;
    if (t.skip.count(t.test_name + "/" + full_)) {
      std::printf("skip %s / %s\n", t.test_name.c_str(), full_.c_str());
      t.done.insert(full_);
      return;
    }
    if (t.entered_at_level[level]) {
      t.pending_at_level[level] = true;  // explore it in a later run
      return;
    }
    t.entered_at_level[level] = true;
    t.stack.push_back(name);
    t.entered_at_level[level + 1] = false;
    t.pending_at_level[level + 1] = false;
    entered_ = true;
  }
  ~Section() {
    if (!entered_) return;
    Tracker& t = *tracker();
    const std::size_t child = t.stack.size();
    const bool children_pending = child < t.pending_at_level.size() && t.pending_at_level[child];
    // a REQUIRE failure unwinds through here: the section counts as explored
    if (!children_pending || std::uncaught_exceptions() > 0) t.done.insert(full_);
    t.stack.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  std::string full_;
  bool entered_ = false;
};

inline void report(const char* kind, const char* expr, const char* file, int line) {
  std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, kind, expr);
}

inline void check(bool ok, bool fatal, const char* kind, const char* expr, const char* file,
                  int line) {
  Tracker& t = *tracker();
  ++t.assertions;
  if (ok) return;
  ++t.failures;
  report(kind, expr, file, line);
  if (fatal) throw RequireFailed{};
}

// CATCH_SHIM_SKIP: ';'-separated "test case name/section path" entries.
inline std::set<std::string> skip_list() {
  std::set<std::string> out;
  const char* env = std::getenv("CATCH_SHIM_SKIP");
  std::string s = env ? env : "";
  std::size_t b = 0;
  while (b < s.size()) {
    std::size_t e = s.find(';', b);
    if (e == std::string::npos) e = s.size();
    if (e > b) out.insert(s.substr(b, e - b));
    b = e + 1;
  }
  return out;
}

inline int run_all(const char* filter) {
  int failed_cases = 0, total_assertions = 0, total_failures = 0;
  const std::set<std::string> skip = skip_list();
  for (const TestCase& tc : registry()) {
    if (filter && tc.name.find(filter) == std::string::npos) continue;
    Tracker t;
    t.test_name = tc.name;
    t.skip = skip;
    tracker() = &t;
    for (int run = 0; run < 10000; ++run) {
      t.start_run();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++t.failures;
        std::fprintf(stderr, "%s: unexpected exception: %s\n", tc.name.c_str(), e.what());
      } catch (...) {
        ++t.failures;
        std::fprintf(stderr, "%s: unexpected non-std exception\n", tc.name.c_str());
      }
      if (!t.pending_at_level[0]) break;
    }
    tracker() = nullptr;
    total_assertions += t.assertions;
    total_failures += t.failures;
    std::printf("%-4s %s  (%d assertions)\n", t.failures ? "FAIL" : "ok", tc.name.c_str(),
                t.assertions);
    if (t.failures) ++failed_cases;
  }
  std::printf("%d test cases failed, %d assertions, %d failures\n", failed_cases, total_assertions,
              total_failures);
  return failed_cases ? 1 : 0;
}

}  // namespace catch_shim

namespace Catch {

/// Catch::Approx: |a - b| <= margin, or <= epsilon * (scale + |value|).
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double other) const {
    if (std::fabs(other - value_) <= margin_) return true;
    const double tol = epsilon_ * (scale_ + (std::isinf(value_) ? 0.0 : std::fabs(value_)));
    return other == value_ || std::fabs(other - value_) <= tol;
  }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& b, double a) { return b.matches(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.matches(a); }

 private:
  double value_;
  double margin_ = 0.0;
  double epsilon_ = std::numeric_limits<float>::epsilon() * 100.0;
  double scale_ = 0.0;
};

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST(fn, ...)                                                          \
  static void fn();                                                                       \
  static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(CATCH_SHIM_NAME(__VA_ARGS__, ""), \
                                                        CATCH_SHIM_TAGS(__VA_ARGS__, ""), fn); \
  static void fn()
#define CATCH_SHIM_NAME(name, ...) name
#define CATCH_SHIM_TAGS(name, tags, ...) tags

#define TEST_CASE(...) CATCH_SHIM_TEST(CATCH_SHIM_CAT(catch_shim_test_, __LINE__), __VA_ARGS__)
#define SECTION(name) if (catch_shim::Section CATCH_SHIM_CAT(catch_shim_sec_, __LINE__){name})

#define REQUIRE(...) \
  catch_shim::check(static_cast<bool>(__VA_ARGS__), true, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK(...) \
  catch_shim::check(static_cast<bool>(__VA_ARGS__), false, "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE_FALSE(...) \
  catch_shim::check(!static_cast<bool>(__VA_ARGS__), true, "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  catch_shim::check(!static_cast<bool>(__VA_ARGS__), false, "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define CATCH_SHIM_THROWS_AS(fatal, kind, expr, type)                         \
  do {                                                                        \
    bool caught_ = false;                                                     \
    try {                                                                     \
      static_cast<void>(expr);                                                \
    } catch (const type&) {                                                   \
      caught_ = true;                                                         \
    } catch (...) {                                                           \
    }                                                                         \
    catch_shim::check(caught_, fatal, kind, #expr " throws " #type, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(false, "CHECK_THROWS_AS", expr, type)
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(true, "REQUIRE_THROWS_AS", expr, type)
#define FAIL(msg) catch_shim::check(false, true, "FAIL", msg, __FILE__, __LINE__)
