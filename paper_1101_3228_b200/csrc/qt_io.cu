// qt_io.cu -- tree and grid files: the QTRE v1 binary tree
// format of quant_tree.hpp:138-207 and the grid text format of grid.hpp:84-117,
// byte-identical to the reference's save_tree / save_grid, and loaders with the
// reference's error taxonomy and messages (IoError -> status 3, NumericError
// from the grid invariants -> status 4).
//
// The B200 part is the device-resident writer: a tree estimated on the GPU is
// written straight from HBM (counts and pi are 2.4-2.9 GB each at C4/C5) through
// two pinned staging buffers, the DMA of chunk c+1 overlapping the file write of
// chunk c, without materialising a host copy of the tree.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qtree_cuda.h"
#include "qt_internal.h"

namespace {

struct IoFailure {
  qt_status code;
  std::string msg;
};

[[noreturn]] void fail(qt_status c, const std::string& m) { throw IoFailure{c, m}; }

template <class F>
qt_status io_guarded(F&& f) {
  try {
    f();
    return QT_OK;
  } catch (const IoFailure& e) {
    qt::note_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    qt::note_error("host allocation failed");
    return QT_ERR_IO;
  }
}

constexpr char kMagic[4] = {'Q', 'T', 'R', 'E'};
constexpr uint32_t kVersion = 1;

// grid.hpp:78-82 format_double + quant_tree.hpp:112-124 grid_text
std::string grid_text(int dim, uint64_t n, const double* pts) {
  std::string s = std::to_string(n) + ' ' + std::to_string(dim) + '\n';
  char buf[40];
  for (uint64_t i = 0; i < n; ++i) {
    for (int j = 0; j < dim; ++j) {
      if (j) s += ' ';
      std::snprintf(buf, sizeof buf, "%.17g", pts[i * dim + j]);
      s += buf;
    }
    s += '\n';
  }
  return s;
}

// QuantGrid invariants (grid.hpp:24-31): finite, pairwise distinct -> NumericError
void check_points(int dim, uint64_t n, const double* p, const char* where) {
  for (uint64_t i = 0; i < n * static_cast<uint64_t>(dim); ++i)
    if (!std::isfinite(p[i])) fail(QT_ERR_NUMERIC, std::string(where) + ": non-finite point coordinate");
  std::vector<uint64_t> ord(n);
  for (uint64_t i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](uint64_t a, uint64_t b) {
    return std::lexicographical_compare(p + a * dim, p + (a + 1) * dim, p + b * dim, p + (b + 1) * dim);
  });
  for (uint64_t i = 1; i < n; ++i)
    if (std::equal(p + ord[i - 1] * dim, p + (ord[i - 1] + 1) * dim, p + ord[i] * dim))
      fail(QT_ERR_NUMERIC, std::string(where) + ": duplicate points");
}

// "N d" + N*d doubles, istream >> semantics (whitespace separated)
struct TextGrid {
  int dim = 0;
  std::vector<double> pts;
};
bool parse_grid(const char* s, const char* end, TextGrid& g, bool allow_trailing) {
  char* e = nullptr;
  auto skip = [&](const char* c) {
    while (c < end && (*c == ' ' || *c == '\n' || *c == '\t' || *c == '\r')) ++c;
    return c;
  };
  const char* c = skip(s);
  errno = 0;
  const unsigned long long n = std::strtoull(c, &e, 10);
  if (e == c || errno) return false;
  c = skip(e);
  const long d = std::strtol(c, &e, 10);
  if (e == c || n == 0 || d < 1) return false;
  g.dim = static_cast<int>(d);
  g.pts.resize(n * static_cast<uint64_t>(d));
  for (auto& v : g.pts) {
    c = skip(e);
    if (c >= end) return false;
    v = std::strtod(c, &e);
    if (e == c) return false;
  }
  if (!allow_trailing && skip(e) < end) return false;
  return true;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

void put(FILE* f, const void* p, size_t n, const std::string& path) {
  if (n && std::fwrite(p, 1, n, f) != n) fail(QT_ERR_IO, "save_tree: write failed for " + path);
}

void get(FILE* f, void* p, size_t n) {
  if (n && std::fread(p, 1, n, f) != n) fail(QT_ERR_IO, "tree file: truncated");
}

// Device -> file through two pinned buffers (DMA of chunk c+1 overlaps the
// write of chunk c).
void put_device(FILE* f, const void* src, size_t bytes, const std::string& path) {
  constexpr size_t kChunk = 64u << 20;
  static std::mutex mu;
  static uint8_t* pin[2] = {nullptr, nullptr};
  std::lock_guard<std::mutex> lk(mu);
  auto cuda = [&](cudaError_t e) {
    if (e != cudaSuccess) fail(QT_ERR_DEVICE, std::string("cuda: ") + cudaGetErrorString(e));
  };
  if (!pin[0]) {
    cuda(cudaHostAlloc(reinterpret_cast<void**>(&pin[0]), kChunk, cudaHostAllocDefault));
    cuda(cudaHostAlloc(reinterpret_cast<void**>(&pin[1]), kChunk, cudaHostAllocDefault));
  }
  cudaStream_t st;
  cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t ev[2];
  cuda(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  cuda(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t c) {
    const size_t off = c * kChunk, n = std::min(kChunk, bytes - off);
    cuda(cudaMemcpyAsync(pin[c & 1], static_cast<const uint8_t*>(src) + off, n,
                         cudaMemcpyDeviceToHost, st));
    cuda(cudaEventRecord(ev[c & 1], st));
  };
  try {
    if (nch) issue(0);
    for (size_t c = 0; c < nch; ++c) {
      if (c + 1 < nch) issue(c + 1);
      cuda(cudaEventSynchronize(ev[c & 1]));
      put(f, pin[c & 1], std::min(kChunk, bytes - c * kChunk), path);
    }
  } catch (...) {
    cudaStreamSynchronize(st);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    cudaStreamDestroy(st);
    throw;
  }
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  cudaStreamDestroy(st);
}

}  // namespace

extern "C" {

// save_tree (quant_tree.hpp:138-163)
QT_API qt_status qt_save_tree(const char* path, int32_t layers, int32_t dim, const uint64_t* sizes,
                              const double* points_all, uint64_t samples, const uint64_t* visits,
                              const uint64_t* joint, const double* pi, int32_t device_arrays) {
  return io_guarded([&] {
    if (!path || !sizes || !points_all || !visits || !joint || !pi || layers < 1 || dim < 1)
      fail(QT_ERR_INVALID_ARGUMENT, "save_tree: null or empty argument");
    const std::string p(path);
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) fail(QT_ERR_IO, "save_tree: cannot open " + p);
    put(out.f, kMagic, 4, p);
    put(out.f, &kVersion, 4, p);
    const uint32_t n = static_cast<uint32_t>(layers);
    put(out.f, &n, 4, p);
    put(out.f, &samples, 8, p);
    const double* g = points_all;
    uint64_t nvis = 0;
    for (int k = 0; k <= layers; ++k) {
      const std::string t = grid_text(dim, sizes[k], g);
      const uint64_t len = t.size();
      put(out.f, &len, 8, p);
      put(out.f, t.data(), t.size(), p);
      g += sizes[k] * static_cast<uint64_t>(dim);
      nvis += sizes[k];
    }
    auto arr = [&](const void* a, size_t bytes) {
      if (device_arrays) put_device(out.f, a, bytes, p);
      else put(out.f, a, bytes, p);
    };
    arr(visits, nvis * 8);
    uint64_t off = 0;
    for (int k = 1; k <= layers; ++k) {
      const uint64_t r = sizes[k - 1], c = sizes[k];
      put(out.f, &r, 8, p);
      put(out.f, &c, 8, p);
      arr(joint + off, r * c * 8);
      arr(pi + off, r * c * 8);
      off += r * c;
    }
    if (std::fflush(out.f) != 0) fail(QT_ERR_IO, "save_tree: write failed for " + p);
  });
}

// The header of a tree file and its total sizes: layers n, dim, M and sizes[0..n]
// (nullable; written only when sizes_cap >= n + 1), so a caller can allocate the
// arrays qt_load_tree fills. Every embedded grid must have the first grid's dim
// (the flat layout holds one dim; the reference's make_tree_shell requires it,
// estimate.hpp:55-58).
QT_API qt_status qt_tree_file_info(const char* path, int32_t* layers, int32_t* dim,
                                   uint64_t* samples, uint64_t* sizes, uint64_t sizes_cap) {
  return io_guarded([&] {
    if (!path) fail(QT_ERR_INVALID_ARGUMENT, "load_tree: null path");
    const std::string p(path);
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) fail(QT_ERR_IO, "load_tree: cannot open " + p);
    char magic[4];
    if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
      fail(QT_ERR_IO, "load_tree: bad magic in " + p);
    uint32_t version = 0, n = 0;
    get(in.f, &version, 4);
    if (version != kVersion) fail(QT_ERR_IO, "load_tree: unsupported version " + std::to_string(version));
    get(in.f, &n, 4);
    if (n == 0) fail(QT_ERR_IO, "load_tree: empty tree");
    uint64_t m = 0;
    get(in.f, &m, 8);
    int d = 0;
    for (uint32_t k = 0; k <= n; ++k) {
      uint64_t len = 0;
      get(in.f, &len, 8);
      std::string text(len, '\0');
      get(in.f, text.data(), len);
      TextGrid tg;
      if (!parse_grid(text.data(), text.data() + text.size(), tg, true))
        fail(QT_ERR_IO, "tree file: malformed embedded grid");
      if (k == 0) d = tg.dim;
      else if (tg.dim != d) fail(QT_ERR_IO, "load_tree: grids of differing dimension in " + p);
      if (sizes && sizes_cap >= static_cast<uint64_t>(n) + 1)
        sizes[k] = tg.pts.size() / static_cast<uint64_t>(tg.dim);
    }
    if (layers) *layers = static_cast<int32_t>(n);
    if (dim) *dim = d;
    if (samples) *samples = m;
  });
}

// load_tree (quant_tree.hpp:165-205) into caller-allocated host arrays laid out
// like qt_estimate's (points_all includes layer 0). The caller states what it
// allocated (from qt_tree_file_info): sizes holds layers + 1 entries,
// points_all visits_cap * dim doubles, visits visits_cap, joint and pi
// joint_cap each. A file that needs more (or changed since the info call)
// fails with QT_ERR_IO before anything past a capacity is written.
QT_API qt_status qt_load_tree(const char* path, int32_t layers, int32_t dim, uint64_t* sizes,
                              double* points_all, uint64_t* visits, uint64_t visits_cap,
                              uint64_t* joint, double* pi, uint64_t joint_cap) {
  return io_guarded([&] {
    if (!path || !sizes || !points_all || !visits || !joint || !pi || layers < 1 || dim < 1)
      fail(QT_ERR_INVALID_ARGUMENT, "load_tree: null argument");
    const std::string p(path);
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) fail(QT_ERR_IO, "load_tree: cannot open " + p);
    char magic[4];
    if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
      fail(QT_ERR_IO, "load_tree: bad magic in " + p);
    uint32_t version = 0, n = 0;
    get(in.f, &version, 4);
    if (version != kVersion) fail(QT_ERR_IO, "load_tree: unsupported version " + std::to_string(version));
    get(in.f, &n, 4);
    if (n == 0) fail(QT_ERR_IO, "load_tree: empty tree");
    if (n != static_cast<uint32_t>(layers))
      fail(QT_ERR_IO, "load_tree: " + p + " has " + std::to_string(n) + " layers, caller allocated " +
                          std::to_string(layers));
    uint64_t m = 0;
    get(in.f, &m, 8);
    double* g = points_all;
    uint64_t nvis = 0;
    for (uint32_t k = 0; k <= n; ++k) {
      uint64_t len = 0;
      get(in.f, &len, 8);
      std::string text(len, '\0');
      get(in.f, text.data(), len);
      TextGrid tg;
      if (!parse_grid(text.data(), text.data() + text.size(), tg, true))
        fail(QT_ERR_IO, "tree file: malformed embedded grid");
      if (tg.dim != dim) fail(QT_ERR_IO, "load_tree: grids of differing dimension in " + p);
      const uint64_t N = tg.pts.size() / static_cast<uint64_t>(tg.dim);
      check_points(tg.dim, N, tg.pts.data(), "grid");
      if (N > visits_cap - nvis) fail(QT_ERR_IO, "load_tree: " + p + " exceeds the caller's capacity");
      sizes[k] = N;
      std::memcpy(g, tg.pts.data(), tg.pts.size() * 8);
      g += tg.pts.size();
      nvis += N;
    }
    get(in.f, visits, nvis * 8);
    uint64_t off = 0;
    for (uint32_t k = 1; k <= n; ++k) {
      uint64_t r = 0, c = 0;
      get(in.f, &r, 8);
      get(in.f, &c, 8);
      if (r != sizes[k - 1] || c != sizes[k])
        fail(QT_ERR_IO, "load_tree: transition dimensions disagree with grids");
      if (r * c > joint_cap - off) fail(QT_ERR_IO, "load_tree: " + p + " exceeds the caller's capacity");
      get(in.f, joint + off, r * c * 8);
      get(in.f, pi + off, r * c * 8);
      off += r * c;
    }
  });
}

// save_grid (grid.hpp:86-99)
QT_API qt_status qt_save_grid(const char* path, int32_t dim, uint64_t n, const double* pts) {
  return io_guarded([&] {
    if (!path || !pts || dim < 1 || n == 0) fail(QT_ERR_INVALID_ARGUMENT, "save_grid: empty grid");
    const std::string p(path);
    File out;
    out.f = std::fopen(path, "w");
    if (!out.f) fail(QT_ERR_IO, "save_grid: cannot open " + p);
    const std::string t = grid_text(dim, n, pts);
    if (std::fwrite(t.data(), 1, t.size(), out.f) != t.size() || std::fflush(out.f) != 0)
      fail(QT_ERR_IO, "save_grid: write failed for " + p);
  });
}

// load_grid (grid.hpp:101-117): *n and *dim always; pts (nullable) receives the
// points when its capacity `cap` (doubles) suffices.
QT_API qt_status qt_load_grid(const char* path, int32_t* dim, uint64_t* n, double* pts, uint64_t cap) {
  return io_guarded([&] {
    if (!path || !dim || !n) fail(QT_ERR_INVALID_ARGUMENT, "load_grid: null argument");
    const std::string p(path);
    File in;
    in.f = std::fopen(path, "r");
    if (!in.f) fail(QT_ERR_IO, "load_grid: cannot open " + p);
    std::string text;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, in.f)) > 0) text.append(buf, got);
    // header first (its own message), then the body
    {
      char* e = nullptr;
      const char* c = text.c_str();
      const unsigned long long hn = std::strtoull(c, &e, 10);
      const char* c2 = e;
      const long hd = std::strtol(c2, &e, 10);
      if (e == c2 || c2 == c || hn == 0 || hd < 1)
        fail(QT_ERR_IO, "load_grid: malformed header in " + p);
    }
    TextGrid tg;
    if (!parse_grid(text.data(), text.data() + text.size(), tg, true)) {
      char* e = nullptr;
      const unsigned long long hn = std::strtoull(text.c_str(), &e, 10);
      const long hd = std::strtol(e, nullptr, 10);
      fail(QT_ERR_IO, "load_grid: expected " + std::to_string(hn) + " rows of " +
                          std::to_string(hd) + " values in " + p);
    }
    if (!parse_grid(text.data(), text.data() + text.size(), tg, false))
      fail(QT_ERR_IO, "load_grid: trailing data in " + p);
    const uint64_t N = tg.pts.size() / static_cast<uint64_t>(tg.dim);
    try {
      check_points(tg.dim, N, tg.pts.data(), "grid");
    } catch (const IoFailure& e) {
      fail(QT_ERR_IO, "load_grid: " + e.msg + " in " + p);
    }
    *dim = tg.dim;
    *n = N;
    if (pts && cap >= tg.pts.size()) std::memcpy(pts, tg.pts.data(), tg.pts.size() * 8);
  });
}

}  // extern "C"
