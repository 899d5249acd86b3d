// qt_bdp.cu -- K5: backward dynamic programming on the estimated tree
// (pricer/bdp.hpp:36-96, pricer/swing.hpp:47-129).
//
// pi^k is compressed on the device to CSR (ascending column order per row).
// Every conditional expectation E(f(X_{k+1}) | X_k = x_i) is then one thread's
// sequential, separately rounded sum over the row's non-zeros: skipped zero
// terms add exactly +-0 to an accumulator that can never be -0, so the result
// is bit-identical to the reference's dense j-ascending loop (bdp.hpp:49-50).
// Stopping: one thread per node. Swing: one thread per (node, consumption
// slice m') for the continuation table, then one per (node, m) for the
// bang-bang decision with the reference's window rules and tie preference.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/qtree_cuda.h"
#include "qt_internal.h"

namespace {

struct BdpFail {
  qt_status code;
  std::string msg;
};
[[noreturn]] void bdp_raise(qt_status c, const std::string& m) { throw BdpFail{c, m}; }

#define BDP_CUDA(expr)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      bdp_raise(QT_ERR_DEVICE, std::string("cuda: ") + cudaGetErrorString(e_) + " (" #expr ")"); \
  } while (0)

// nnz per row: one warp per row
__global__ void k_row_nnz(const double* pi, uint64_t rows, uint64_t cols, uint64_t* nnz) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t r = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += warps) {
    uint64_t c = 0;
    for (uint64_t j = lane; j < cols; j += 32) c += pi[r * cols + j] != 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) nnz[r] = c;
  }
}

// ascending-column fill of one row per warp
__global__ void k_row_fill(const double* pi, uint64_t rows, uint64_t cols, const uint64_t* rowptr,
                           uint32_t* colidx, double* val) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t r = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += warps) {
    uint64_t base = rowptr[r];
    for (uint64_t j0 = 0; j0 < cols; j0 += 32) {
      const uint64_t j = j0 + lane;
      const double v = j < cols ? pi[r * cols + j] : 0.0;
      const uint32_t mask = __ballot_sync(0xffffffffu, v != 0.0);
      if (v != 0.0) {
        const uint64_t at = base + __popc(mask & ((1u << lane) - 1u));
        colidx[at] = static_cast<uint32_t>(j);
        val[at] = v;
      }
      base += __popc(mask);
    }
  }
}

__device__ __forceinline__ double row_dot(const uint64_t* rowptr, const uint32_t* colidx,
                                          const double* val, uint64_t r, const double* f) {
  double acc = 0.0;
  for (uint64_t e = rowptr[r]; e < rowptr[r + 1]; ++e)
    acc = __dadd_rn(acc, __dmul_rn(val[e], f[colidx[e]]));
  return acc;
}

// The reference's dense row sum sum_j pi[i][j] f[j], j ascending (bdp.hpp:49-50),
// for an f with non-finite entries: there 0 * inf = NaN terms matter, so the
// CSR shortcut (skipping pi == 0) would differ. One thread per row.
__global__ void k_row_dense(uint64_t rows, uint64_t cols, const double* pi, const uint64_t* visits,
                            const double* f, double* out) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  if (visits[i] == 0) {
    out[i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double acc = 0.0;
  for (uint64_t j = 0; j < cols; ++j) acc = __dadd_rn(acc, __dmul_rn(pi[i * cols + j], f[j]));
  out[i] = acc;
}

// V_k = max(phi_k, E V_{k+1}); unvisited rows absorb (bdp.hpp:79-93)
__global__ void k_stop_layer(uint64_t rows, const uint64_t* rowptr, const uint32_t* colidx,
                             const double* val, const uint64_t* visits, const double* phi,
                             const double* vnext, double* v, uint8_t* ex) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const double f = phi[i];
  if (visits[i] == 0) {
    v[i] = f;
    ex[i] = 1;
    return;
  }
  const double c = row_dot(rowptr, colidx, val, i, vnext);
  v[i] = f < c ? c : f;  // std::max(phi, cont)
  ex[i] = f >= c ? 1 : 0;
}

// continuation of every stored m' slice of layer k+1 (swing.hpp:182-189)
__global__ void k_swing_cont(uint64_t rows, uint64_t cols_next, int cnt_next,
                             const uint64_t* rowptr, const uint32_t* colidx, const double* val,
                             const uint64_t* visits, const double* pnext, double* cont) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * static_cast<uint64_t>(cnt_next)) return;
  const uint64_t i = t % rows, mi = t / rows;
  cont[mi * rows + i] = visits[i] == 0 ? __longlong_as_double(0x7ff8000000000000ll)
                                       : row_dot(rowptr, colidx, val, i, pnext + mi * cols_next);
}

// bang-bang decision per (m, i), swing.hpp:197-223
__global__ void k_swing_decide(uint64_t rows, int lo, int cnt, int lo_next, int n, int k, int qmin,
                               int qmax, const double* phi, const double* cont, double* p,
                               uint8_t* take) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * static_cast<uint64_t>(cnt)) return;
  const uint64_t i = t % rows;
  const int m = lo + static_cast<int>(t / rows);
  const bool can_wait = m + (n - k - 1) >= qmin;
  const bool can_take = m + 1 <= qmax;
  const double v = phi[i];
  double best = -__longlong_as_double(0x7ff0000000000000ll);
  uint8_t bx = 0;
  if (can_wait) {
    const double c = cont[static_cast<uint64_t>(m - lo_next) * rows + i];
    best = isnan(c) ? 0.0 : c;
  }
  if (can_take) {
    const double c = cont[static_cast<uint64_t>(m + 1 - lo_next) * rows + i];
    const double cand = __dadd_rn(v, isnan(c) ? 0.0 : c);
    if (cand >= best) {
      best = cand;
      bx = 1;
    }
  }
  p[t] = best;
  take[t] = bx;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  void alloc(size_t n) {
    cudaFree(p);
    p = nullptr;
    if (n) BDP_CUDA(cudaMalloc(&p, n * sizeof(T)));
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Device CSR of all transitions.
struct Csr {
  std::vector<uint64_t> rp_off;  // per transition: offset into rowptr (rows+1 entries each)
  std::vector<uint64_t> nz_off;  // per transition: offset into colidx/val
  DevBuf<uint64_t> rowptr;
  DevBuf<uint32_t> colidx;
  DevBuf<double> val;
};

void build_csr(int n, const std::vector<uint64_t>& sizes, const double* d_pi,
               const std::vector<uint64_t>& poff, Csr& c) {
  uint64_t rows_total = 0;
  c.rp_off.resize(n);
  for (int t = 0; t < n; ++t) {
    c.rp_off[t] = rows_total + t;  // each transition owns rows+1 rowptr slots
    rows_total += sizes[t];
  }
  DevBuf<uint64_t> nnz(rows_total + n);
  c.rowptr.alloc(rows_total + n);
  BDP_CUDA(cudaMemset(nnz.p, 0, (rows_total + n) * sizeof(uint64_t)));
  for (int t = 0; t < n; ++t) {
    const uint64_t rows = sizes[t], cols = sizes[t + 1];
    const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((rows * 32 + 255) / 256, 8192));
    k_row_nnz<<<blocks, 256>>>(d_pi + poff[t], rows, cols, nnz.p + c.rp_off[t]);
    qt::note_launches(1);
  }
  // One exclusive scan over all transitions' (rows + 1)-blocks: the zero slot
  // closing each block makes rowptr[t][rows] that block's end; the values are
  // global offsets into colidx/val.
  size_t tmp_bytes = 0;
  BDP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, nnz.p, c.rowptr.p, rows_total + n));
  DevBuf<uint8_t> tmp(tmp_bytes);
  BDP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, nnz.p, c.rowptr.p, rows_total + n));
  qt::note_launches(1);
  uint64_t total_nnz = 0;
  BDP_CUDA(cudaMemcpy(&total_nnz, c.rowptr.p + rows_total + n - 1, 8, cudaMemcpyDeviceToHost));
  c.colidx.alloc(total_nnz ? total_nnz : 1);
  c.val.alloc(total_nnz ? total_nnz : 1);
  for (int t = 0; t < n; ++t) {
    const uint64_t rows = sizes[t], cols = sizes[t + 1];
    const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((rows * 32 + 255) / 256, 8192));
    k_row_fill<<<blocks, 256>>>(d_pi + poff[t], rows, cols, c.rowptr.p + c.rp_off[t], c.colidx.p,
                                c.val.p);
    qt::note_launches(1);
  }
  BDP_CUDA(cudaGetLastError());
}

template <class F>
qt_status bdp_guarded(F&& f) {
  qt::DeviceRestore keep_device;
  try {
    f();
    return QT_OK;
  } catch (const BdpFail& e) {
    qt::note_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    qt::note_error(e.what());
    return QT_ERR_DEVICE;
  }
}

// The tree on the device: visits and pi either uploaded from host arrays
// (owned) or borrowed from the caller's device buffers (the estimate -> price
// path of qt_dtree_*: no pi round trip), plus the CSR of pi and phi.
struct TreeOnDevice {
  int n;
  std::vector<uint64_t> sizes, voff, poff;
  DevBuf<uint64_t> visits_own;
  DevBuf<double> pi_own, phi;
  const uint64_t* visits = nullptr;
  const double* pi = nullptr;
  Csr csr;
  TreeOnDevice(int layers, const uint64_t* sz, const uint64_t* vis, const double* pi_in,
               const double* h_phi, bool device_arrays)
      : n(layers), sizes(sz, sz + layers + 1), voff(layers + 2, 0), poff(layers + 1, 0) {
    for (int k = 0; k <= n; ++k) voff[k + 1] = voff[k] + sizes[k];
    for (int t = 0; t < n; ++t) poff[t + 1] = poff[t] + sizes[t] * sizes[t + 1];
    if (device_arrays) {
      visits = vis;
      pi = pi_in;
    } else {
      visits_own.alloc(voff[n + 1]);
      pi_own.alloc(poff[n]);
      BDP_CUDA(cudaMemcpy(visits_own.p, vis, voff[n + 1] * 8, cudaMemcpyHostToDevice));
      BDP_CUDA(qt::staged_copy(pi_own.p, pi_in, poff[n] * 8, true, 0));  // GBs for d >= 2 trees
      visits = visits_own.p;
      pi = pi_own.p;
    }
    phi.alloc(voff[n + 1]);
    BDP_CUDA(cudaMemcpy(phi.p, h_phi, voff[n + 1] * 8, cudaMemcpyHostToDevice));
    build_csr(n, sizes, pi, poff, csr);
  }
  const uint64_t* rowptr(int t) const { return csr.rowptr.p + csr.rp_off[t]; }
};

void check_device() {
  int avail = 0;
  if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
    bdp_raise(QT_ERR_DEVICE, "cuda: no CUDA device available (the pricer has no CPU path)");
  // runs on the caller's current device
}

void check_tree_args(int layers, const uint64_t* sizes, const uint64_t* visits, const double* pi,
                     const double* phi) {
  if (layers < 1 || !sizes || !visits || !pi || !phi)
    bdp_raise(QT_ERR_INVALID_ARGUMENT, "pricer: incomplete problem");
  for (int k = 0; k <= layers; ++k)
    if (sizes[k] == 0) bdp_raise(QT_ERR_INVALID_ARGUMENT, "pricer: empty layer");
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

void stopping_impl(int32_t layers, const uint64_t* sizes, const uint64_t* visits, const double* pi,
                   const double* phi, double* value, uint8_t* exercise, double* price,
                   bool device_arrays) {
  {
    check_tree_args(layers, sizes, visits, pi, phi);
    if (!price) bdp_raise(QT_ERR_INVALID_ARGUMENT, "solve_stopping: null output");
    uint64_t nodes = 0;
    for (int k = 0; k <= layers; ++k) nodes += sizes[k];
    for (uint64_t i = 0; i < nodes; ++i)
      if (!std::isfinite(phi[i])) bdp_raise(QT_ERR_NUMERIC, "solve_stopping: non-finite payoff");
    check_device();
    TreeOnDevice t(layers, sizes, visits, pi, phi, device_arrays);
    const int n = layers;
    DevBuf<double> v(t.voff[n + 1]);
    DevBuf<uint8_t> ex(t.voff[n + 1]);
    // terminal layer: V_n = phi_n, exercise where phi > 0 (bdp.hpp:71-77)
    BDP_CUDA(cudaMemcpy(v.p + t.voff[n], phi + t.voff[n], sizes[n] * 8, cudaMemcpyHostToDevice));
    std::vector<uint8_t> ex_n(sizes[n]);
    for (uint64_t i = 0; i < sizes[n]; ++i) ex_n[i] = phi[t.voff[n] + i] > 0.0 ? 1 : 0;
    BDP_CUDA(cudaMemcpy(ex.p + t.voff[n], ex_n.data(), sizes[n], cudaMemcpyHostToDevice));
    for (int k = n - 1; k >= 0; --k) {
      const uint64_t rows = sizes[k];
      k_stop_layer<<<static_cast<uint32_t>((rows + 127) / 128), 128>>>(
          rows, t.rowptr(k), t.csr.colidx.p, t.csr.val.p, t.visits + t.voff[k],
          t.phi.p + t.voff[k], v.p + t.voff[k + 1], v.p + t.voff[k], ex.p + t.voff[k]);
      qt::note_launches(1);
    }
    BDP_CUDA(cudaGetLastError());
    BDP_CUDA(cudaMemcpy(price, v.p, 8, cudaMemcpyDeviceToHost));
    if (value) BDP_CUDA(qt::staged_copy(value, v.p, t.voff[n + 1] * 8, false, 0));
    if (exercise) BDP_CUDA(qt::staged_copy(exercise, ex.p, t.voff[n + 1], false, 0));
  }
}

void swing_impl(int32_t layers, const uint64_t* sizes, const uint64_t* visits, const double* pi,
                const double* phi, int32_t qmin, int32_t qmax, double* price, double* value_all,
                uint8_t* take_all, bool device_arrays) {
  {
    check_tree_args(layers, sizes, visits, pi, phi);
    const int n = layers;
    if (qmin < 0 || qmin > qmax) bdp_raise(QT_ERR_CONFIG, "swing: need 0 <= q_min <= q_max");
    if (qmax > n) bdp_raise(QT_ERR_CONFIG, "swing: q_max exceeds the number of exercise dates");
    if (qmin > n) bdp_raise(QT_ERR_CONFIG, "swing: q_min infeasible at the root");
    if (!price) bdp_raise(QT_ERR_INVALID_ARGUMENT, "solve_swing: null output");
    uint64_t nodes = 0;
    for (int k = 0; k < n; ++k) nodes += sizes[k];
    {
      uint64_t o = 0;
      for (int k = 0; k < n; ++k)
        for (uint64_t i = 0; i < sizes[k]; ++i, ++o)
          if (!std::isfinite(phi[o])) bdp_raise(QT_ERR_NUMERIC, "solve_swing: non-finite payoff");
    }
    check_device();
    TreeOnDevice t(n, sizes, visits, pi, phi, device_arrays);
    std::vector<int> lo(n + 1), cnt(n + 1);
    std::vector<uint64_t> soff(n + 2, 0);
    for (int k = 0; k <= n; ++k) {
      lo[k] = std::max(0, qmin - (n - k));
      cnt[k] = std::min(k, qmax) - lo[k] + 1;
      soff[k + 1] = soff[k] + static_cast<uint64_t>(cnt[k]) * sizes[k];
    }
    DevBuf<double> P(soff[n + 1]);
    DevBuf<uint8_t> take(soff[n] ? soff[n] : 1);
    BDP_CUDA(cudaMemset(P.p + soff[n], 0, (soff[n + 1] - soff[n]) * 8));  // P_n = 0
    uint64_t max_cont = 1;
    for (int k = 0; k < n; ++k)
      max_cont = std::max<uint64_t>(max_cont, static_cast<uint64_t>(cnt[k + 1]) * sizes[k]);
    DevBuf<double> cont(max_cont);
    for (int k = n - 1; k >= 0; --k) {
      const uint64_t rows = sizes[k];
      const uint64_t tc = rows * static_cast<uint64_t>(cnt[k + 1]);
      k_swing_cont<<<static_cast<uint32_t>((tc + 127) / 128), 128>>>(
          rows, sizes[k + 1], cnt[k + 1], t.rowptr(k), t.csr.colidx.p, t.csr.val.p,
          t.visits + t.voff[k], P.p + soff[k + 1], cont.p);
      const uint64_t td = rows * static_cast<uint64_t>(cnt[k]);
      k_swing_decide<<<static_cast<uint32_t>((td + 127) / 128), 128>>>(
          rows, lo[k], cnt[k], lo[k + 1], n, k, qmin, qmax, t.phi.p + t.voff[k], cont.p,
          P.p + soff[k], take.p + soff[k]);
      qt::note_launches(2);
    }
    BDP_CUDA(cudaGetLastError());
    BDP_CUDA(cudaMemcpy(price, P.p, 8, cudaMemcpyDeviceToHost));
    if (value_all) BDP_CUDA(qt::staged_copy(value_all, P.p, soff[n + 1] * 8, false, 0));
    if (take_all && soff[n]) BDP_CUDA(qt::staged_copy(take_all, take.p, soff[n], false, 0));
  }
}

}  // namespace

namespace qt {
// estimate -> price on the device (qt_capi.cu's qt_dtree_*): visits / pi are
// device arrays of the current device, phi and the outputs host arrays.
void bdp_stopping_device(int32_t layers, const uint64_t* sizes, const uint64_t* d_visits,
                         const double* d_pi, const double* phi, double* value, uint8_t* exercise,
                         double* price) {
  try {
    stopping_impl(layers, sizes, d_visits, d_pi, phi, value, exercise, price, true);
  } catch (const BdpFail& e) {
    throw BdpError{e.code, e.msg};
  }
}
void bdp_swing_device(int32_t layers, const uint64_t* sizes, const uint64_t* d_visits,
                      const double* d_pi, const double* phi, int32_t qmin, int32_t qmax,
                      double* price, double* value_all, uint8_t* take_all) {
  try {
    swing_impl(layers, sizes, d_visits, d_pi, phi, qmin, qmax, price, value_all, take_all, true);
  } catch (const BdpFail& e) {
    throw BdpError{e.code, e.msg};
  }
}
}  // namespace qt

extern "C" {

QT_API qt_status qt_bdp_stopping(int32_t layers, const uint64_t* sizes, const uint64_t* visits,
                                 const double* pi, const double* phi, double* value,
                                 uint8_t* exercise, double* price) {
  return bdp_guarded(
      [&] { stopping_impl(layers, sizes, visits, pi, phi, value, exercise, price, false); });
}

QT_API qt_status qt_bdp_swing(int32_t layers, const uint64_t* sizes, const uint64_t* visits,
                              const double* pi, const double* phi, int32_t qmin, int32_t qmax,
                              double* price, double* value_all, uint8_t* take_all) {
  return bdp_guarded([&] {
    swing_impl(layers, sizes, visits, pi, phi, qmin, qmax, price, value_all, take_all, false);
  });
}


QT_API qt_status qt_bdp_cond_expectation(uint64_t rows, uint64_t cols, const uint64_t* row_visits,
                                         const double* pi, const double* f, double* out) {
  return bdp_guarded([&] {
    if (rows == 0 || cols == 0 || !row_visits || !pi || !f || !out)
      bdp_raise(QT_ERR_INVALID_ARGUMENT, "cond_expectation: empty or null argument");
    check_device();
    const uint64_t sz[2] = {rows, cols};
    std::vector<double> no_phi(rows + cols, 0.0);
    std::vector<uint64_t> vis(rows + cols, 0);  // layer-1 visits are never read
    std::copy(row_visits, row_visits + rows, vis.begin());
    bool finite = true;
    for (uint64_t j = 0; j < cols && finite; ++j) finite = std::isfinite(f[j]);
    if (!finite) {  // the dense loop, exactly as the reference (0 * inf = NaN included)
      DevBuf<double> dpi(rows * cols), df(cols), dout(rows);
      DevBuf<uint64_t> dvis(rows);
      BDP_CUDA(qt::staged_copy(dpi.p, pi, rows * cols * 8, true, 0));
      BDP_CUDA(cudaMemcpy(df.p, f, cols * 8, cudaMemcpyHostToDevice));
      BDP_CUDA(cudaMemcpy(dvis.p, row_visits, rows * 8, cudaMemcpyHostToDevice));
      k_row_dense<<<static_cast<uint32_t>((rows + 127) / 128), 128>>>(rows, cols, dpi.p, dvis.p,
                                                                       df.p, dout.p);
      qt::note_launches(1);
      BDP_CUDA(cudaGetLastError());
      BDP_CUDA(cudaMemcpy(out, dout.p, rows * 8, cudaMemcpyDeviceToHost));
      return;
    }
    TreeOnDevice t(1, sz, vis.data(), pi, no_phi.data(), false);
    DevBuf<double> df(cols), dout(rows);
    BDP_CUDA(cudaMemcpy(df.p, f, cols * 8, cudaMemcpyHostToDevice));
    // one stored slice, unvisited rows -> quiet NaN (bdp.hpp:45-48)
    k_swing_cont<<<static_cast<uint32_t>((rows + 127) / 128), 128>>>(
        rows, cols, 1, t.rowptr(0), t.csr.colidx.p, t.csr.val.p, t.visits, df.p, dout.p);
    qt::note_launches(1);
    BDP_CUDA(cudaGetLastError());
    BDP_CUDA(cudaMemcpy(out, dout.p, rows * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
