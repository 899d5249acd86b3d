// qt_cell.cu -- K2 for d >= 2 as an exact cell-list search (TwoFactorChain
// d = 2, GbmChain3d d = 3): the default projection of k_paths_cell (Alg I/II,
// estimate.hpp:88-126) and k_alg3_cell (Alg III, estimate.hpp:213-265).
//
// The reference's nearest_brute (nn.hpp:18-46) is an argmin of the FP64 d2
// over all N_k points in index order with strict <; its kd-tree backend
// (nn.hpp:51-147) returns the same cells by visiting only the points that can
// win. This kernel does the same with a bucket grid built on the host
// (build_cell_table, qt_capi.cu): the query's bucket lists, in ascending
// index order, every point that can be the nearest one -- or tie with it --
// for some query in the bucket, and the kernel evaluates exactly the
// reference's d2 (dx*dx + dy*dy for d = 2, the coordinate-order accumulation
// from 0.0 for d = 3) over that list with strict <. The answer is therefore
// the brute-force index bit for bit (ties included); queries outside the
// bucket grid, non-finite ones, and layers without a grid take the full FP64
// scan. Per query this is ~10-40 FP64 distance evaluations instead of N_k:
// the FP32 scan of qt_scan.cu stays available (QT_NN=scan) and is the
// independent cross-check in the tests.
//
// The index lives in global memory (read through L1/L2 with __ldg) and is
// built on the device when the plan is made (k_cell_count, a scan, k_cell_fill:
// one warp per bucket over all N_k points, O(buckets x N_k) FP64 work).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cub/cub.cuh>
#include <vector>

#include "qt_device.cuh"
#include "qt_internal.h"

namespace qt {

constexpr int kCellThreads = 256;
#ifndef QT_CELL_U  // candidates gathered per batch in the list scan
#define QT_CELL_U 4
#endif
#ifndef QT_CELL_MINB  // resident CTAs per SM the register allocation must allow
#define QT_CELL_MINB 3  // the kernel is load-latency bound: warps in flight pay (C4 +24 %)
#endif

// The reference's d2 of point idx (nn.hpp:25-45), FP64, read through the
// read-only path.
template <int D>
__device__ __forceinline__ double cell_d2(const double* P, uint32_t idx, const double (&q)[D]) {
  if constexpr (D == 2) {
    const double2 p = __ldg(reinterpret_cast<const double2*>(P) + idx);
    const double dx = __dsub_rn(q[0], p.x);
    const double dy = __dsub_rn(q[1], p.y);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  } else {
    const double* pp = P + 3ull * idx;
    const double d0 = __dsub_rn(q[0], __ldg(pp));
    const double d1 = __dsub_rn(q[1], __ldg(pp + 1));
    const double d2 = __dsub_rn(q[2], __ldg(pp + 2));
    double acc = __dadd_rn(0.0, __dmul_rn(d0, d0));
    acc = __dadd_rn(acc, __dmul_rn(d1, d1));
    return __dadd_rn(acc, __dmul_rn(d2, d2));
  }
}

// The reference's nearest index of q on one layer (see the file header).
// With bucket records (crec), the candidates of most buckets come with the
// record itself: one dependent L2 load fewer per query.
template <int D>
__device__ __forceinline__ uint32_t cell_nearest(const CellHdr* hp, const uint32_t* cstart,
                                                 const uint16_t* clist, const uint4* crec,
                                                 const uint8_t* xb, const double (&q)[D],
                                                 const uint8_t* gtables) {
  const LayerTable& hx = *reinterpret_cast<const LayerTable*>(xb);
  bool in = __ldg(&hp->ok) != 0;
  uint32_t b = 0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double t = __dmul_rn(__dsub_rn(q[c], __ldg(hp->lo + c)), __ldg(hp->inv_w + c));
    const uint32_t g = __ldg(hp->g + c);
    in = in && t >= 0.0 && t < static_cast<double>(g);  // false for NaN
    const uint32_t ci = in ? static_cast<uint32_t>(t) : 0u;
    b = b * g + ci;
  }
  if (!in) return nearest<D>(hx, xb, q, gtables);  // exact full scan (nn.hpp:18-46)
  const uint64_t sb = __ldg(reinterpret_cast<const unsigned long long*>(&hp->start_off)) + b;
  const double* P = reinterpret_cast<const double*>(xb + hx.off_rec);
  uint32_t s, e;
  if (crec) {
    const uint4 rr = __ldg(crec + sb);
    const uint32_t n = rr.x & 0xFFFFu;
    if (n != 0xFFFFu) {  // inline: n <= 7 candidates, ascending
      const uint32_t c[7] = {rr.x >> 16, rr.y & 0xFFFFu, rr.y >> 16, rr.z & 0xFFFFu, rr.z >> 16,
                             rr.w & 0xFFFFu, rr.w >> 16};
      uint32_t best = c[0];
      double bd = cell_d2<D>(P, best, q);
#pragma unroll
      for (uint32_t u = 1; u < 7; ++u) {
        if (u < n) {
          const double d = cell_d2<D>(P, c[u], q);
          if (d < bd) {
            bd = d;
            best = c[u];
          }
        }
      }
      return best;
    }
    s = rr.y;
    e = rr.y + rr.z;
  } else {
    s = __ldg(cstart + sb);
    e = __ldg(cstart + sb + 1);
  }
  uint32_t best = __ldg(clist + s);
  double bd = cell_d2<D>(P, best, q);
  uint32_t u = s + 1;
  // QT_CELL_U candidates per batch: their list entries and points are loaded
  // before any is compared, so the dependent L2 gathers overlap; the compares
  // stay in list (ascending index) order, so ties resolve as in the scan
  for (; u + QT_CELL_U <= e; u += QT_CELL_U) {
    uint32_t id[QT_CELL_U];
    double d[QT_CELL_U];
#pragma unroll
    for (int t = 0; t < QT_CELL_U; ++t) id[t] = __ldg(clist + u + t);
#pragma unroll
    for (int t = 0; t < QT_CELL_U; ++t) d[t] = cell_d2<D>(P, id[t], q);
#pragma unroll
    for (int t = 0; t < QT_CELL_U; ++t) {
      if (d[t] < bd) {  // strict <: the smallest index among ties (lists are ascending)
        bd = d[t];
        best = id[t];
      }
    }
  }
  for (; u < e; ++u) {
    const uint32_t idx = __ldg(clist + u);
    const double d = cell_d2<D>(P, idx, q);
    if (d < bd) {
      bd = d;
      best = idx;
    }
  }
  return best;
}

// bucket records from start[] / list[] (see CellArgs::crec), one thread per bucket
__global__ void k_cell_records(uint64_t nb_all, const uint32_t* start, const uint16_t* list,
                               uint4* rec) {
  for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < nb_all;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = start[b], n = start[b + 1] - s;
    uint4 r;
    if (n <= 7 && n > 0) {
      uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (uint32_t u = 0; u < n; ++u) c[u + 1] = list[s + u];
      c[0] = n;
      r = make_uint4(c[0] | (c[1] << 16), c[2] | (c[3] << 16), c[4] | (c[5] << 16), c[6] | (c[7] << 16));
    } else {
      r = make_uint4(0xFFFFu, s, n, 0u);
    }
    rec[b] = r;
  }
}

// ---------------------------------------------------------------------------
// Index build, one warp per bucket. Bucket box R (inflated by 1e-6 of a bucket
// width against the query map's rounding): every point p' bounds the nearest
// distance of every query in R by dmax(R, p'), so U = min_p' dmax^2(R, p')
// bounds it, and only points with dmin^2(R, p) <= U (1 + 2e-9) can be the
// nearest point or tie with it; the relative slack covers the FP64 rounding
// of these bounds and of the reference's d2 (2^-50). Both kernels compute U
// and the test identically, so the fill writes exactly the counted points.
// ---------------------------------------------------------------------------
template <int D>
struct CellBox {
  double lo[D], hi[D];
};

template <int D>
__device__ __forceinline__ CellBox<D> cell_box(const CellHdr& h, uint64_t b) {
  uint32_t cc[D];
#pragma unroll
  for (int c = D - 1; c >= 0; --c) {
    cc[c] = static_cast<uint32_t>(b % h.g[c]);
    b /= h.g[c];
  }
  CellBox<D> r;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double eps = 1e-6 * h.w[c];
    r.lo[c] = h.lo[c] + cc[c] * h.w[c] - eps;
    r.hi[c] = h.lo[c] + (cc[c] + 1.0) * h.w[c] + eps;
  }
  return r;
}

template <int D>
__device__ __forceinline__ double box_dmin2(const CellBox<D>& r, const double* p) {
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double v = p[c];
    const double d = v < r.lo[c] ? r.lo[c] - v : (v > r.hi[c] ? v - r.hi[c] : 0.0);
    s = fma(d, d, s);
  }
  return s;
}

template <int D>
__device__ __forceinline__ double box_dmax2(const CellBox<D>& r, const double* p) {
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double d = fmax(fabs(p[c] - r.lo[c]), fabs(p[c] - r.hi[c]));
    s = fma(d, d, s);
  }
  return s;
}

template <int D>
__device__ __forceinline__ double cell_bound(const CellBox<D>& r, const double* P, uint32_t N,
                                             uint32_t lane) {
  double u = __longlong_as_double(0x7ff0000000000000ll);
  for (uint32_t i = lane; i < N; i += 32) u = fmin(u, box_dmax2<D>(r, P + static_cast<uint64_t>(i) * D));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u = fmin(u, __shfl_xor_sync(0xffffffffu, u, o));
  return u * (1.0 + 2e-9);
}

template <int D>
__global__ void __launch_bounds__(256) k_cell_count(const CellHdr h, const double* P, uint32_t N,
                                                    uint32_t* counts) {
  const uint64_t nb = static_cast<uint64_t>(h.g[0]) * h.g[1] * h.g[2];
  const uint64_t b = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (b >= nb) return;
  const CellBox<D> r = cell_box<D>(h, b);
  const double U = cell_bound<D>(r, P, N, lane);
  uint32_t c = 0;
  for (uint32_t i = lane; i < N; i += 32) c += box_dmin2<D>(r, P + static_cast<uint64_t>(i) * D) <= U;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) counts[h.start_off + b] = c;
}

template <int D>
__global__ void __launch_bounds__(256) k_cell_fill(const CellHdr h, const double* P, uint32_t N,
                                                   const uint32_t* start, uint16_t* list) {
  const uint64_t nb = static_cast<uint64_t>(h.g[0]) * h.g[1] * h.g[2];
  const uint64_t b = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (b >= nb) return;
  const CellBox<D> r = cell_box<D>(h, b);
  const double U = cell_bound<D>(r, P, N, lane);
  uint32_t pos = start[h.start_off + b];
  for (uint32_t i0 = 0; i0 < N; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool take = i < N && box_dmin2<D>(r, P + static_cast<uint64_t>(i) * D) <= U;
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    if (take) list[pos + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(i);
    pos += __popc(m);
  }
}

cudaError_t build_cell_lists(int dim, int n, const CellHdr* hdr, const uint64_t* npts,
                             const uint8_t* tables, const uint64_t* pts_off, CellHdr** d_hdr,
                             uint32_t** d_start, uint16_t** d_list, uint4** d_rec,
                             uint64_t* total) {
  uint64_t nb_all = 0;
  for (int k = 0; k < n; ++k) nb_all += static_cast<uint64_t>(hdr[k].g[0]) * hdr[k].g[1] * hdr[k].g[2];
  uint32_t* counts = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cudaMalloc(d_hdr, n * sizeof(CellHdr));
  if (e == cudaSuccess) e = cudaMemcpy(*d_hdr, hdr, n * sizeof(CellHdr), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&counts, (nb_all + 1) * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(counts, 0, (nb_all + 1) * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(d_start, (nb_all + 1) * sizeof(uint32_t));
  auto grid = [](uint64_t nb) { return static_cast<uint32_t>((nb * 32 + 255) / 256); };
  for (int k = 0; k < n && e == cudaSuccess; ++k) {
    if (!hdr[k].ok) continue;  // one bucket, count 0: the full scan answers every query
    const uint64_t nb = static_cast<uint64_t>(hdr[k].g[0]) * hdr[k].g[1] * hdr[k].g[2];
    const double* P = reinterpret_cast<const double*>(tables + pts_off[k]);
    const uint32_t N = static_cast<uint32_t>(npts[k]);
    if (dim == 2) k_cell_count<2><<<grid(nb), 256>>>(hdr[k], P, N, counts);
    else k_cell_count<3><<<grid(nb), 256>>>(hdr[k], P, N, counts);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, *d_start, nb_all + 1);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, *d_start, nb_all + 1);
  uint32_t tot = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&tot, *d_start + nb_all, 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMalloc(d_list, (tot ? tot : 1) * sizeof(uint16_t));
  for (int k = 0; k < n && e == cudaSuccess; ++k) {
    if (!hdr[k].ok) continue;
    const uint64_t nb = static_cast<uint64_t>(hdr[k].g[0]) * hdr[k].g[1] * hdr[k].g[2];
    const double* P = reinterpret_cast<const double*>(tables + pts_off[k]);
    const uint32_t N = static_cast<uint32_t>(npts[k]);
    if (dim == 2) k_cell_fill<2><<<grid(nb), 256>>>(hdr[k], P, N, *d_start, *d_list);
    else k_cell_fill<3><<<grid(nb), 256>>>(hdr[k], P, N, *d_start, *d_list);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && d_rec) {
    e = cudaMalloc(d_rec, (nb_all ? nb_all : 1) * sizeof(uint4));
    if (e == cudaSuccess) {
      k_cell_records<<<static_cast<uint32_t>(std::min<uint64_t>((nb_all + 255) / 256, 148 * 64)), 256>>>(
          nb_all, *d_start, *d_list, *d_rec);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(counts);
  cudaFree(tmp);
  *total = tot;
  return e;
}

// Alg I / II: P paths per thread, every layer's tables from global memory.
// Slot v = gid P + p owns a contiguous run of paths (one serial stream).
template <int K, int SRC, int P>
__global__ void __launch_bounds__(kCellThreads, QT_CELL_MINB) k_paths_cell(const __grid_constant__ CellArgs f) {
  using C = Chain<K>;
  constexpr int D = C::D;
  const PathArgs& a = f.p;
  const uint64_t rounds = a.q + (a.rem ? 1u : 0u);
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * kCellThreads + threadIdx.x;
  Source<SRC> src[P];
  uint64_t beg[P], cnt[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t v = gid * P + p;
    cnt[p] = a.q + (v < a.rem ? 1u : 0u);
    beg[p] = a.first + v * a.q + (v < a.rem ? v : a.rem);
    if (cnt[p]) src[p].start(a.src, beg[p]);
  }
  for (uint64_t r = 0; r < rounds; ++r) {
    double x[P][D];
    uint32_t i[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (r < cnt[p] && r > 0) src[p].next_unit(a.src, beg[p] + r);
#pragma unroll
      for (int c = 0; c < D; ++c) x[p][c] = 0.0;  // initial(): the origin
      i[p] = 0;
    }
    for (uint32_t k = 1; k <= a.n; ++k) {
      const uint8_t* xb = a.tables + __ldg(a.tab_off + k - 1);
      const CellHdr* ch = f.chdr + (k - 1);
      const LayerTable& hx = *reinterpret_cast<const LayerTable*>(xb);
      double stp[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) stp[c] = __ldg(hx.step + c);
      const uint64_t joff = __ldg(&hx.joff);
      const uint32_t npts = __ldg(&hx.n_pts);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (r < cnt[p]) {
          double e[C::NPS], xn[D];
#pragma unroll
          for (int q = 0; q < C::NPS; ++q) e[q] = src[p].normal();
          C::step(stp, x[p], xn, e);
#pragma unroll
          for (int c = 0; c < D; ++c) x[p][c] = xn[c];
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (r < cnt[p]) {
          const uint32_t j = cell_nearest<D>(ch, f.cstart, f.clist, f.crec, xb, x[p], a.tables);
          if (!a.probe_nored) red_add_u64(a.joint + joff + static_cast<uint64_t>(i[p]) * npts + j, 1ull);
          i[p] = j;
        }
      }
    }
  }
}

// Alg III: CTA = (slice of layer k's M samples, layer k), as k_alg3 / k_alg3_scan:
// X_{k-1} from its closed-form marginal, X_k = step(X_{k-1}), both projected.
template <int K, int SRC>
__global__ void __launch_bounds__(kCellThreads) k_alg3_cell(const __grid_constant__ Alg3CellArgs f) {
  using C = Chain<K>;
  constexpr int D = C::D;
  const Alg3Args& a = f.a;
  const uint32_t k = blockIdx.y + 1;  // transition k-1 -> k
  const uint64_t layer0 = static_cast<uint64_t>(k - 1) * a.M;
  uint64_t lo = layer0 + a.M * blockIdx.x / gridDim.x;
  uint64_t hi = layer0 + a.M * (blockIdx.x + 1) / gridDim.x;
  lo = lo > a.first ? lo : a.first;
  hi = hi < a.first + a.count ? hi : a.first + a.count;
  if (lo >= hi) return;
  const uint8_t* xk = a.tables + __ldg(a.tab_off + k - 1);
  const CellHdr* ck = f.chdr + (k - 1);
  const uint8_t* xp = k >= 2 ? a.tables + __ldg(a.tab_off + k - 2) : nullptr;
  const CellHdr* cp = k >= 2 ? f.chdr + (k - 2) : nullptr;
  const LayerTable& hx = *reinterpret_cast<const LayerTable*>(xk);
  double stp[6], mg[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    stp[c] = hx.step[c];
    mg[c] = hx.marg_prev[c];
  }
  unsigned long long* jl = a.joint + hx.joff;
  const uint32_t npts = hx.n_pts;
  const uint64_t len = hi - lo;
  const uint64_t q = len / kCellThreads, rem = len % kCellThreads;
  const uint64_t v = threadIdx.x;
  const uint64_t cnt = q + (v < rem ? 1u : 0u);
  const uint64_t beg = lo + v * q + (v < rem ? v : rem);
  if (cnt == 0) return;
  Source<SRC> src;
  src.start(a.src, beg);
  for (uint64_t r = 0; r < cnt; ++r) {
    if (r > 0) src.next_unit(a.src, beg + r);
    double e[D + C::NPS], x[D], xn[D];
#pragma unroll
    for (int q2 = 0; q2 < D + C::NPS; ++q2) e[q2] = src.normal();
    C::marginal(mg, k == 1, x, e);  // sample_marginal(k-1, ...)
    C::step(stp, x, xn, e + D);      // step(k-1, ...)
    const uint32_t j = cell_nearest<D>(ck, f.cstart, f.clist, f.crec, xk, xn, a.tables);
    const uint32_t i = k >= 2 ? cell_nearest<D>(cp, f.cstart, f.clist, f.crec, xp, x, a.tables) : 0u;
    if (!a.probe_nored) red_add_u64(jl + static_cast<uint64_t>(i) * npts + j, 1ull);
  }
}

template <int K, int SRC, int P>
static const void* cell_fn() {
  return reinterpret_cast<const void*>(k_paths_cell<K, SRC, P>);
}

template <int K, int SRC>
static cudaError_t launch_cell_t(int P, const CellArgs& a, uint32_t blocks, cudaStream_t st,
                                 int* bps) {
  const void* fn = P == 1 ? cell_fn<K, SRC, 1>() : cell_fn<K, SRC, 2>();
  if (bps) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, fn, kCellThreads, 0) != cudaSuccess ||
        *bps < 1)
      *bps = 1;
    return cudaSuccess;
  }
  if (P == 1) k_paths_cell<K, SRC, 1><<<blocks, kCellThreads, 0, st>>>(a);
  else k_paths_cell<K, SRC, 2><<<blocks, kCellThreads, 0, st>>>(a);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_cell_k(int src, int P, const CellArgs& a, uint32_t blocks,
                                 cudaStream_t st, int* bps) {
  switch (src) {
    case kSrcLcg48: return launch_cell_t<K, kSrcLcg48>(P, a, blocks, st, bps);
    case kSrcMrg: return launch_cell_t<K, kSrcMrg>(P, a, blocks, st, bps);
    case kSrcXorwow: return launch_cell_t<K, kSrcXorwow>(P, a, blocks, st, bps);
    default: return launch_cell_t<K, kSrcNormalsIn>(P, a, blocks, st, bps);
  }
}

// kind 1 = TwoFactorChain (d = 2), 3 = GbmChain3d (d = 3)
cudaError_t launch_paths_cell(int kind, int src, int P, const CellArgs& a, uint32_t blocks,
                              cudaStream_t st) {
  return kind == 1 ? launch_cell_k<1>(src, P, a, blocks, st, nullptr)
                   : launch_cell_k<3>(src, P, a, blocks, st, nullptr);
}

int paths_cell_blocks_per_sm(int kind, int src, int P) {
  int b = 1;
  if (kind == 1) launch_cell_k<1>(src, P, CellArgs{}, 0, nullptr, &b);
  else launch_cell_k<3>(src, P, CellArgs{}, 0, nullptr, &b);
  return b;
}

template <int K>
static cudaError_t launch_alg3_cell_k(int src, const Alg3CellArgs& a, dim3 g, cudaStream_t st) {
  switch (src) {
    case kSrcLcg48: k_alg3_cell<K, kSrcLcg48><<<g, kCellThreads, 0, st>>>(a); break;
    case kSrcMrg: k_alg3_cell<K, kSrcMrg><<<g, kCellThreads, 0, st>>>(a); break;
    case kSrcXorwow: k_alg3_cell<K, kSrcXorwow><<<g, kCellThreads, 0, st>>>(a); break;
    default: k_alg3_cell<K, kSrcNormalsIn><<<g, kCellThreads, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_alg3_cell(int kind, int src, const Alg3CellArgs& a, uint32_t slices,
                             cudaStream_t st) {
  const dim3 g(slices, a.a.n);
  return kind == 1 ? launch_alg3_cell_k<1>(src, a, g, st) : launch_alg3_cell_k<3>(src, a, g, st);
}

}  // namespace qt
