// qt_scan.cu -- K2 for d >= 2: the Voronoi projection as an FP32 brute-force
// scan with an exact FP64 decision (TwoFactorChain d = 2, GbmChain3d d = 3).
//
// k_paths_scan runs Alg I / II paths like k_paths (exact FP64 normals and
// chain step, estimate.hpp:88-126), but projects with
//   pass 1  s_i = h_i - q . p_i for every grid point, two points per FFMA2
//           (the query coordinate is the broadcast scalar operand), the
//           per-chunk minimum by FMNMX3, and the three best chunk minima
//           m1 <= m2 <= m3 per query (with the chunks of m1, m2);
//   bound   |s_i - S_i| <= B(q) for the exact S_i = |p_i|^2/2 - q.p_i, and the
//           reference's FP64 d2 (nn.hpp:25-45) orders like 2 S_i + |q|^2 up to
//           a relative 2^-50, so every reference minimiser satisfies
//           s_i <= tau = m1 + 2 B + 2^-48 (|m1| + B + |q|^2);
//   pass 2  if the third-best chunk minimum m3 > tau, only the best (and,
//           when m2 <= tau, the second-best) chunk of 32 points can hold a
//           minimiser: each lane rescans its query's chunk(s) with the pass-1 FFMA2 and
//           counts the points with s <= tau; one candidate is the answer,
//           several are resolved with the reference's FP64 d2 in index order
//           (strict <, smallest index on ties). Otherwise (or for a
//           non-finite / huge query) the exact FP64 scan of nearest_2d /
//           nearest_3d runs.
// The cell is therefore always the reference's argmin; the FP32 scan only
// decides which points need the FP64 arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qt_device.cuh"
#include "qt_internal.h"

namespace qt {

// threads per CTA: d = 3 tables are 64 KB, so one CTA per SM; it gets 16 warps
template <int K>
__host__ __device__ constexpr int scan_threads() { return Chain<K>::D == 3 ? 512 : 256; }
constexpr int kScanMaxStages = 4;

// {s, s} * b + c on the FP32x2 pipe (SASS FFMA2 with a broadcast scalar)
__device__ __forceinline__ float2 ffma2(float s, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 a, b, c, d;\n\t"
      "mov.b64 a, {%2, %2};\n\t"
      "mov.b64 b, {%3, %4};\n\t"
      "mov.b64 c, {%5, %6};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\t"
      "mov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(s), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// s of one pair of points against the query -q (negated, FP32)
template <int D>
__device__ __forceinline__ float2 pair_score(const float4* XY, const float4* B4, const float2* B2,
                                             uint32_t pair, const float (&nq)[D]) {
  const float4 xy = XY[pair];
  float2 s;
  if constexpr (D == 2) {
    s = ffma2(nq[0], make_float2(xy.x, xy.y), B2[pair]);
  } else {
    const float4 zh = B4[pair];
    s = ffma2(nq[2], make_float2(zh.x, zh.y), make_float2(zh.z, zh.w));
    s = ffma2(nq[0], make_float2(xy.x, xy.y), s);
  }
  return ffma2(nq[1], make_float2(xy.z, xy.w), s);
}

// The reference's d2 of point idx (nn.hpp:25-45), FP64, from the exact table.
template <int D>
__device__ __forceinline__ double ref_d2(const LayerTable& hx, const uint8_t* xb, uint32_t idx,
                                         const double (&q)[D]) {
  const double* P = reinterpret_cast<const double*>(xb + hx.off_rec) + static_cast<uint64_t>(idx) * D;
  if constexpr (D == 2) {
    const double dx = __dsub_rn(q[0], P[0]);
    const double dy = __dsub_rn(q[1], P[1]);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  } else {
    const double d0 = __dsub_rn(q[0], P[0]);
    const double d1 = __dsub_rn(q[1], P[1]);
    const double d2 = __dsub_rn(q[2], P[2]);
    double acc = __dadd_rn(0.0, __dmul_rn(d0, d0));
    acc = __dadd_rn(acc, __dmul_rn(d1, d1));
    return __dadd_rn(acc, __dmul_rn(d2, d2));
  }
}

// Projection of P queries against one staged scan table (see the file header).
template <int D, int P>
__device__ __forceinline__ void scan_project(const uint8_t* tb, const uint8_t* xtables,
                                             const double (&x)[P][D], uint32_t (&cell)[P]) {
  const ScanHdr& h = *reinterpret_cast<const ScanHdr*>(tb);
  const float4* XY = reinterpret_cast<const float4*>(tb + sizeof(ScanHdr));
  const float4* B4 = reinterpret_cast<const float4*>(tb + h.off_b);
  const float2* B2 = reinterpret_cast<const float2*>(tb + h.off_b);
  const uint32_t nch = h.n_chunks;
  const float inf = __int_as_float(0x7f800000);
  // best / second-best chunk minima and their chunks, third-best minimum
  float nq[P][D], m1[P], m2[P], m3[P];
  uint32_t b1[P], b2[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
#pragma unroll
    for (int c = 0; c < D; ++c) nq[p][c] = -__double2float_rn(x[p][c]);
    m1[p] = m2[p] = m3[p] = inf;
    b1[p] = b2[p] = 0;
  }
  // pass 1: chunk minima, four pairs (eight points) per step reduced as a
  // two-level FMNMX3 tree so the running minimum is not one long chain
  for (uint32_t ch = 0; ch < nch; ++ch) {
    float cm[P];
#pragma unroll
    for (int p = 0; p < P; ++p) cm[p] = inf;
#pragma unroll
    for (uint32_t j4 = 0; j4 < kScanChunkPairs; j4 += 4) {  // whole chunk: one base address
      const uint32_t pair0 = ch * kScanChunkPairs + j4;
      float2 sv[P][4];
      float2 hb[4];
      if constexpr (D == 2) {  // h of four pairs in two 16-byte loads
        const float4 h01 = B4[pair0 / 2], h23 = B4[pair0 / 2 + 1];
        hb[0] = make_float2(h01.x, h01.y);
        hb[1] = make_float2(h01.z, h01.w);
        hb[2] = make_float2(h23.x, h23.y);
        hb[3] = make_float2(h23.z, h23.w);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 xy = XY[pair0 + u];
        float4 zh;
        if constexpr (D == 3) zh = B4[pair0 + u];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float2 t;
          if constexpr (D == 2) {
            t = ffma2(nq[p][0], make_float2(xy.x, xy.y), hb[u]);
          } else {
            t = ffma2(nq[p][2], make_float2(zh.x, zh.y), make_float2(zh.z, zh.w));
            t = ffma2(nq[p][0], make_float2(xy.x, xy.y), t);
          }
          sv[p][u] = ffma2(nq[p][1], make_float2(xy.z, xy.w), t);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {  // FMNMX3 tree over 8 scores + the running min
        const float a = fminf(fminf(sv[p][0].x, sv[p][0].y), sv[p][1].x);
        const float b = fminf(fminf(sv[p][1].y, sv[p][2].x), sv[p][2].y);
        const float c = fminf(fminf(sv[p][3].x, sv[p][3].y), cm[p]);
        cm[p] = fminf(fminf(a, b), c);
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const bool lt1 = cm[p] < m1[p], lt2 = cm[p] < m2[p];
      m3[p] = fminf(m3[p], lt2 ? m2[p] : cm[p]);
      m2[p] = lt1 ? m1[p] : (lt2 ? cm[p] : m2[p]);
      b2[p] = lt1 ? b1[p] : (lt2 ? ch : b2[p]);
      m1[p] = lt1 ? cm[p] : m1[p];
      b1[p] = lt1 ? ch : b1[p];
    }
  }
  const LayerTable& hx = *reinterpret_cast<const LayerTable*>(xtables + h.exact_off);
  const uint8_t* xb = xtables + h.exact_off;
  const uint32_t lane = threadIdx.x & 31u;
  float tau[P];
  bool ok[P], two[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    // B = 2^-24 1.01 (c_h hmax + c_q sum |q_c| pmax_c), all rounded up
    float sq = 0.0f, qq = 0.0f, qmax = 0.0f;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const float av = fabsf(nq[p][c]);
      sq = __fmaf_ru(av, h.pmax[c], sq);
      qq = __fmaf_ru(av, av, qq);
      qmax = fmaxf(qmax, av);
    }
    const float ch_ = D == 2 ? 3.1f : 4.1f, cq = D == 2 ? 4.1f : 5.1f;
    const float B = __fmul_ru(0x1.02p-24f, __fmaf_ru(ch_, h.hmax, __fmul_ru(cq, sq)));
    const float marg = __fmaf_ru(2.0f, B, __fmul_ru(0x1p-48f, __fadd_ru(__fadd_ru(fabsf(m1[p]), B), qq)));
    tau[p] = __fadd_ru(m1[p], marg);
    // candidates (s <= tau) lie in the best chunk, or also the second-best one
    // when m2 <= tau, if the third-best chunk minimum m3 > tau
    ok[p] = h.fp32_ok && qmax < 0x1p40f && m3[p] > tau[p];  // false for NaN too
    two[p] = !(m2[p] > tau[p]);
    if (two[p]) {  // candidate chunks in index order
      const uint32_t lo = min(b1[p], b2[p]), hi = max(b1[p], b2[p]);
      b1[p] = lo;
      b2[p] = hi;
    }
  }
  // pass 2, per lane: each query rescans its candidate chunk(s) with the
  // pass-1 FFMA2 (same operands, same order, so the same bits) and counts the
  // points with s <= tau, keeping the smallest index. Pairs are visited from a
  // lane-rotated start so the 32 lanes' random chunks spread over the banks
  // (chunks are 256 B apart: without the rotation every lane hits one bank group).
  uint32_t cnt[P], first[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    cnt[p] = 0;
    first[p] = 0xffffffffu;
    if (!ok[p]) continue;
    for (uint32_t w = 0; w < (two[p] ? 2u : 1u); ++w) {
      const uint32_t base = (w ? b2[p] : b1[p]) * kScanChunkPairs;
#pragma unroll 4
      for (uint32_t jj = 0; jj < kScanChunkPairs; ++jj) {
        const uint32_t pair = base + ((jj + lane) & (kScanChunkPairs - 1));
        const float2 sc = pair_score<D>(XY, B4, B2, pair, nq[p]);
        if (sc.x <= tau[p]) {
          ++cnt[p];
          first[p] = min(first[p], 2 * pair);
        }
        if (sc.y <= tau[p]) {
          ++cnt[p];
          first[p] = min(first[p], 2 * pair + 1);
        }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (ok[p] && cnt[p] == 1) {
      cell[p] = first[p];
    } else if (ok[p]) {  // several candidates: the reference's d2 among them, in index order
      uint32_t best = first[p];
      double bd = ref_d2<D>(hx, xb, first[p], x[p]);
      for (uint32_t w = 0; w < (two[p] ? 2u : 1u); ++w) {
        const uint32_t cc = w ? b2[p] : b1[p];
        for (uint32_t jj = 0; jj < kScanChunkPairs; ++jj) {
          const uint32_t pair = cc * kScanChunkPairs + jj;
          const float2 sc = pair_score<D>(XY, B4, B2, pair, nq[p]);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t idx = 2 * pair + e;
            if ((e ? sc.y : sc.x) <= tau[p] && idx > first[p]) {
              const double d = ref_d2<D>(hx, xb, idx, x[p]);
              if (d < bd) {
                bd = d;
                best = idx;
              }
            }
          }
        }
      }
      cell[p] = best;
    } else {  // exact FP64 scan (nn.hpp:18-46)
      cell[p] = nearest<D>(hx, xb, x[p], xtables);
    }
  }
}

template <int K, int SRC, bool RESIDENT, int P>
#ifndef QT_SCAN_MINB2
#define QT_SCAN_MINB2 3
#endif
__global__ void __launch_bounds__(scan_threads<K>(), (P >= 4 || Chain<K>::D == 3) ? 1 : QT_SCAN_MINB2) k_paths_scan(const __grid_constant__ ScanArgs f) {
  using C = Chain<K>;
  constexpr int D = C::D;
  const PathArgs& a = f.p;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kScanMaxStages];
  const uint32_t tid = threadIdx.x;
  const uint32_t S = f.sstages;
  const uint64_t rounds = a.q + (a.rem ? 1u : 0u);
  const uint64_t steps_total = rounds * a.n;
  if (steps_total == 0) return;

  auto issue = [&](uint64_t g) {
    const uint32_t k = static_cast<uint32_t>(g % a.n);
    const uint32_t st = static_cast<uint32_t>(g % S);
    const uint32_t bytes = __ldg(f.stab_bytes + k);
    mbar_expect_tx(&full[st], bytes);
    bulk_g2s(smem + st * f.sbuf_bytes, f.stables + __ldg(f.stab_off + k), bytes, &full[st]);
  };
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    if constexpr (RESIDENT) {
      mbar_expect_tx(&full[0], f.sresident_bytes);
      for (uint32_t k = 0; k < a.n; ++k)
        bulk_g2s(smem + f.stab_off[k], f.stables + f.stab_off[k], f.stab_bytes[k], &full[0]);
    } else {
      for (uint64_t g = 0; g < S && g < steps_total; ++g) issue(g);
    }
  }
  __syncthreads();

  // P slots per thread, slot v = gid P + p owns a contiguous run of paths
  constexpr uint32_t kNT = scan_threads<K>();
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * kNT + tid;
  Source<SRC> src[P];
  uint64_t beg[P], cnt[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t v = gid * P + p;
    cnt[p] = a.q + (v < a.rem ? 1u : 0u);
    beg[p] = a.first + v * a.q + (v < a.rem ? v : a.rem);
    if (cnt[p]) src[p].start(a.src, beg[p]);
  }
  if constexpr (RESIDENT) mbar_wait(&full[0], 0);
  const uint32_t full0 = smem_u32(full);
  uint32_t s = 0, ph = 0;
  uint64_t g = 0;
  const uint8_t* tb = smem;
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
    for (uint32_t k = 1; k <= a.n; ++k, ++g) {
      if constexpr (RESIDENT) {
        tb = smem + f.stab_off[k - 1];
      } else {
        mbar_wait_u32(full0 + 8u * s, ph);
      }
      const ScanHdr& h = *reinterpret_cast<const ScanHdr*>(tb);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (r < cnt[p]) {
          double e[C::NPS], xn[D];
#pragma unroll
          for (int q = 0; q < C::NPS; ++q) e[q] = src[p].normal();
          C::step(h.step, x[p], xn, e);
#pragma unroll
          for (int c = 0; c < D; ++c) x[p][c] = xn[c];
        }
      }
      uint32_t j[P];
      scan_project<D, P>(tb, a.tables, x, j);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (r < cnt[p]) {
          red_add_u64(a.joint + h.joff + static_cast<uint64_t>(i[p]) * h.n_pts + j[p], 1ull);
          i[p] = j[p];
        }
      }
      if constexpr (!RESIDENT) {
        named_barrier_sync(1, kNT);  // every thread is done with stage s
        if (tid == 0 && g + S < steps_total) issue(g + S);
        tb += f.sbuf_bytes;
        if (++s == S) {
          s = 0;
          ph ^= 1u;
          tb = smem;
        }
      }
    }
  }
}

// Alg III (estimate.hpp:213-265) for d >= 2 with the FP32 scan projection:
// CTA = (slice, layer k) as k_alg3, the scan tables of layers k-1 and k in
// shared memory, P samples per thread, both projections through
// scan_project (warp-uniform loops; dummy queries in idle slots).
template <int K, int SRC, int P>
__global__ void __launch_bounds__(256) k_alg3_scan(const __grid_constant__ Alg3ScanArgs f) {
  using C = Chain<K>;
  constexpr int D = C::D;
  const Alg3Args& a = f.a;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t tid = threadIdx.x;
  const uint32_t k = blockIdx.y + 1;  // transition k-1 -> k
  const uint64_t layer0 = static_cast<uint64_t>(k - 1) * a.M;
  uint64_t lo = layer0 + a.M * blockIdx.x / gridDim.x;
  uint64_t hi = layer0 + a.M * (blockIdx.x + 1) / gridDim.x;
  lo = lo > a.first ? lo : a.first;
  hi = hi < a.first + a.count ? hi : a.first + a.count;
  if (lo >= hi) return;
  const uint8_t* tk = smem;
  const uint8_t* tp = smem + f.sbuf_bytes;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t bytes = f.stab_bytes[k - 1] + (k >= 2 ? f.stab_bytes[k - 2] : 0u);
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(smem, f.stables + f.stab_off[k - 1], f.stab_bytes[k - 1], &bar);
    if (k >= 2) bulk_g2s(smem + f.sbuf_bytes, f.stables + f.stab_off[k - 2], f.stab_bytes[k - 2], &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  // layer k's exact header (global): the step and the marginal factor of layer k-1
  const LayerTable& hx = *reinterpret_cast<const LayerTable*>(a.tables + __ldg(a.tab_off + k - 1));
  double stp[6], mg[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    stp[c] = hx.step[c];
    mg[c] = hx.marg_prev[c];
  }
  const ScanHdr& sh = *reinterpret_cast<const ScanHdr*>(tk);
  unsigned long long* jl = a.joint + sh.joff;
  const uint32_t npts = sh.n_pts;
  const uint64_t len = hi - lo, T = static_cast<uint64_t>(blockDim.x) * P;
  const uint64_t q = len / T, rem = len % T;
  Source<SRC> src[P];
  uint64_t cnt[P], beg[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t v = static_cast<uint64_t>(tid) * P + p;
    cnt[p] = q + (v < rem ? 1u : 0u);
    beg[p] = lo + v * q + (v < rem ? v : rem);
    if (cnt[p]) src[p].start(a.src, beg[p]);
  }
  const uint64_t rounds = q + (rem ? 1u : 0u);
  for (uint64_t r = 0; r < rounds; ++r) {
    double x[P][D], xn[P][D];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (r < cnt[p]) {
        if (r > 0) src[p].next_unit(a.src, beg[p] + r);
        double e[D + C::NPS];
#pragma unroll
        for (int q2 = 0; q2 < D + C::NPS; ++q2) e[q2] = src[p].normal();
        C::marginal(mg, k == 1, x[p], e);  // sample_marginal(k-1, ...)
        C::step(stp, x[p], xn[p], e + D);   // step(k-1, ...)
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) x[p][c] = xn[p][c] = 0.0;
      }
    }
    uint32_t j[P], i[P];
    scan_project<D, P>(tk, a.tables, xn, j);
    if (k >= 2) {
      scan_project<D, P>(tp, a.tables, x, i);
    } else {
#pragma unroll
      for (int p = 0; p < P; ++p) i[p] = 0;
    }
#pragma unroll
    for (int p = 0; p < P; ++p)
      if (r < cnt[p]) red_add_u64(jl + static_cast<uint64_t>(i[p]) * npts + j[p], 1ull);
  }
}

template <int K, int SRC>
static cudaError_t launch_alg3_scan_t(const Alg3ScanArgs& a, dim3 g, size_t smem, cudaStream_t st) {
  auto fn = k_alg3_scan<K, SRC, 2>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fn<<<g, 256, smem, st>>>(a);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_alg3_scan_k(int src, const Alg3ScanArgs& a, dim3 g, size_t smem,
                                      cudaStream_t st) {
  switch (src) {
    case kSrcLcg48: return launch_alg3_scan_t<K, kSrcLcg48>(a, g, smem, st);
    case kSrcMrg: return launch_alg3_scan_t<K, kSrcMrg>(a, g, smem, st);
    case kSrcXorwow: return launch_alg3_scan_t<K, kSrcXorwow>(a, g, smem, st);
    default: return launch_alg3_scan_t<K, kSrcNormalsIn>(a, g, smem, st);
  }
}

cudaError_t launch_alg3_scan(int kind, int src, const Alg3ScanArgs& a, uint32_t slices,
                             size_t smem, cudaStream_t st) {
  const dim3 g(slices, a.a.n);
  return kind == 1 ? launch_alg3_scan_k<1>(src, a, g, smem, st)
                   : launch_alg3_scan_k<3>(src, a, g, smem, st);
}

// Batch K2 (NnIndex::nearest over many queries, nn.hpp:150-167) for d >= 2:
// the scan table staged once per CTA, P queries per thread, scan_project's
// exact decision. Loops are warp-uniform (scan_project's rescan is
// warp-cooperative); out-of-range slots query point 0 and are discarded.
// `xtable` is the layer's exact table (LayerTable + FP64 points); the scan
// table's exact_off is relative to it (0).
template <int D, int P>
__global__ void __launch_bounds__(256) k_nearest_scan(const uint8_t* stable, uint32_t sbytes,
                                                      const uint8_t* xtable, const double* q,
                                                      uint64_t nq, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, sbytes);
    bulk_g2s(smem, stable, sbytes, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const uint64_t per_iter = static_cast<uint64_t>(gridDim.x) * blockDim.x * P;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x * P; base < nq;
       base += per_iter) {
    double x[P][D];
    uint64_t qi[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      qi[p] = base + static_cast<uint64_t>(threadIdx.x) * P + p;
      const uint64_t src = qi[p] < nq ? qi[p] : 0;
#pragma unroll
      for (int c = 0; c < D; ++c) x[p][c] = q[src * D + c];
    }
    uint32_t cell[P];
    scan_project<D, P>(smem, xtable, x, cell);
#pragma unroll
    for (int p = 0; p < P; ++p)
      if (qi[p] < nq) out[qi[p]] = cell[p];
  }
}

cudaError_t launch_nearest_scan(int dim, const uint8_t* stable, uint32_t sbytes,
                                const uint8_t* xtable, const double* q, uint64_t nq,
                                unsigned long long* out, cudaStream_t st) {
  constexpr int P = 2;
  const uint64_t want = (nq + 256 * P - 1) / (256 * P);
  const uint32_t blocks = static_cast<uint32_t>(want < 148u * 4u ? (want ? want : 1) : 148u * 4u);
  auto go = [&](auto fn) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sbytes));
    if (e != cudaSuccess) return e;
    fn<<<blocks, 256, sbytes, st>>>(stable, sbytes, xtable, q, nq, out);
    return cudaGetLastError();
  };
  return dim == 2 ? go(k_nearest_scan<2, P>) : go(k_nearest_scan<3, P>);
}

template <int K, int SRC, bool RES, int P>
static cudaError_t launch_scan_t(const ScanArgs& a, uint32_t blocks, size_t smem, cudaStream_t st) {
  auto fn = k_paths_scan<K, SRC, RES, P>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fn<<<blocks, scan_threads<K>(), smem, st>>>(a);
  return cudaGetLastError();
}

template <int K, int SRC, bool RES, int P>
static int scan_bps_t(size_t smem) {
  auto fn = k_paths_scan<K, SRC, RES, P>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, scan_threads<K>(), smem) != cudaSuccess)
    return 1;
  return nb > 0 ? nb : 1;
}

template <int K, int SRC>
static cudaError_t scan_dispatch_p(bool query, int* bps, bool res, int P, const ScanArgs& a,
                                   uint32_t blocks, size_t smem, cudaStream_t st) {
#define QT_SCAN_CASE(PP)                                                                    \
  if (P == PP) {                                                                            \
    if (query) {                                                                            \
      *bps = res ? scan_bps_t<K, SRC, true, PP>(smem) : scan_bps_t<K, SRC, false, PP>(smem); \
      return cudaSuccess;                                                                   \
    }                                                                                       \
    return res ? launch_scan_t<K, SRC, true, PP>(a, blocks, smem, st)                       \
               : launch_scan_t<K, SRC, false, PP>(a, blocks, smem, st);                     \
  }
  QT_SCAN_CASE(1)
  QT_SCAN_CASE(4)
  QT_SCAN_CASE(2)
#undef QT_SCAN_CASE
  return cudaErrorInvalidValue;
}

template <int K>
static cudaError_t scan_dispatch_s(bool query, int* bps, int src, bool res, int P,
                                   const ScanArgs& a, uint32_t blocks, size_t smem,
                                   cudaStream_t st) {
  switch (src) {
    case kSrcLcg48: return scan_dispatch_p<K, kSrcLcg48>(query, bps, res, P, a, blocks, smem, st);
    case kSrcMrg: return scan_dispatch_p<K, kSrcMrg>(query, bps, res, P, a, blocks, smem, st);
    case kSrcXorwow: return scan_dispatch_p<K, kSrcXorwow>(query, bps, res, P, a, blocks, smem, st);
    default: return scan_dispatch_p<K, kSrcNormalsIn>(query, bps, res, P, a, blocks, smem, st);
  }
}

// k_paths_scan for kind 1 (TwoFactorChain, d = 2) / 3 (GbmChain3d, d = 3)
cudaError_t launch_paths_scan(int kind, int src, bool resident, int P, const ScanArgs& a,
                              uint32_t blocks, size_t smem, cudaStream_t st) {
  int dummy = 0;
  return kind == 1 ? scan_dispatch_s<1>(false, &dummy, src, resident, P, a, blocks, smem, st)
                   : scan_dispatch_s<3>(false, &dummy, src, resident, P, a, blocks, smem, st);
}

int paths_scan_blocks_per_sm(int kind, int src, bool resident, int P, size_t smem) {
  int bps = 1;
  ScanArgs dummy{};
  if (kind == 1) scan_dispatch_s<1>(true, &bps, src, resident, P, dummy, 0, smem, nullptr);
  else scan_dispatch_s<3>(true, &bps, src, resident, P, dummy, 0, smem, nullptr);
  return bps;
}

}  // namespace qt
