// qt_layout.h -- host/device shared layout of the per-layer "grid tables"
// that the path kernels stage into shared memory with cp.async.bulk.
//
// One table per layer k = 1..n, 16-byte aligned, contiguous in HBM ("hot"
// part, staged into shared memory):
//
//   LayerTable header (192 B)
//   d == 1 : Thr[N + 1]        per sorted cell c: {t_c, original index of c,
//                              t_{c-1} rounded up to FP32};
//                              t_c is the exact FP64 decision threshold between
//                              sorted cells c and c+1 (t_{N-1} = t_N = +inf)
//            uint16 start[nb]  bucket b -> #{thresholds whose bucket < b}
//   d >= 2 : double pts[N * d] points in ORIGINAL order (row-major), the
//                              reference's scan order (nn.hpp:25-45)
//
// plus, for d == 1, a "cold" block (never staged, read from global memory by
// the exact fallback scan only): Rec1[N] sorted {value, original index}.
//
// The header also carries the chain coefficients of the transition that lands
// on this layer (step of k-1 -> k) and the marginal factor of layer k-1, so a
// CTA that holds a layer's table in shared memory has everything one step needs.
#pragma once
#include <stdint.h>

#include <cmath>

namespace qt {

struct alignas(16) LayerTable {
  double lo;            // d == 1: bucket origin (smallest threshold)
  double inv_w;         // d == 1: buckets per unit of x
  double x_safe;        // d == 1: |x| < x_safe => threshold rule is exact
  double nb_d;          // (double)nb
  double step[6];       // chain coefficients of transition k-1 -> k
  double marg_prev[6];  // marginal factor of layer k-1 (Alg III)
  uint64_t joff;        // element offset of joint[k-1] in the flat joint array
  uint64_t cold_off;    // d == 1: byte offset (from the tables base) of Rec1[N]
  uint32_t n_pts;       // N_k
  uint32_t n_prev;      // N_{k-1}
  uint32_t nb;          // d == 1: number of buckets
  uint32_t off_rec;     // byte offset of Thr[] / pts[] from the table start
  uint32_t off_start;   // byte offset of start[] (d == 1)
  uint32_t bytes;       // hot table bytes (multiple of 16)
  uint32_t layer;       // k
  uint32_t dim;
  float fa;             // d == 1 fast path: |a| of x' = a x + s eps, rounded up (FP32)
  float fs;             // d == 1 fast path: |s|, rounded up (FP32)
  float cert_c;         // d == 1 certified path (x-tables): RU(2^-50 (|a| X_{k-1} + |s| 6.7 + X_k)),
                        // the rounding term of the state bound for |x_{k-1}| < X_{k-1}, |x_k| < X_k
  float cert_xmax;      // d == 1 certified path: X_k = min(x_safe, 8 max |t|) rounded down;
                        // a state beyond it is not certified (replayed)
};
static_assert(sizeof(LayerTable) == 192, "LayerTable header is 192 bytes");

struct alignas(16) Thr {
  double t;
  uint32_t orig;
  float tp;  // t_{c-1} rounded UP to FP32 (-inf for c = 0): x >= tp implies
             // x >= t_{c-1}, the fast path's lower certification bound for cell c
};
static_assert(sizeof(Thr) == 16, "Thr is 16 bytes");

struct alignas(16) Rec1 {
  double v;
  uint32_t orig;
  uint32_t pad;
};
static_assert(sizeof(Rec1) == 16, "Rec1 is 16 bytes");

// ---------------------------------------------------------------------------
// Fast-path layer table (d == 1 only; k_paths_fast). One 16-byte record per
// bucket of an FP32 bucket map b(x) = min(u32_rz(fmaf(g(x), bk_a, bk_b)),
// nb - 1) over the density-equalising coordinate g(x) = x / sqrt(1 + gc x^2)
// (the Lloyd cells are ~5x narrower at the centre than in the tails). With
// c = #{thresholds t whose b(t) < b}, the record holds the thresholds around
// c rounded OUTWARD to FP32 and the original indices of cells c and c + 1, so
// one 16-byte shared-memory load decides and certifies a transition:
//   x in [xl, xh], xh < t0      and xl >= tl      -> cell o0
//   x in [xl, xh], xh < t1      and xl >= up(t0)  -> cell o1
// Any other case is left uncertified (-> exact replay). The record carries the
// bounds of the cell it certifies, so correctness never depends on the bucket
// map: the device's approximate g (MUFU rsqrt) may differ from the host's at
// bucket edges, which only costs a (vanishingly rare) replay.
// ---------------------------------------------------------------------------
struct alignas(16) FastHdr {
  double c0, c2;      // step coefficients: Brownian x + c0 eps; OU c0 x + c2 eps
  uint64_t joff;      // element offset of joint[k-1]
  float fa, fs;       // |a|, |s| rounded up
  float bk_a, bk_b;   // FP32 bucket map
  float x_safe;       // exact-kernel x_safe rounded down (0: never certify)
  uint32_t nb1;       // buckets - 1
  uint32_t n_pts;     // N_k
  uint32_t bytes;     // table bytes (multiple of 16)
  float gc;           // density-equalising map u = x / sqrt(1 + gc x^2) before bucketing
  uint32_t pad_;
};
static_assert(sizeof(FastHdr) == 64, "FastHdr is 64 bytes");

struct alignas(16) FRec {
  float tl;            // t_{c-1} rounded up (-inf for c = 0)
  float t0;            // t_c rounded down (never -0)
  float t1;            // t_{c+1} rounded down (+inf past the last cell)
  uint16_t o0, o1;     // original indices of cells c, c + 1
};
static_assert(sizeof(FRec) == 16, "FRec is 16 bytes");

// The bucket map: host (table build, FP64) and device (query, FP32 + MUFU).
#if defined(__CUDACC__)
__device__ __forceinline__ uint32_t fbucket(float xs, float gc, float bk_a, float bk_b,
                                            uint32_t nb1) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fmaf_rn(gc, __fmul_rn(xs, xs), 1.0f)));
  const uint32_t b = __float2uint_rz(__fmaf_rn(__fmul_rn(xs, r), bk_a, bk_b));
  return b < nb1 ? b : nb1;
}
#endif
inline double fmap_g(double x, double gc) { return x / std::sqrt(1.0 + gc * x * x); }
inline uint32_t fbucket_host(double x, double gc, double bk_a, double bk_b, uint32_t nb1) {
  const double v = fmap_g(x, gc) * bk_a + bk_b;
  const uint32_t b = !(v > 0.0) ? 0u : (v >= 4294967295.0 ? 0xFFFFFFFFu : static_cast<uint32_t>(v));
  return b < nb1 ? b : nb1;
}

// ---------------------------------------------------------------------------
// FP32 scan table (d >= 2; k_paths_scan). Points in ORIGINAL order, padded to
// whole chunks of kScanChunkPairs pairs, stored as pairs of FP32 lanes so one
// FFMA2 evaluates two points against a broadcast query coordinate:
//   d == 2:  float4 XY[pair] = {x_a, x_b, y_a, y_b};  float2 H[pair] = {h_a, h_b}
//   d == 3:  float4 XY[pair];                           float4 ZH[pair] = {z_a, z_b, h_a, h_b}
// with h = fl32(|p|^2 / 2); the score s = h - q.p orders the points like
// |q - p|^2 (= 2 s + |q|^2). Padding points have p = 0, h = +inf.
// ---------------------------------------------------------------------------
constexpr uint32_t kScanChunkPairs = 16;  // 32 points per chunk

// ---------------------------------------------------------------------------
// Cell-list index of one d >= 2 layer (qt_cell.cu), in global memory: a
// CellHdr per layer, one start[] array over all layers' buckets (u32, the
// list position of each bucket, plus a final end) and one list[] of u16 point
// indices (ascending per bucket). The bounding box [lo, lo + g w) of the
// layer's points (plus a margin) is cut into g[0] x g[1] (x g[2]) buckets;
// bucket b lists every point that can be the reference's nearest point
// (nn.hpp:18-46, FP64 d2, strict <) -- or tie with it -- for some query in b,
// so the exact argmin over the list equals the brute-force one. Queries
// outside the box (or non-finite) take the exact full scan. The lists are
// built on the device (k_cell_count / k_cell_fill).
// ---------------------------------------------------------------------------
struct alignas(16) CellHdr {
  double lo[3];        // box origin per axis
  double w[3];         // bucket width per axis
  double inv_w[3];     // buckets per unit length per axis (the query's bucket map)
  uint64_t start_off;  // index of this layer's bucket 0 in start[]
  uint32_t g[3];       // buckets per axis (1 on unused axes)
  uint32_t ok;         // 0: no bucket grid (degenerate layer): always the full scan
};
static_assert(sizeof(CellHdr) == 96, "CellHdr is 96 bytes");

struct alignas(16) ScanHdr {
  double step[6];     // chain coefficients of transition k-1 -> k
  uint64_t joff;      // element offset of joint[k-1]
  uint64_t exact_off; // byte offset (from the exact tables base) of this layer's LayerTable
  float hmax;         // max h over the layer
  float pmax[3];      // max |p_c| per coordinate
  uint32_t n_pts;     // N_k
  uint32_t n_chunks;  // chunks of kScanChunkPairs pairs
  uint32_t off_b;     // byte offset of H[] (d == 2) / ZH[] (d == 3)
  uint32_t bytes;     // table bytes (multiple of 16)
  uint32_t fp32_ok;   // all |p_c| < 2^40 (else every query takes the exact FP64 scan)
  uint32_t pad_[7];
};
static_assert(sizeof(ScanHdr) == 128, "ScanHdr is 128 bytes");

constexpr uint32_t kNoIndex = 0xFFFFFFFFu;

// Bucket of x under a layer's (lo, inv_w, nb): identical IEEE operations on
// host and device (one subtraction, one multiplication, truncation), so the
// start[] table built on the host is exact for every device query.
#if defined(__CUDACC__)
__host__ __device__
#endif
inline uint32_t bucket_of(double x, double lo, double inv_w, double nb_d, uint32_t nb) {
#if defined(__CUDA_ARCH__)
  const double t = __dmul_rn(__dsub_rn(x, lo), inv_w);
#else
  volatile double d = x - lo;  // volatile: no contraction or reassociation
  const double t = d * inv_w;
#endif
  return t > 0.0 ? (t < nb_d ? static_cast<uint32_t>(t) : nb - 1u) : 0u;
}

}  // namespace qt
