// qt_kernels.cu -- the sm_100a kernels of the transition estimator.
//
//  k_paths_x   the default 1-D path kernel (Brownian / OU, MRG32k3a): Alg I/II
//              (estimate.hpp:88-126) fused K1+K2+K3 -- MRG32k3a block substream per
//              path, FP64 Box-Muller, chain step, exact threshold projection, one
//              red.global.add.u64 into joint[k-1][i*N_k + j]. Lockstep CTA
//              pipeline: thread 0 prefetches two-layer table stages with
//              cp.async.bulk, one named barrier per two layers, P paths per thread.
//  k_paths     the same path for every engine and for parity mode (normals in),
//              d = 1..3: a warp-specialised TMA producer and a full/empty mbarrier
//              ring of layer tables.
//  k_paths_fast + k_replay  opt-in 1-D fast path: FP32 Box-Muller with verified
//              error bounds, certified FP32 cell records, exact replay of the
//              uncertified paths (identical counts).
//  k_alg3_x / k_alg3  K4: Alg III layer-parallel pair sampler (estimate.hpp:213-265):
//              CTA = (layer k, slice of its M samples), tables of layers k-1 and k
//              resident in shared memory, two projections per sample.
//  k_colsum / k_rowsum / k_normalize
//              visits from the joint counts + row normalisation (quant_tree.hpp:69-83).
//  k_nearest, k_path_normals, k_uniforms, k_fast_bounds_check  standalone K2, RNG
//              probes and the exhaustive FP32 Box-Muller bound check.
// d >= 2 path kernels live in qt_scan.cu, the pricers in qt_bdp.cu, grid
// construction in qt_lloyd.cu, micro-benchmarks in qt_bench.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qt_device.cuh"
#include "qt_internal.h"
#include "qt_math_fast.h"

namespace qt {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Alg I / II. Warp-specialised: warp 8 is the TMA producer, warps 0-7 the
// consumers. Layer tables cycle through S shared-memory stages guarded by a
// full/empty mbarrier ring, so consumer warps never meet at a CTA barrier and
// may drift up to S layers apart.
// ---------------------------------------------------------------------------
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kPathThreads = kConsumers + 32;
constexpr int kMaxStages = 8;
constexpr int kFastThreads = 256;  // k_paths_fast: 8 warps in layer lockstep

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int K, int SRC, bool RESIDENT>
__global__ void __launch_bounds__(kPathThreads) k_paths(const PathArgs a) {
  using C = Chain<K>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ __align__(8) uint64_t empty[kMaxStages];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  const uint32_t S = a.stages;
  const uint64_t rounds = a.q + (a.rem ? 1u : 0u);
  const uint64_t steps_total = rounds * a.n;
  if (steps_total == 0) return;

  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {  // ---- producer warp ----
    if (lane == 0) {
      if constexpr (RESIDENT) {
        mbar_expect_tx(&full[0], a.resident_bytes);
        for (uint32_t k = 0; k < a.n; ++k)
          bulk_g2s(smem + (a.tab_off[k] - a.tab_off[0]), a.tables + a.tab_off[k], a.tab_bytes[k],
                   &full[0]);
      } else {
        uint32_t k = 0, s = 0, ph = 0;
        for (uint64_t g = 0; g < steps_total; ++g) {
          mbar_wait(&empty[s], ph ^ 1u);  // a fresh barrier passes parity 1 at once
          const uint32_t bytes = __ldg(a.tab_bytes + k);
          mbar_expect_tx(&full[s], bytes);
          bulk_g2s(smem + s * a.buf_bytes, a.tables + __ldg(a.tab_off + k), bytes, &full[s]);
          k = k + 1 == a.n ? 0 : k + 1;
          if (++s == S) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ---- consumer warps: one path at a time per thread ----
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * kConsumers + tid;
  const uint64_t mycount = a.q + (gid < a.rem ? 1u : 0u);
  const uint64_t mybeg = a.first + gid * a.q + (gid < a.rem ? gid : a.rem);
  if constexpr (RESIDENT) mbar_wait(&full[0], 0);

  Source<SRC> src;
  if (mycount) src.start(a.src, mybeg);
  uint32_t s = 0, ph = 0;  // ring position
  for (uint64_t r = 0; r < rounds; ++r) {
    const bool active = r < mycount;
    if (active && r > 0) src.next_unit(a.src, mybeg + r);
    double x[C::D];
#pragma unroll
    for (int d = 0; d < C::D; ++d) x[d] = 0.0;  // initial(): the origin (chains.hpp:43-46,81)
    uint32_t i = 0;                             // layer 0 is the singleton {x0}
    for (uint32_t k = 1; k <= a.n; ++k) {
      const uint8_t* tb;
      if constexpr (RESIDENT) {
        tb = smem + (a.tab_off[k - 1] - a.tab_off[0]);
      } else {
        tb = smem + s * a.buf_bytes;
        mbar_wait(&full[s], ph);
      }
      const LayerTable& h = *reinterpret_cast<const LayerTable*>(tb);
      if (active) {
        double e[C::NPS], xn[C::D];
#pragma unroll
        for (int q = 0; q < C::NPS; ++q) e[q] = src.normal();
        C::step(h.step, x, xn, e);
#pragma unroll
        for (int d = 0; d < C::D; ++d) x[d] = xn[d];
        const uint32_t j = nearest<C::D>(h, tb, x, a.tables);
        red_add_u64(a.joint + h.joff + static_cast<uint64_t>(i) * h.n_pts + j, 1ull);
        i = j;
      }
      if constexpr (!RESIDENT) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Fast 1-D path (Brownian / OU chains, MRG32k3a): the same warp-specialised
// ring as k_paths, but the normals come from the FP32 Box-Muller of
// qt_device.cuh with a rigorous error bound, the state x~ is carried in FP64
// together with an FP32 bound e >= |x~ - x| on the exact kernel's state x, and
// a transition is counted only when [x~ - e, x~ + e] lies inside one cell
// (t_{c-1} <= x~ - e, x~ + e < t_c). The first uncertified transition of a
// path ends its counting here; the path is appended to the replay list and
// k_replay recomputes it with the exact FP64 arithmetic of k_paths, counting
// from that layer on. The counts are therefore identical to k_paths' counts.
// ---------------------------------------------------------------------------

// Per-slot state of the fast kernel (one path in flight).
struct FastPath {
  Mrg st;
  uint64_t beg, count;  // this slot's contiguous run of paths
  double x;             // x~
  float e;              // |x~ - x| <= e
  float xs;             // x~ rounded to FP32 (bucket + rounding term)
  float zs, bzs;        // Box-Muller mate and its bound
  uint32_t i;           // cell at the previous layer
  uint32_t amb_k;       // first uncertified layer (0: none so far)
};

// One layer k for the P slots of a thread, against the layer's fast table
// (FastHdr + FRec[], qt_layout.h). Written as straight-line phases over the
// slots, so the compiler interleaves the P independent dependency chains.
// Per transition: one 16-byte shared-memory record and FP32 compares decide
// and certify the cell; nothing on this path is FP64 except the state x~.
template <int K, int P>
__device__ __forceinline__ void fast_layer(FastPath (&ps)[P], const bool (&act)[P],
                                           const uint8_t* tb, uint32_t k,
                                           unsigned long long* joint, bool count) {
  const FastHdr& h = *reinterpret_cast<const FastHdr*>(tb);
  const double c0 = h.c0;
  const double c2 = K == 0 ? 0.0 : h.c2;
  const float fa = h.fa, fs = h.fs, bk_a = h.bk_a, bk_b = h.bk_b, x_safe = h.x_safe, gc = h.gc;
  const uint32_t nb1 = h.nb1, npts = h.n_pts;
  const FRec* R = reinterpret_cast<const FRec*>(tb + sizeof(FastHdr));
  unsigned long long* jl = joint + h.joff;

  float z[P], bz[P];
  if (k & 1u) {  // a fresh pair (stream.hpp:97-108): z = r cos, mate = r sin
    uint32_t u1[P], u2[P];
#pragma unroll
    for (int p = 0; p < P; ++p) mrg_step2(ps[p].st, u1[p], u2[p]);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float rr = fast_radius(u1[p]);
      float c, sn;
      fast_angle(u2[p], c, sn);
      z[p] = __fmul_rn(rr, c);
      ps[p].zs = __fmul_rn(rr, sn);
      bz[p] = __fmaf_ru(kBzB, rr, kBzA);
      ps[p].bzs = bz[p];
    }
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      z[p] = ps[p].zs;
      bz[p] = ps[p].bzs;
    }
  }
  FRec rec[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const double zd = static_cast<double>(z[p]);
    double xn;
    if constexpr (K == 0) xn = __fma_rn(c0, zd, ps[p].x);            // x + s eps
    else xn = __fma_rn(c0, ps[p].x, __dmul_rn(c2, zd));             // a x + s eps
    const float xns = __double2float_rn(xn);
    // e' = fa e + fs bz + 2^-49 (|x| + 2 |x'|): the FP64 roundings of both
    // recurrences (|x| <= |xs| (1 + 2^-23)); fs |z| 2^-50 is inside kBzB's slack
    ps[p].e = __fmaf_ru(fa, ps[p].e,
                        __fmaf_ru(fs, bz[p], __fmul_ru(0x1p-49f, __fmaf_ru(2.0f, fabsf(xns),
                                                                            fabsf(ps[p].xs)))));
    ps[p].x = xn;
    ps[p].xs = xns;
    rec[p] = R[fbucket(xns, gc, bk_a, bk_b, nb1)];
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const float xs = ps[p].xs;
    // [x~ - e, x~ + e] inside [xl, xh]: E also covers |xs - x~| <= 2^-24 |x~|
    const float E = __fmaf_ru(fabsf(xs), 0x1p-23f, ps[p].e);
    const float xl = __fadd_rd(xs, -E), xh = __fadd_ru(xs, E);
    const FRec& r = rec[p];
    const bool lo = xs < r.t0;
    const float up0 = __int_as_float(__float_as_int(r.t0) + (r.t0 >= 0.0f ? 1 : -1));  // >= t_c
    const float lb = lo ? r.tl : up0;
    const float ub = lo ? r.t0 : r.t1;
    const uint32_t cell = lo ? r.o0 : r.o1;
    const bool ok = xl >= lb && xh < ub && __fadd_ru(fabsf(xs), E) < x_safe;
    const bool live = act[p] && ps[p].amb_k == 0;
    if (live && ok && count) red_add_u64(jl + static_cast<uint64_t>(ps[p].i) * npts + cell, 1ull);
    ps[p].i = cell;
    if (live && !ok) ps[p].amb_k = k;
  }
}

// Replay of an ambiguous path from its stored start state (no jump-ahead).
template <int K>
__device__ __noinline__ void replay_entry(const PathArgs& a, unsigned long long* joint,
                                          const AmbEntry& ent) {
  using C = Chain<K>;
  Source<kSrcMrg> src;
  src.s = Mrg{ent.st[0], ent.st[1], ent.st[2], ent.st[3], ent.st[4], ent.st[5]};
  src.has = false;
  const uint32_t k0 = static_cast<uint32_t>(ent.key & 0xFFFFu);
  double x[1] = {0.0};
  uint32_t i = 0;
  for (uint32_t k = 1; k <= a.n; ++k) {
    const uint8_t* tb = a.tables + __ldg(a.tab_off + k - 1);
    const LayerTable& h = *reinterpret_cast<const LayerTable*>(tb);
    double e[1], xn[1];
    e[0] = src.normal();
    C::step(h.step, x, xn, e);
    x[0] = xn[0];
    if (k + 1 < k0) continue;  // the prefix only needs the exact state, not its cells
    const uint32_t j = nearest_1d(h, tb, x[0], a.tables);
    if (k >= k0) red_add_u64(joint + h.joff + static_cast<uint64_t>(i) * h.n_pts + j, 1ull);
    i = j;
  }
}

// state <- M state with M = 18 residues in generic (param-space) memory
__device__ __forceinline__ void mrg_apply(const uint32_t* M, Mrg& s) {
  uint32_t r[6];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    r[i] = red_m1(static_cast<uint64_t>(red_m1(mulw(M[3 * i], s.a0))) + red_m1(mulw(M[3 * i + 1], s.a1)) +
                  red_m1(mulw(M[3 * i + 2], s.a2)));
    r[3 + i] = red_m2(static_cast<uint64_t>(red_m2(mulw(M[9 + 3 * i], s.b0))) +
                      red_m2(mulw(M[9 + 3 * i + 1], s.b1)) + red_m2(mulw(M[9 + 3 * i + 2], s.b2)));
  }
  s = Mrg{r[0], r[1], r[2], r[3], r[4], r[5]};
}

// The fast path kernel. All 256 threads of a CTA walk the layers in lockstep
// (one named barrier per layer); thread 0 keeps the next fstages - 1 layer
// tables in flight with cp.async.bulk, each stage reused only after the
// barrier that ends its layer. Slot v = gid P + p owns a contiguous run of
// paths, so its MRG32k3a stream flows from path to path without jumps.
template <int K, bool RESIDENT, int P>
__global__ void __launch_bounds__(kFastThreads) k_paths_fast(const __grid_constant__ FastArgs f) {
  const PathArgs& a = f.p;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  const uint32_t tid = threadIdx.x;
  const uint32_t S = f.fstages;
  // layers per stage: 2 = the pair sharing one Box-Muller draw (one table wait and
  // one barrier per pair), 1 = half the ring's shared memory (more CTAs per SM)
  const uint32_t L = f.flayers == 1 ? 1u : 2u;
  const uint32_t spr = (a.n + L - 1) / L;
  const uint64_t rounds = a.q + (a.rem ? 1u : 0u);
  const uint64_t steps_total = rounds * spr;
  if (steps_total == 0) return;

  // issue the tables of global stage step g into its stage (thread 0 only)
  auto issue = [&](uint64_t g) {
    const uint32_t k0 = static_cast<uint32_t>(g % spr) * L;
    const uint32_t k1 = min(k0 + L, a.n) - 1;
    const uint32_t st = static_cast<uint32_t>(g % S);
    const uint32_t off = __ldg(f.ftab_off + k0);
    const uint32_t bytes = __ldg(f.ftab_off + k1) + __ldg(f.ftab_bytes + k1) - off;
    mbar_expect_tx(&full[st], bytes);
    bulk_g2s(smem + st * f.fbuf_bytes, f.ftables + off, bytes, &full[st]);
  };
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    if constexpr (RESIDENT) {
      mbar_expect_tx(&full[0], f.fresident_bytes);
      for (uint32_t k = 0; k < a.n; ++k)
        bulk_g2s(smem + f.ftab_off[k], f.ftables + f.ftab_off[k], f.ftab_bytes[k], &full[0]);
    } else {
      for (uint64_t g = 0; g < S && g < steps_total; ++g) issue(g);
    }
  }
  __syncthreads();

  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * kFastThreads + tid;
  FastPath ps[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t v = gid * P + p;
    ps[p].count = a.q + (v < a.rem ? 1u : 0u);
    ps[p].beg = a.first + v * a.q + (v < a.rem ? v : a.rem);
    ps[p].st = Mrg{};
    if (ps[p].count) {
      Source<kSrcMrg> src;
      src.start(a.src, ps[p].beg);
      ps[p].st = src.s;
    }
  }
  if constexpr (RESIDENT) mbar_wait(&full[0], 0);
  const uint32_t full0 = smem_u32(full);
  uint32_t s = 0, ph = 0;
  uint64_t g = 0;
  const uint8_t* tb = smem;
  for (uint64_t r = 0; r < rounds; ++r) {
    bool act[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      act[p] = r < ps[p].count;
      ps[p].x = 0.0;  // chains.hpp:43-46,81: the origin
      ps[p].e = 0.0f;
      ps[p].xs = 0.0f;
      ps[p].i = 0;
      ps[p].amb_k = 0;
    }
    for (uint32_t k = 1; k <= a.n; k += L, ++g) {
      if constexpr (RESIDENT) {
        tb = smem + f.ftab_off[k - 1];
      } else {
        mbar_wait_u32(full0 + 8u * s, ph);
      }
      fast_layer<K, P>(ps, act, tb, k, f.sjoint, f.probe_nored == 0);
      if (L == 2 && k + 1 <= a.n)
        fast_layer<K, P>(ps, act, tb + __ldg(f.ftab_bytes + k - 1), k + 1, f.sjoint,
                         f.probe_nored == 0);
      if constexpr (!RESIDENT) {
        named_barrier_sync(1, kFastThreads);  // every thread is done with stage s
        if (tid == 0 && g + S < steps_total) issue(g + S);
        tb += f.fbuf_bytes;
        if (++s == S) {
          s = 0;
          ph ^= 1u;
          tb = smem;
        }
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (act[p] && ps[p].amb_k != 0) {
        AmbEntry ent;
        ent.key = ((ps[p].beg + r) << 16) | ps[p].amb_k;
        Mrg st0 = ps[p].st;
        mrg_apply(f.back, st0);  // the path's start state
        ent.st[0] = st0.a0;
        ent.st[1] = st0.a1;
        ent.st[2] = st0.a2;
        ent.st[3] = st0.b0;
        ent.st[4] = st0.b1;
        ent.st[5] = st0.b2;
        const unsigned long long idx = atomicAdd(f.stats, 1ull);
        if (idx < f.cap) {
          f.amb[idx] = ent;
        } else {  // list full: replay here (correct, slow; never expected)
          replay_entry<K>(a, a.joint, ent);
          atomicAdd(f.stats + 2, 1ull);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_paths_x: the exact 1-D path kernel for MRG32k3a (Brownian / OU), i.e.
// k_paths' arithmetic bit for bit, in the lockstep CTA pipeline of
// k_paths_fast: no producer warp, one named barrier per layer, thread 0
// prefetching the next S - 1 layer tables, P paths in flight per thread so
// one table wait and one header read serve P transitions, and the Box-Muller
// pair drawn with two interleaved MRG32k3a steps.
// ---------------------------------------------------------------------------
struct ExactPath {
  Mrg st;
  double x;     // state (chains.hpp: origin at the path start); CERT: x~
  double zs;    // Box-Muller mate
  uint32_t i;   // cell at the previous layer
  // CERT only: |x~ - x| <= e against the exact kernel's state x, the mate's
  // bound (both FP32, rounded up), and the first layer whose cell was not
  // certified (0: none yet)
  float e;
  float bzs;
  uint32_t amb_k;
};

// Sorted position (not the original index) of the exact scan's answer: the
// same (d2, original index) order as nearest_1d_scan.
static __device__ __noinline__ uint32_t nearest_1d_scan_pos(const Rec1* R, uint32_t n, double x) {
  uint32_t best = 0, best_orig = 0;
  double bd = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (uint32_t s = 0; s < n; ++s) {
    const Rec1 r = R[s];
    const double d = __dsub_rn(x, r.v);
    const double d2 = __dmul_rn(d, d);
    if (d2 < bd || (d2 == bd && r.orig < best_orig)) {
      bd = d2;
      best = s;
      best_orig = r.orig;
    }
  }
  return best;
}

// The sorted cell of x on an x-table (threshold pairs PT[c] = {t_c, t_c+1}):
// nearest_1d's rule with one 16-byte record per query.
__device__ __forceinline__ uint32_t nearest_1d_pos(const LayerTable& h, const uint8_t* tb, double x,
                                                   const uint8_t* gtables) {
  if (!(fabs(x) < h.x_safe))
    return nearest_1d_scan_pos(reinterpret_cast<const Rec1*>(gtables + h.cold_off), h.n_pts, x);
  const double2* PT = reinterpret_cast<const double2*>(tb + h.off_rec);
  const uint16_t* start = reinterpret_cast<const uint16_t*>(tb + h.off_start);
  const uint32_t c = start[bucket_of(x, h.lo, h.inv_w, h.nb_d, h.nb)];  // all t_{<c} < x
  const double2 r = PT[c];
  if (x < r.x) return c;
  if (x < r.y) return c + 1;
  uint32_t cc = c + 2;
  while (!(x < PT[cc].x)) ++cc;  // t_{N-1} = +inf stops the walk
  return cc;
}

// One layer of P paths. The staged table is the x-table: Thr[] replaced by the
// threshold pairs PT[c] = {t_c, t_c+1} (one 16-byte load decides the usual
// two-step bracket), and the cell is kept as its SORTED position c; the
// counts land in sorted-cell space (sjoint) and launch_permute_add maps them
// to the reference's original indices once per count call.
template <int K, int P, bool CERT>
__device__ __forceinline__ void exact_layer(ExactPath (&ps)[P], const bool (&act)[P],
                                            const uint8_t* tb, uint32_t k,
                                            unsigned long long* joint, const uint8_t* gtables,
                                            bool count, uint32_t* hist1) {
  using C = Chain<K>;
  const LayerTable& h = *reinterpret_cast<const LayerTable*>(tb);
  const double x_safe = h.x_safe, lo = h.lo, inv_w = h.inv_w, nb_d = h.nb_d;
  const uint32_t nb = h.nb, npts = h.n_pts;
  const double2* PT = reinterpret_cast<const double2*>(tb + h.off_rec);
  const uint16_t* start = reinterpret_cast<const uint16_t*>(tb + h.off_start);
  unsigned long long* jl = joint + h.joff;
  double z[P];
  float bz[P];
  if (k & 1u) {  // a fresh pair (stream.hpp:97-108): z1 now, z2 cached
    double u1[P], u2[P], zs[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      uint32_t a1, a2;
      mrg_step2(ps[p].st, a1, a2);
      u1[p] = mrg_to_unit(a1);
      u2[p] = mrg_to_unit(a2);
    }
    if constexpr (CERT) {  // approximate FP64 pair with its verified bound (qt_math_fast.h)
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double r = apx::radius(u1[p]);
        double sn, cs;
        apx::sincos(__dmul_rn(kTwoPi, u2[p]), &sn, &cs);
        z[p] = __dmul_rn(r, cs);
        zs[p] = __dmul_rn(r, sn);
        bz[p] = __double2float_ru(__dmul_ru(r, apx::kApxZ));
        ps[p].bzs = bz[p];
      }
    } else {
      box_muller_batch<P>(u1, u2, z, zs);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) ps[p].zs = zs[p];
  } else {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      z[p] = ps[p].zs;
      if constexpr (CERT) bz[p] = ps[p].bzs;
    }
  }
  uint32_t c[P];
  bool safe[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    double xn[1], e[1] = {z[p]}, xo[1] = {ps[p].x};
    C::step(h.step, xo, xn, e);
    if constexpr (CERT) {
      // e' >= |x~' - x'| for x' = RN(RN(a x) + RN(s z)) (Brownian: a = 1, no
      // product): |a| e + |s| bz, plus 2^-50 of every operand for the roundings
      // that may differ; FP32 with every operation rounded up (fa, fs >= |a|, |s|)
      // |x_{k-1}| < X_{k-1} (certified, or the origin) and |x_k| < X_k (checked
      // below) bound those operands: the per-layer h.cert_c (make_plan)
      const float lin = __fmaf_ru(h.fa, ps[p].e, __fmul_ru(h.fs, bz[p]));
      ps[p].e = __fadd_ru(__fmaf_ru(lin, 0x1p-50f, lin), h.cert_c);
      const double ed = static_cast<double>(ps[p].e);
      const double xl = __dsub_rd(xn[0], ed);
      safe[p] = __dadd_ru(fabs(xn[0]), ed) < static_cast<double>(h.cert_xmax);
      c[p] = start[bucket_of(safe[p] ? xl : 0.0, lo, inv_w, nb_d, nb)];  // all t_{<c} < xl
    } else {
      safe[p] = fabs(xn[0]) < x_safe;
      c[p] = start[bucket_of(safe[p] ? xn[0] : 0.0, lo, inv_w, nb_d, nb)];  // all t_{<c} < x
    }
    ps[p].x = xn[0];
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const double x = ps[p].x;
    uint32_t j;
    if constexpr (CERT) {
      // the cell of every state in [x~ - e, x~ + e]: c if xh < t_c, c + 1 if
      // t_c <= xl and xh < t_c+1; anything else (or |x| near x_safe) is not
      // certified and the path is replayed exactly from its start
      const double ed = static_cast<double>(ps[p].e);
      const double xl = __dsub_rd(x, ed), xh = __dadd_ru(x, ed);
      const double2 r = PT[c[p]];
      const bool in0 = xh < r.x;
      const bool in1 = !(xl < r.x) && xh < r.y;
      j = in0 ? c[p] : c[p] + 1;
      if (act[p] && ps[p].amb_k == 0) {
        if (safe[p] && (in0 || in1)) {
          if (hist1 && k == 1) atomicAdd(hist1 + j, 1u);  // row 0 of joint[0], per CTA
          else if (count) red_add_u64(jl + static_cast<uint64_t>(ps[p].i) * npts + j, 1ull);
        } else {
          ps[p].amb_k = k;
        }
      }
    } else {
      if (safe[p]) {
        const double2 r = PT[c[p]];
        if (x < r.x) {
          j = c[p];
        } else if (x < r.y) {
          j = c[p] + 1;
        } else {
          uint32_t cc = c[p] + 2;
          while (!(x < PT[cc].x)) ++cc;  // t_{N-1} = +inf stops the walk
          j = cc;
        }
      } else {  // exact scan over the cold block (NaN / inf / |x| >= x_safe)
        j = nearest_1d_scan_pos(reinterpret_cast<const Rec1*>(gtables + h.cold_off), npts, x);
      }
      if (act[p]) {
        if (hist1 && k == 1) atomicAdd(hist1 + j, 1u);
        else if (count) red_add_u64(jl + static_cast<uint64_t>(ps[p].i) * npts + j, 1ull);
      }
    }
    ps[p].i = j;
  }
}

// L = layers per pipeline stage: with L = 2 one stage holds the (contiguous)
// tables of layers 2q+1 and 2q+2, which share one Box-Muller pair, so the table
// wait and the barrier are paid once per two layers.
template <int K, bool RESIDENT, int P, int L, bool CERT>
__global__ void __launch_bounds__(kXThreads, QT_X_MINB) k_paths_x(const __grid_constant__ PathArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  const uint32_t tid = threadIdx.x;
  const uint32_t S = a.stages;
  const uint32_t spr = (a.n + L - 1) / L;  // stage steps per round
  uint32_t* hist1 = a.n1 ? reinterpret_cast<uint32_t*>(smem + a.hist1_off) : nullptr;
  for (uint32_t c = tid; c < a.n1; c += kXThreads) hist1[c] = 0u;
  const uint64_t rounds = a.q + (a.rem ? 1u : 0u);
  const uint64_t steps_total = rounds * spr;
  if (steps_total == 0) return;
  auto issue = [&](uint64_t g) {
    const uint32_t k0 = static_cast<uint32_t>(g % spr) * L;
    const uint32_t k1 = min(k0 + L, a.n) - 1;
    const uint32_t st = static_cast<uint32_t>(g % S);
    const uint32_t off = __ldg(a.tab_off + k0);
    const uint32_t bytes = __ldg(a.tab_off + k1) + __ldg(a.tab_bytes + k1) - off;
    mbar_expect_tx(&full[st], bytes);
    bulk_g2s(smem + st * a.buf_bytes, a.xtables + off, bytes, &full[st]);
  };
  if (tid == 0) {
    for (uint32_t s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    if constexpr (RESIDENT) {
      mbar_expect_tx(&full[0], a.resident_bytes);
      for (uint32_t k = 0; k < a.n; ++k)
        bulk_g2s(smem + (a.tab_off[k] - a.tab_off[0]), a.xtables + a.tab_off[k], a.tab_bytes[k],
                 &full[0]);
    } else {
      for (uint64_t g = 0; g < S && g < steps_total; ++g) issue(g);
    }
  }
  __syncthreads();

  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * kXThreads + tid;
  ExactPath ps[P];
  uint64_t cnt[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t v = gid * P + p;
    cnt[p] = a.q + (v < a.rem ? 1u : 0u);
    const uint64_t beg = a.first + v * a.q + (v < a.rem ? v : a.rem);
    ps[p].st = Mrg{};
    if (cnt[p]) {
      Source<kSrcMrg> src;
      src.start(a.src, beg);
      ps[p].st = src.s;
    }
  }
  if constexpr (RESIDENT) mbar_wait(&full[0], 0);
  const uint32_t full0 = smem_u32(full);
  uint32_t s = 0, ph = 0;
  uint64_t g = 0;
  const uint8_t* tb = smem;
  for (uint64_t r = 0; r < rounds; ++r) {
    bool act[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      act[p] = r < cnt[p];
      ps[p].x = 0.0;  // chains.hpp:43-46,81: the origin
      ps[p].i = 0;    // layer 0 is the singleton {x0}
      ps[p].e = 0.0f;
      ps[p].amb_k = 0;
    }
    for (uint32_t k = 1; k <= a.n; k += L, ++g) {
      if constexpr (RESIDENT) {
        tb = smem + (a.tab_off[k - 1] - a.tab_off[0]);
      } else {
        mbar_wait_u32(full0 + 8u * s, ph);
      }
      exact_layer<K, P, CERT>(ps, act, tb, k, a.joint, a.tables, a.probe_nored == 0, hist1);
      if (L == 2 && k + 1 <= a.n)  // the next table follows this one (header.bytes)
        exact_layer<K, P, CERT>(ps, act, tb + reinterpret_cast<const LayerTable*>(tb)->bytes,
                                k + 1, a.joint, a.tables, a.probe_nored == 0, hist1);
      if constexpr (!RESIDENT) {
        named_barrier_sync(1, kXThreads);  // every thread is done with stage s
        if (tid == 0 && g + S < steps_total) issue(g + S);
        tb += a.buf_bytes;
        if (++s == S) {
          s = 0;
          ph ^= 1u;
          tb = smem;
        }
      }
    }
    if constexpr (CERT) {  // uncertified paths -> the replay list (path start state)
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (act[p] && ps[p].amb_k != 0) {
          const uint64_t v = gid * P + p;
          const uint64_t beg = a.first + v * a.q + (v < a.rem ? v : a.rem);
          AmbEntry ent;
          ent.key = ((beg + r) << 16) | ps[p].amb_k;
          Mrg st0 = ps[p].st;
          mrg_apply(a.back, st0);
          ent.st[0] = st0.a0;
          ent.st[1] = st0.a1;
          ent.st[2] = st0.a2;
          ent.st[3] = st0.b0;
          ent.st[4] = st0.b1;
          ent.st[5] = st0.b2;
          const unsigned long long idx = atomicAdd(a.stats, 1ull);
          if (idx < a.amb_cap) {
            a.amb[idx] = ent;
          } else {  // list full: replay here into the original-index counts
            replay_entry<K>(a, a.ojoint, ent);
            atomicAdd(a.stats + 2, 1ull);
          }
        }
      }
    }
  }
  if (hist1) {  // the CTA's first-transition counts: one RED per visited cell of row 0
    __syncthreads();
    for (uint32_t c = tid; c < a.n1; c += kXThreads)
      if (hist1[c]) red_add_u64(a.joint + c, static_cast<unsigned long long>(hist1[c]));
  }
}

template <int K, bool RES, int P, bool CERT>
static cudaError_t launch_x_t(const PathArgs& a, uint32_t blocks, size_t smem, cudaStream_t st,
                              int* bps) {
  auto fn = a.layers_per_stage == 2 ? k_paths_x<K, RES, P, 2, CERT> : k_paths_x<K, RES, P, 1, CERT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (bps) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, fn, kXThreads, smem) != cudaSuccess ||
        *bps < 1)
      *bps = 1;
    return cudaSuccess;
  }
  fn<<<blocks, kXThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_x_k(bool res, int P, bool cert, const PathArgs& a, uint32_t blocks,
                              size_t smem, cudaStream_t st, int* bps) {
  if (cert) {
    if (P == 1)
      return res ? launch_x_t<K, true, 1, true>(a, blocks, smem, st, bps)
                 : launch_x_t<K, false, 1, true>(a, blocks, smem, st, bps);
    if (P == 4)
      return res ? launch_x_t<K, true, 4, true>(a, blocks, smem, st, bps)
                 : launch_x_t<K, false, 4, true>(a, blocks, smem, st, bps);
    return res ? launch_x_t<K, true, 2, true>(a, blocks, smem, st, bps)
               : launch_x_t<K, false, 2, true>(a, blocks, smem, st, bps);
  }
  if (P == 1)
    return res ? launch_x_t<K, true, 1, false>(a, blocks, smem, st, bps)
               : launch_x_t<K, false, 1, false>(a, blocks, smem, st, bps);
  if (P == 4)
    return res ? launch_x_t<K, true, 4, false>(a, blocks, smem, st, bps)
               : launch_x_t<K, false, 4, false>(a, blocks, smem, st, bps);
  return res ? launch_x_t<K, true, 2, false>(a, blocks, smem, st, bps)
             : launch_x_t<K, false, 2, false>(a, blocks, smem, st, bps);
}

// k_paths_x (kind 0 = Brownian, 2 = OU; MRG32k3a); cert: the certified variant
// (approximate FP64 Box-Muller, uncertified paths to a.amb). bps != nullptr:
// occupancy query only.
cudaError_t launch_paths_x(int kind, bool resident, int P, bool cert, const PathArgs& a,
                           uint32_t blocks, size_t smem, cudaStream_t st, int* bps) {
  return kind == 0 ? launch_x_k<0>(resident, P, cert, a, blocks, smem, st, bps)
                   : launch_x_k<2>(resident, P, cert, a, blocks, smem, st, bps);
}


// The replay list of one k_paths_fast launch, grid-stride.
template <int K>
__global__ void __launch_bounds__(256) k_replay(const __grid_constant__ FastArgs f) {
  const unsigned long long entries = *reinterpret_cast<volatile unsigned long long*>(f.stats);
  const uint64_t n = entries < f.cap ? entries : f.cap;
  const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g0 == 0) atomicAdd(f.stats + 1, static_cast<unsigned long long>(n));
  for (uint64_t g = g0; g < n; g += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    replay_entry<K>(f.p, f.p.joint, f.amb[g]);
}

// The replay list of a certified launch (k_paths_x<CERT> or k_paths_fast), grid-stride.
cudaError_t launch_replay(int kind, const FastArgs& f, uint32_t blocks, cudaStream_t st) {
  if (kind == 0) k_replay<0><<<blocks, 256, 0, st>>>(f);
  else k_replay<2><<<blocks, 256, 0, st>>>(f);
  return cudaGetLastError();
}

// Exhaustive check of the FP32 Box-Muller bounds over all 2^32 - 209 MRG32k3a
// outputs x (both u1 and u2 roles): out[0] = max(|r~ - r| - kRadB r~),
// out[1] = max |c~ - c|, out[2] = max |s~ - s|, out[3] = max(|c~|, |s~|),
// as FP32 bit patterns (non-negative floats order like their bits).
__global__ void __launch_bounds__(256) k_fast_bounds_check(unsigned int* out) {
  float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f;
  for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < kM1;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t x = static_cast<uint32_t>(g);
    const double u = mrg_to_unit(x);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, qt_log_unit(u)));
    const float rt = fast_radius(x);
    const double dr = fabs(static_cast<double>(rt) - r) - static_cast<double>(kRadB) * rt;
    m0 = fmaxf(m0, __double2float_ru(dr));
    double sn, cs;
    qt_sincos_2pi(__dmul_rn(kTwoPi, u), &sn, &cs);
    float c, s;
    fast_angle(x, c, s);
    m1 = fmaxf(m1, __double2float_ru(fabs(static_cast<double>(c) - cs)));
    m2 = fmaxf(m2, __double2float_ru(fabs(static_cast<double>(s) - sn)));
    m3 = fmaxf(m3, fmaxf(fabsf(c), fabsf(s)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
    m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    m3 = fmaxf(m3, __shfl_xor_sync(0xffffffffu, m3, o));
  }
  if ((threadIdx.x & 31u) == 0) {
    atomicMax(out + 0, __float_as_uint(m0));
    atomicMax(out + 1, __float_as_uint(m1));
    atomicMax(out + 2, __float_as_uint(m2));
    atomicMax(out + 3, __float_as_uint(m3));
  }
}

// Exhaustive device check of the Box-Muller transcendentals over an engine's
// whole uniform domain (domain 0: MRG32k3a u = (x + 1)/(m1 + 1), x < m1;
// domain 1: XORWOW u = v 2^-32, v < 2^32): out[0..2] = sum over inputs i of
// mix(i, bits(f(u_i))) mod 2^64 for f = log (u = 0 clamped to 2^-64), sin and
// cos of 2 pi u. tests/tools/check_math.cpp computes the same sums from the
// live glibc (tests/golden/glibc_checksums.json); equal sums = the device's
// log/sincos equal glibc's on every input of the domain.
__device__ __forceinline__ uint64_t mix_checksum(uint64_t i, double v) {
  uint64_t z = static_cast<uint64_t>(__double_as_longlong(v)) + 0x9E3779B97F4A7C15ull * (i + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void __launch_bounds__(256) k_math_checksum(int domain, unsigned long long* out) {
  const uint64_t n = domain == 0 ? kM1 : (1ull << 32);
  uint64_t sl = 0, ss = 0, sc = 0;
  for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < n;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double u = domain == 0 ? mrg_to_unit(static_cast<uint32_t>(g))
                                 : __dmul_rn(static_cast<double>(g), 0x1p-32);
    sl += mix_checksum(g, qt_log_unit(u <= 0.0 ? 0x1p-64 : u));
    double sn, cs;
    qt_sincos_2pi(__dmul_rn(kTwoPi, u), &sn, &cs);
    ss += mix_checksum(g, sn);
    sc += mix_checksum(g, cs);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sl += __shfl_xor_sync(0xffffffffu, sl, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
  }
  if ((threadIdx.x & 31u) == 0) {
    atomicAdd(out + 0, static_cast<unsigned long long>(sl));
    atomicAdd(out + 1, static_cast<unsigned long long>(ss));
    atomicAdd(out + 2, static_cast<unsigned long long>(sc));
  }
}

// ---------------------------------------------------------------------------
// Alg III: grid = (slices, n). Slice s of layer k covers samples
// [M s / S, M (s+1) / S) of that layer; each thread a contiguous sub-run, so
// its stream again flows sample to sample without jumps.
// ---------------------------------------------------------------------------
template <int K, int SRC>
__global__ void __launch_bounds__(kThreads) k_alg3(const Alg3Args a) {
  using C = Chain<K>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t tid = threadIdx.x;
  const uint32_t k = blockIdx.y + 1;  // transition k-1 -> k
  const uint64_t layer0 = static_cast<uint64_t>(k - 1) * a.M;
  // slice of this layer, intersected with the unit window [first, first+count)
  uint64_t lo = layer0 + a.M * blockIdx.x / gridDim.x;
  uint64_t hi = layer0 + a.M * (blockIdx.x + 1) / gridDim.x;
  lo = lo > a.first ? lo : a.first;
  hi = hi < a.first + a.count ? hi : a.first + a.count;
  if (lo >= hi) return;
  const uint64_t len = hi - lo;
  const uint64_t q = len / blockDim.x, rem = len % blockDim.x;
  const uint64_t mycount = q + (tid < rem ? 1u : 0u);
  const uint64_t mybeg = lo + tid * q + (tid < rem ? tid : rem);

  // tables: layer k at buffer 0, layer k-1 (k >= 2) at buffer 1
  const uint8_t* tk = smem;
  const uint8_t* tp = smem + a.buf_bytes;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t bytes = a.tab_bytes[k - 1] + (k >= 2 ? a.tab_bytes[k - 2] : 0u);
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(smem, a.tables + a.tab_off[k - 1], a.tab_bytes[k - 1], &bar);
    if (k >= 2) bulk_g2s(smem + a.buf_bytes, a.tables + a.tab_off[k - 2], a.tab_bytes[k - 2], &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const LayerTable& hk = *reinterpret_cast<const LayerTable*>(tk);
  const LayerTable& hp = *reinterpret_cast<const LayerTable*>(tp);

  Source<SRC> src;
  if (mycount) src.start(a.src, mybeg);
  for (uint64_t r = 0; r < mycount; ++r) {
    if (r > 0) src.next_unit(a.src, mybeg + r);
    double e[C::D + C::NPS], x[C::D], xn[C::D];
#pragma unroll
    for (int q2 = 0; q2 < C::D + C::NPS; ++q2) e[q2] = src.normal();
    C::marginal(hk.marg_prev, k == 1, x, e);  // sample_marginal(k-1, ...)
    C::step(hk.step, x, xn, e + C::D);        // step(k-1, ...)
    const uint32_t i = k == 1 ? 0u : nearest<C::D>(hp, tp, x, a.tables);
    const uint32_t j = nearest<C::D>(hk, tk, xn, a.tables);
    red_add_u64(a.joint + hk.joff + static_cast<uint64_t>(i) * hk.n_pts + j, 1ull);
  }
}

// ---------------------------------------------------------------------------
// k_alg3_x: Alg III for the 1-D chains with MRG32k3a (C3), k_alg3's arithmetic
// bit for bit. A sample consumes exactly one Box-Muller pair (d + nps = 2:
// z1 -> sample_marginal(k-1), z2 -> step), drawn with two interleaved MRG32k3a
// steps; each thread keeps P samples in flight (contiguous sub-runs of its
// slice) so the P dependency chains interleave. Tables k-1 and k stay in
// shared memory for the CTA's lifetime.
// ---------------------------------------------------------------------------
// Exact replay of one uncertified Alg III sample (k_alg3's arithmetic, exact
// tables in global memory) into the original-index counts a.ojoint.
template <int K>
__device__ __noinline__ void replay3_entry(const Alg3Args& a, const AmbEntry& ent) {
  using C = Chain<K>;
  Source<kSrcMrg> src;
  src.s = Mrg{ent.st[0], ent.st[1], ent.st[2], ent.st[3], ent.st[4], ent.st[5]};
  src.has = false;
  const uint32_t k = static_cast<uint32_t>(ent.key & 0xFFFFu);
  const uint8_t* tk = a.tables + __ldg(a.tab_off + k - 1);
  const LayerTable& hk = *reinterpret_cast<const LayerTable*>(tk);
  double e[2], x[1], xn[1];
  e[0] = src.normal();
  e[1] = src.normal();
  C::marginal(hk.marg_prev, k == 1, x, e);
  C::step(hk.step, x, xn, e + 1);
  uint32_t i = 0;
  if (k >= 2) {
    const uint8_t* tp = a.tables + __ldg(a.tab_off + k - 2);
    i = nearest_1d(*reinterpret_cast<const LayerTable*>(tp), tp, x[0], a.tables);
  }
  const uint32_t j = nearest_1d(hk, tk, xn[0], a.tables);
  red_add_u64(a.ojoint + hk.joff + static_cast<uint64_t>(i) * hk.n_pts + j, 1ull);
}

template <int K>
__global__ void __launch_bounds__(256) k_replay3(const __grid_constant__ Alg3Args a) {
  const unsigned long long entries = *reinterpret_cast<volatile unsigned long long*>(a.stats);
  const uint64_t n = entries < a.amb_cap ? entries : a.amb_cap;
  const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g0 == 0) atomicAdd(a.stats + 1, static_cast<unsigned long long>(n));
  for (uint64_t g = g0; g < n; g += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    replay3_entry<K>(a, a.amb[g]);
}

cudaError_t launch_replay3(int kind, const Alg3Args& a, uint32_t blocks, cudaStream_t st) {
  if (kind == 0) k_replay3<0><<<blocks, 256, 0, st>>>(a);
  else k_replay3<2><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// The cell of every state in [x - e, x + e] on an x-table, if there is one
// (the certificate of k_paths_x<CERT>, for a single query).
__device__ __forceinline__ bool cert_cell(const LayerTable& h, const uint8_t* tb, double x, float e,
                                          uint32_t& j) {
  const double ed = static_cast<double>(e);
  const double xl = __dsub_rd(x, ed), xh = __dadd_ru(x, ed);
  const bool safe = __dadd_ru(fabs(x), ed) < static_cast<double>(h.cert_xmax);
  const uint16_t* start = reinterpret_cast<const uint16_t*>(tb + h.off_start);
  const double2* PT = reinterpret_cast<const double2*>(tb + h.off_rec);
  const uint32_t c = start[bucket_of(safe ? xl : 0.0, h.lo, h.inv_w, h.nb_d, h.nb)];
  const double2 r = PT[c];
  const bool in0 = xh < r.x;
  const bool in1 = !(xl < r.x) && xh < r.y;
  j = in0 ? c : c + 1;
  return safe && (in0 || in1);
}

// PRIV: the layer's counts privatised in a shared-memory tile (one CTA = one
// slice of one layer, 1024 threads, one CTA per SM) and flushed once per CTA
// with one RED per non-zero cell; otherwise one L2 RED per sample.
template <int K, int P, bool CERT, bool PRIV>
__global__ void __launch_bounds__(PRIV ? 1024 : kThreads) k_alg3_x(const __grid_constant__ Alg3Args a) {
  using C = Chain<K>;
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
  const uint8_t* tp = smem + a.buf_bytes;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + 2ull * a.buf_bytes);
  if constexpr (PRIV) {
    for (uint32_t c = tid; c < a.priv_bytes / 4; c += blockDim.x) hist[c] = 0u;
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    const uint32_t bytes = a.tab_bytes[k - 1] + (k >= 2 ? a.tab_bytes[k - 2] : 0u);
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(smem, a.xtables + a.tab_off[k - 1], a.tab_bytes[k - 1], &bar);
    if (k >= 2) bulk_g2s(smem + a.buf_bytes, a.xtables + a.tab_off[k - 2], a.tab_bytes[k - 2], &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const LayerTable& hk = *reinterpret_cast<const LayerTable*>(tk);
  const LayerTable& hp = *reinterpret_cast<const LayerTable*>(tp);
  // CERT: the marginal sample x = RN(m z1) is within fm b1 (1 + 2^-50) + cx of the
  // exact one (|z1| <= 6.7 for every MRG32k3a uniform bounds the rounding term)
  const float fm = __double2float_ru(fabs(hk.marg_prev[0]));
  const float cx = __fmul_ru(__fmul_ru(fm, 6.7f), 0x1p-50f);
  // the slice split over blockDim.x * P slots, slot v = tid * P + p
  const uint64_t len = hi - lo, T = static_cast<uint64_t>(blockDim.x) * P;
  const uint64_t q = len / T, rem = len % T;
  Mrg st[P];
  uint64_t cnt[P], beg[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const uint64_t v = static_cast<uint64_t>(tid) * P + p;
    cnt[p] = q + (v < rem ? 1u : 0u);
    beg[p] = lo + v * q + (v < rem ? v : rem);
    st[p] = Mrg{};
    if (cnt[p]) {
      Source<kSrcMrg> src;
      src.start(a.src, beg[p]);
      st[p] = src.s;
    }
  }
  const uint64_t rounds = q + (rem ? 1u : 0u);
  unsigned long long* jl = a.joint + hk.joff;
  const uint32_t npts = hk.n_pts;
  for (uint64_t r = 0; r < rounds; ++r) {
    double z1[P], z2[P], v1[P], v2[P];
    float b[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      uint32_t u1, u2;
      mrg_step2(st[p], u1, u2);
      v1[p] = mrg_to_unit(u1);
      v2[p] = mrg_to_unit(u2);
    }
    if constexpr (CERT) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const double rr = apx::radius(v1[p]);
        double sn, cs;
        apx::sincos(__dmul_rn(kTwoPi, v2[p]), &sn, &cs);
        z1[p] = __dmul_rn(rr, cs);
        z2[p] = __dmul_rn(rr, sn);
        b[p] = __double2float_ru(__dmul_ru(rr, apx::kApxZ));
      }
    } else {
      box_muller_batch<P>(v1, v2, z1, z2);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double e0[1] = {z1[p]}, e1[1] = {z2[p]}, x[1], xn[1];
      C::marginal(hk.marg_prev, k == 1, x, e0);  // sample_marginal(k-1, ...)
      C::step(hk.step, x, xn, e1);               // step(k-1, ...)
      if constexpr (CERT) {
        const float ex = k == 1 ? 0.0f : __fadd_ru(__fmaf_ru(__fmul_ru(fm, b[p]), 0x1p-50f,
                                                             __fmul_ru(fm, b[p])), cx);
        const float lin = __fmaf_ru(hk.fa, ex, __fmul_ru(hk.fs, b[p]));
        const float exn = __fadd_ru(__fmaf_ru(lin, 0x1p-50f, lin), hk.cert_c);
        uint32_t i = 0, j;
        const bool oki = k == 1 || cert_cell(hp, tp, x[0], ex, i);
        const bool okj = cert_cell(hk, tk, xn[0], exn, j);
        if (r < cnt[p]) {
          if (oki && okj) {
            if constexpr (PRIV) atomicAdd(hist + i * npts + j, 1u);
            else if (!a.probe_nored) red_add_u64(jl + static_cast<uint64_t>(i) * npts + j, 1ull);
          } else {  // the sample's start state -> the replay list (or inline when full)
            Mrg s0 = st[p];
            mrg_apply(a.back2, s0);
            AmbEntry ent;
            ent.key = ((beg[p] + r) << 16) | k;
            ent.st[0] = s0.a0;
            ent.st[1] = s0.a1;
            ent.st[2] = s0.a2;
            ent.st[3] = s0.b0;
            ent.st[4] = s0.b1;
            ent.st[5] = s0.b2;
            const unsigned long long idx = atomicAdd(a.stats, 1ull);
            if (idx < a.amb_cap) {
              a.amb[idx] = ent;
            } else {
              replay3_entry<K>(a, ent);
              atomicAdd(a.stats + 2, 1ull);
            }
          }
        }
      } else {
        const uint32_t i = k == 1 ? 0u : nearest_1d_pos(hp, tp, x[0], a.tables);
        const uint32_t j = nearest_1d_pos(hk, tk, xn[0], a.tables);
        if constexpr (PRIV) {
          if (r < cnt[p]) atomicAdd(hist + i * npts + j, 1u);
        } else if (r < cnt[p] && !a.probe_nored) {
          red_add_u64(jl + static_cast<uint64_t>(i) * npts + j, 1ull);
        }
      }
    }
  }
  if constexpr (PRIV) {  // flush the tile: one RED per non-zero cell
    __syncthreads();
    const uint32_t cells = (k == 1 ? 1u : hp.n_pts) * npts;
    for (uint32_t c = tid; c < cells; c += blockDim.x) {
      const uint32_t v = hist[c];
      if (v) red_add_u64(jl + c, static_cast<unsigned long long>(v));
    }
  }
}

// ---------------------------------------------------------------------------
// Grids whose tables exceed the shared-memory staging limit (e.g. 1-D N above
// ~6800): the same exact arithmetic with every table read from global memory
// through L1/L2 -- Alg I/II one path per thread slot, Alg III one sample.
// ---------------------------------------------------------------------------
template <int K, int SRC>
__global__ void __launch_bounds__(256) k_paths_gmem(const __grid_constant__ PathArgs a) {
  using C = Chain<K>;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t mycount = a.q + (gid < a.rem ? 1u : 0u);
  const uint64_t mybeg = a.first + gid * a.q + (gid < a.rem ? gid : a.rem);
  if (!mycount) return;
  Source<SRC> src;
  src.start(a.src, mybeg);
  for (uint64_t r = 0; r < mycount; ++r) {
    if (r > 0) src.next_unit(a.src, mybeg + r);
    double x[C::D];
#pragma unroll
    for (int d = 0; d < C::D; ++d) x[d] = 0.0;
    uint32_t i = 0;
    for (uint32_t k = 1; k <= a.n; ++k) {
      const uint8_t* tb = a.tables + __ldg(a.tab_off + k - 1);
      const LayerTable& h = *reinterpret_cast<const LayerTable*>(tb);
      double e[C::NPS], xn[C::D];
#pragma unroll
      for (int q = 0; q < C::NPS; ++q) e[q] = src.normal();
      C::step(h.step, x, xn, e);
#pragma unroll
      for (int d = 0; d < C::D; ++d) x[d] = xn[d];
      const uint32_t j = nearest<C::D>(h, tb, x, a.tables);
      red_add_u64(a.joint + h.joff + static_cast<uint64_t>(i) * h.n_pts + j, 1ull);
      i = j;
    }
  }
}

template <int K, int SRC>
__global__ void __launch_bounds__(256) k_alg3_gmem(const __grid_constant__ Alg3Args a) {
  using C = Chain<K>;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t q = a.count / T, rem = a.count % T;
  const uint64_t mycount = q + (gid < rem ? 1u : 0u);
  const uint64_t mybeg = a.first + gid * q + (gid < rem ? gid : rem);
  if (!mycount) return;
  Source<SRC> src;
  src.start(a.src, mybeg);
  for (uint64_t r = 0; r < mycount; ++r) {
    if (r > 0) src.next_unit(a.src, mybeg + r);
    const uint64_t unit = mybeg + r;
    const uint32_t k = static_cast<uint32_t>(unit / a.M) + 1;  // layer-major units (k-1) M + m
    const uint8_t* tk = a.tables + __ldg(a.tab_off + k - 1);
    const LayerTable& hk = *reinterpret_cast<const LayerTable*>(tk);
    double e[C::D + C::NPS], x[C::D], xn[C::D];
#pragma unroll
    for (int q2 = 0; q2 < C::D + C::NPS; ++q2) e[q2] = src.normal();
    C::marginal(hk.marg_prev, k == 1, x, e);
    C::step(hk.step, x, xn, e + C::D);
    uint32_t i = 0;
    if (k >= 2) {
      const uint8_t* tp = a.tables + __ldg(a.tab_off + k - 2);
      i = nearest<C::D>(*reinterpret_cast<const LayerTable*>(tp), tp, x, a.tables);
    }
    const uint32_t j = nearest<C::D>(hk, tk, xn, a.tables);
    red_add_u64(a.joint + hk.joff + static_cast<uint64_t>(i) * hk.n_pts + j, 1ull);
  }
}

template <int K>
static cudaError_t launch_gmem_k(bool alg3, int src, const PathArgs& pa, const Alg3Args& aa,
                                 uint32_t blocks, cudaStream_t st) {
#define QT_GMEM(S)                                                           \
  if (alg3) k_alg3_gmem<K, S><<<blocks, 256, 0, st>>>(aa);                  \
  else k_paths_gmem<K, S><<<blocks, 256, 0, st>>>(pa);                      \
  return cudaGetLastError();
  switch (src) {
    case kSrcLcg48: QT_GMEM(kSrcLcg48)
    case kSrcMrg: QT_GMEM(kSrcMrg)
    case kSrcXorwow: QT_GMEM(kSrcXorwow)
    default: QT_GMEM(kSrcNormalsIn)
  }
#undef QT_GMEM
}

cudaError_t launch_gmem(int kind, int src, bool alg3, const PathArgs& pa, const Alg3Args& aa,
                        uint32_t blocks, cudaStream_t st) {
  switch (kind) {
    case 0: return launch_gmem_k<0>(alg3, src, pa, aa, blocks, st);
    case 1: return launch_gmem_k<1>(alg3, src, pa, aa, blocks, st);
    case 2: return launch_gmem_k<2>(alg3, src, pa, aa, blocks, st);
    default: return launch_gmem_k<3>(alg3, src, pa, aa, blocks, st);
  }
}

// ---------------------------------------------------------------------------
// finalize
// ---------------------------------------------------------------------------
// joint[t][orig_t[a] cols + orig_{t+1}[b]] += sjoint[t][a cols + b]  (grid.y = t):
// k_paths_x's sorted-cell counts mapped to the reference's original indices.
// Reads are coalesced; the writes of one row stay inside one row of joint.
__global__ void k_permute_add(const unsigned long long* sjoint, unsigned long long* joint,
                              const FinalizeArgs a, const uint32_t* orig) {
  const uint32_t t = blockIdx.y;
  const uint64_t rows = a.rows[t], cols = a.cols[t], elems = rows * cols;
  const unsigned long long* S = sjoint + a.joff[t];
  unsigned long long* J = joint + a.joff[t];
  const uint32_t* orow = orig + a.voff_row[t];
  const uint32_t* ocol = orig + a.voff_col[t];
  for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < elems;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long v = S[e];
    if (v == 0) continue;
    const uint64_t r = e / cols, c = e - r * cols;
    J[static_cast<uint64_t>(__ldg(orow + r)) * cols + __ldg(ocol + c)] += v;
  }
}

cudaError_t launch_permute_add(const unsigned long long* sjoint, unsigned long long* joint,
                               const uint64_t* fin, const uint32_t* orig, uint32_t n,
                               uint64_t max_elems, cudaStream_t st) {
  FinalizeArgs f{fin, fin + n, fin + 2 * n, fin + 3 * n, fin + 4 * n};
  const uint64_t want = (max_elems + 255) / 256;
  const uint32_t bx = static_cast<uint32_t>(want < 2048 ? (want ? want : 1) : 2048);
  k_permute_add<<<dim3(bx, n), 256, 0, st>>>(sjoint, joint, f, orig);
  return cudaGetLastError();
}

// visits[k][j] = sum_i joint[k-1][i][j]  (grid.y = transition t = k-1)
__global__ void k_colsum(const unsigned long long* joint, unsigned long long* visits,
                         const FinalizeArgs a) {
  const uint32_t t = blockIdx.y;
  const uint64_t rows = a.rows[t], cols = a.cols[t];
  const unsigned long long* J = joint + a.joff[t];
  unsigned long long* V = visits + a.voff_col[t];
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long s = 0;
    for (uint64_t i = 0; i < rows; ++i) s += J[i * cols + j];
    V[j] = s;
  }
}

// visits[t][i] = sum_j joint[t][i][j]: one warp per row  (Alg III sources)
__global__ void k_rowsum(const unsigned long long* joint, unsigned long long* visits,
                         const FinalizeArgs a) {
  const uint32_t t = blockIdx.y;
  const uint64_t rows = a.rows[t], cols = a.cols[t];
  const unsigned long long* J = joint + a.joff[t];
  unsigned long long* V = visits + a.voff_row[t];
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < rows;
       i += warps) {
    unsigned long long s = 0;
    for (uint64_t j = lane; j < cols; j += 32) s += J[i * cols + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) V[i] = s;
  }
}

// pi[t][i][j] = joint / visits[t][i] (0 on unvisited rows), quant_tree.hpp:69-83
__global__ void k_normalize(const unsigned long long* joint, const unsigned long long* visits,
                            double* pi, const FinalizeArgs a) {
  const uint32_t t = blockIdx.y;
  const uint64_t cols = a.cols[t];
  const uint64_t total = a.rows[t] * cols;
  const unsigned long long* J = joint + a.joff[t];
  const unsigned long long* V = visits + a.voff_row[t];
  double* P = pi + a.joff[t];
  for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long den = V[e / cols];
    P[e] = den == 0 ? 0.0 : __ddiv_rn(__ull2double_rn(J[e]), __ull2double_rn(den));
  }
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// ---------------------------------------------------------------------------
// standalone K2 (NnIndex::nearest in batch) and RNG probes
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kThreads) k_nearest(const uint8_t* table, uint32_t bytes,
                                                      const double* queries, uint64_t nq,
                                                      unsigned long long* out, int in_smem) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint8_t* tb = table;
  if (in_smem) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_expect_tx(&bar, bytes);
      bulk_g2s(smem, table, bytes, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    tb = smem;
  }
  const LayerTable& h = *reinterpret_cast<const LayerTable*>(tb);
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < nq;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double x[D];
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = queries[q * D + d];
    out[q] = nearest<D>(h, tb, x, table);
  }
}

template <int SRC>
__global__ void k_path_normals(const SrcArgs a, uint64_t first, uint64_t count, double* out) {
  const uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= count) return;
  Source<SRC> src;
  src.start(a, first + u);
  for (uint32_t e = 0; e < a.per_unit; ++e) out[u * a.per_unit + e] = src.normal();
}

template <int SRC>
__global__ void k_uniforms(const SrcArgs a, uint64_t offset, uint64_t count, double* out) {
  const uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= count) return;
  SrcArgs b = a;
  b.draws = 1;  // position at serial draw offset + u
  Source<SRC> src;
  src.start(b, offset + u);
  out[u] = src.uniform();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int K, int SRC, bool RES>
static cudaError_t launch_paths_t(const PathArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  auto fn = k_paths<K, SRC, RES>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fn<<<grid, kPathThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int K, int SRC>
static cudaError_t launch_paths_r(const PathArgs& a, bool res, dim3 g, size_t smem,
                                  cudaStream_t st) {
  return res ? launch_paths_t<K, SRC, true>(a, g, smem, st)
             : launch_paths_t<K, SRC, false>(a, g, smem, st);
}

template <int K>
static cudaError_t launch_paths_s(const PathArgs& a, int src, bool res, dim3 g, size_t smem,
                                  cudaStream_t st) {
  switch (src) {
    case kSrcLcg48: return launch_paths_r<K, kSrcLcg48>(a, res, g, smem, st);
    case kSrcMrg: return launch_paths_r<K, kSrcMrg>(a, res, g, smem, st);
    case kSrcXorwow: return launch_paths_r<K, kSrcXorwow>(a, res, g, smem, st);
    default: return launch_paths_r<K, kSrcNormalsIn>(a, res, g, smem, st);
  }
}

cudaError_t launch_paths(int kind, int src, bool resident, const PathArgs& a, uint32_t blocks,
                         size_t smem, cudaStream_t st) {
  const dim3 g(blocks);
  switch (kind) {
    case 0: return launch_paths_s<0>(a, src, resident, g, smem, st);
    case 1: return launch_paths_s<1>(a, src, resident, g, smem, st);
    case 2: return launch_paths_s<2>(a, src, resident, g, smem, st);
    default: return launch_paths_s<3>(a, src, resident, g, smem, st);
  }
}

int paths_blocks_per_sm(int kind, int src, bool resident, size_t smem) {
  const void* fn = nullptr;
#define QT_PICK(K, S)                                                                   \
  fn = resident ? reinterpret_cast<const void*>(k_paths<K, S, true>)                   \
                : reinterpret_cast<const void*>(k_paths<K, S, false>)
#define QT_PICK_S(K)                      \
  switch (src) {                          \
    case kSrcLcg48: QT_PICK(K, kSrcLcg48); break; \
    case kSrcMrg: QT_PICK(K, kSrcMrg); break;     \
    case kSrcXorwow: QT_PICK(K, kSrcXorwow); break; \
    default: QT_PICK(K, kSrcNormalsIn); break;    \
  }
  switch (kind) {
    case 0: QT_PICK_S(0); break;
    case 1: QT_PICK_S(1); break;
    case 2: QT_PICK_S(2); break;
    default: QT_PICK_S(3); break;
  }
#undef QT_PICK_S
#undef QT_PICK
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kPathThreads, smem) != cudaSuccess)
    return 1;
  return nb > 0 ? nb : 1;
}

template <int K, bool RES, int P>
static cudaError_t launch_fast_t(const FastArgs& a, dim3 grid, size_t smem, uint32_t rblocks,
                                 cudaStream_t st) {
  auto fn = k_paths_fast<K, RES, P>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fn<<<grid, kFastThreads, smem, st>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_replay<K><<<rblocks, 256, 0, st>>>(a);

  return cudaGetLastError();
}

template <int K, int P>
static const void* fast_fn(bool res) {
  return res ? reinterpret_cast<const void*>(k_paths_fast<K, true, P>)
             : reinterpret_cast<const void*>(k_paths_fast<K, false, P>);
}

template <int K>
static cudaError_t launch_fast_k(bool res, int P, const FastArgs& a, dim3 g, size_t smem,
                                 uint32_t rb, cudaStream_t st) {
  switch (P) {
    case 1: return res ? launch_fast_t<K, true, 1>(a, g, smem, rb, st)
                       : launch_fast_t<K, false, 1>(a, g, smem, rb, st);
    case 4: return res ? launch_fast_t<K, true, 4>(a, g, smem, rb, st)
                       : launch_fast_t<K, false, 4>(a, g, smem, rb, st);
    default: return res ? launch_fast_t<K, true, 2>(a, g, smem, rb, st)
                        : launch_fast_t<K, false, 2>(a, g, smem, rb, st);
  }
}

// k_paths_fast + k_replay (kind 0 = Brownian, 2 = OU); P paths in flight per thread
cudaError_t launch_paths_fast(int kind, bool resident, int P, const FastArgs& a, uint32_t blocks,
                              size_t smem, uint32_t replay_blocks, cudaStream_t st) {
  const dim3 g(blocks);
  return kind == 0 ? launch_fast_k<0>(resident, P, a, g, smem, replay_blocks, st)
                   : launch_fast_k<2>(resident, P, a, g, smem, replay_blocks, st);
}

int paths_fast_blocks_per_sm(int kind, bool resident, int P, size_t smem) {
  const void* fn;
  if (kind == 0) fn = P == 1 ? fast_fn<0, 1>(resident) : P == 4 ? fast_fn<0, 4>(resident) : fast_fn<0, 2>(resident);
  else fn = P == 1 ? fast_fn<2, 1>(resident) : P == 4 ? fast_fn<2, 4>(resident) : fast_fn<2, 2>(resident);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kFastThreads, smem) != cudaSuccess)
    return 1;
  return nb > 0 ? nb : 1;
}

cudaError_t launch_math_checksum(int domain, unsigned long long* out, cudaStream_t st) {
  k_math_checksum<<<148 * 16, 256, 0, st>>>(domain, out);
  return cudaGetLastError();
}

// Exhaustive check of qt_math_fast.h against the glibc-exact pair over all
// 2^32 - 209 MRG32k3a outputs x (as u1 and as u2): out[0] = max |r~ - r| / r,
// out[1] = max |c~ - c|, out[2] = max |s~ - s|, out[3] = max(|c~|, |s~|), as
// the bit patterns of non-negative doubles (which order like their bits).
__global__ void __launch_bounds__(256) k_apx_bounds_check(unsigned long long* out) {
  double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0;
  for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < kM1;
       g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double u = mrg_to_unit(static_cast<uint32_t>(g));
    const double r = __dsqrt_rn(__dmul_rn(-2.0, qt_log_unit(u)));
    const double ra = apx::radius(u);
    if (r > 0.0) m0 = fmax(m0, fabs(ra - r) / r);
    else if (ra != 0.0) m0 = 1.0;  // u = 1: both must give 0
    const double a = __dmul_rn(kTwoPi, u);
    double s, c, sa, ca;
    qt_sincos_2pi(a, &s, &c);
    apx::sincos(a, &sa, &ca);
    m1 = fmax(m1, fabs(ca - c));
    m2 = fmax(m2, fabs(sa - s));
    m3 = fmax(m3, fmax(fabs(ca), fabs(sa)));
  }
  atomicMax(out + 0, static_cast<unsigned long long>(__double_as_longlong(m0)));
  atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(m1)));
  atomicMax(out + 2, static_cast<unsigned long long>(__double_as_longlong(m2)));
  atomicMax(out + 3, static_cast<unsigned long long>(__double_as_longlong(m3)));
}

cudaError_t launch_apx_bounds_check(unsigned long long* out, cudaStream_t st) {
  k_apx_bounds_check<<<148 * 16, 256, 0, st>>>(out);
  return cudaGetLastError();
}

cudaError_t launch_fast_bounds_check(unsigned int* out, cudaStream_t st) {
  k_fast_bounds_check<<<148 * 16, 256, 0, st>>>(out);
  return cudaGetLastError();
}

template <int K, int SRC>
static cudaError_t launch_alg3_t(const Alg3Args& a, dim3 grid, size_t smem, cudaStream_t st) {
  auto fn = k_alg3<K, SRC>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  fn<<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int K>
static cudaError_t launch_alg3_s(const Alg3Args& a, int src, dim3 g, size_t smem,
                                 cudaStream_t st) {
  switch (src) {
    case kSrcLcg48: return launch_alg3_t<K, kSrcLcg48>(a, g, smem, st);
    case kSrcMrg: return launch_alg3_t<K, kSrcMrg>(a, g, smem, st);
    case kSrcXorwow: return launch_alg3_t<K, kSrcXorwow>(a, g, smem, st);
    default: return launch_alg3_t<K, kSrcNormalsIn>(a, g, smem, st);
  }
}

cudaError_t launch_alg3(int kind, int src, const Alg3Args& a, uint32_t slices, size_t smem,
                        cudaStream_t st) {
  const dim3 g(slices, a.n);
  switch (kind) {
    case 0: return launch_alg3_s<0>(a, src, g, smem, st);
    case 1: return launch_alg3_s<1>(a, src, g, smem, st);
    case 2: return launch_alg3_s<2>(a, src, g, smem, st);
    default: return launch_alg3_s<3>(a, src, g, smem, st);
  }
}

// k_alg3_x (kind 0 = Brownian, 2 = OU; MRG32k3a), P samples in flight per thread
cudaError_t launch_alg3_x(int kind, int P, bool cert, const Alg3Args& a, uint32_t slices,
                          size_t smem, cudaStream_t st) {
  const dim3 g(slices, a.n);
  const bool priv = a.priv_bytes != 0;
  auto go = [&](auto fn) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    fn<<<g, priv ? 1024 : kThreads, smem, st>>>(a);
    return cudaGetLastError();
  };
  if (priv) {
    if (cert) return kind == 0 ? go(k_alg3_x<0, 1, true, true>) : go(k_alg3_x<2, 1, true, true>);
    return kind == 0 ? go(k_alg3_x<0, 1, false, true>) : go(k_alg3_x<2, 1, false, true>);
  }
  if (cert) {
    if (kind == 0) return P == 1 ? go(k_alg3_x<0, 1, true, false>) : go(k_alg3_x<0, 2, true, false>);
    return P == 1 ? go(k_alg3_x<2, 1, true, false>) : go(k_alg3_x<2, 2, true, false>);
  }
  if (kind == 0)
    return P == 1 ? go(k_alg3_x<0, 1, false, false>) : P == 4 ? go(k_alg3_x<0, 4, false, false>)
                                                      : go(k_alg3_x<0, 2, false, false>);
  return P == 1 ? go(k_alg3_x<2, 1, false, false>) : P == 4 ? go(k_alg3_x<2, 4, false, false>)
                                                    : go(k_alg3_x<2, 2, false, false>);
}

cudaError_t launch_finalize(bool alg3, const unsigned long long* joint, unsigned long long* visits,
                            double* pi, uint64_t samples, const FinalizeArgs& f, uint32_t n,
                            uint64_t max_cols, uint64_t max_rows, uint64_t max_elems,
                            cudaStream_t st, int* launches) {
  int l = 0;
  const uint32_t bx_cols = static_cast<uint32_t>((max_cols + 255) / 256);
  if (!alg3) {
    // visits[0][0] = M, visits[k] = column sums of joint[k-1]
    k_set_u64<<<1, 1, 0, st>>>(visits, samples);
    ++l;
    k_colsum<<<dim3(bx_cols, n), 256, 0, st>>>(joint, visits, f);
    ++l;
  } else {
    // visits[k-1] = row sums of joint[k-1] (sources), visits[n] = col sums of joint[n-1]
    const uint32_t bx_rows = static_cast<uint32_t>((max_rows * 32 + 255) / 256);
    k_rowsum<<<dim3(bx_rows < 4096 ? bx_rows : 4096, n), 256, 0, st>>>(joint, visits, f);
    ++l;
    FinalizeArgs last = f;
    last.rows += n - 1;
    last.cols += n - 1;
    last.joff += n - 1;
    last.voff_col += n - 1;
    k_colsum<<<dim3(bx_cols, 1), 256, 0, st>>>(joint, visits, last);
    ++l;
  }
  const uint64_t want = (max_elems + 255) / 256;
  const uint32_t bx = static_cast<uint32_t>(want < 2048 ? want : 2048);
  k_normalize<<<dim3(bx, n), 256, 0, st>>>(joint, visits, pi, f);
  ++l;
  if (launches) *launches += l;
  return cudaGetLastError();
}

cudaError_t launch_nearest(int dim, const uint8_t* table, uint32_t bytes, const double* q,
                           uint64_t nq, unsigned long long* out, cudaStream_t st) {
  const bool in_smem = bytes <= 200u * 1024u;
  const size_t smem = in_smem ? bytes : 0;
  uint64_t want = (nq + kThreads - 1) / kThreads;
  const uint32_t blocks = static_cast<uint32_t>(want < 148u * 16u ? (want ? want : 1) : 148u * 16u);
  cudaError_t e;
  switch (dim) {
    case 1:
      cudaFuncSetAttribute(k_nearest<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_nearest<1><<<blocks, kThreads, smem, st>>>(table, bytes, q, nq, out, in_smem);
      break;
    case 2:
      cudaFuncSetAttribute(k_nearest<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_nearest<2><<<blocks, kThreads, smem, st>>>(table, bytes, q, nq, out, in_smem);
      break;
    default:
      cudaFuncSetAttribute(k_nearest<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_nearest<3><<<blocks, kThreads, smem, st>>>(table, bytes, q, nq, out, in_smem);
  }
  e = cudaGetLastError();
  return e;
}

cudaError_t launch_path_normals(int src, const SrcArgs& a, uint64_t first, uint64_t count,
                                double* out, cudaStream_t st) {
  const uint32_t blocks = static_cast<uint32_t>((count + 127) / 128);
  switch (src) {
    case kSrcLcg48: k_path_normals<kSrcLcg48><<<blocks, 128, 0, st>>>(a, first, count, out); break;
    case kSrcMrg: k_path_normals<kSrcMrg><<<blocks, 128, 0, st>>>(a, first, count, out); break;
    default: k_path_normals<kSrcXorwow><<<blocks, 128, 0, st>>>(a, first, count, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_uniforms(int src, const SrcArgs& a, uint64_t offset, uint64_t count,
                            double* out, cudaStream_t st) {
  const uint32_t blocks = static_cast<uint32_t>((count + 127) / 128);
  if (src == kSrcLcg48)
    k_uniforms<kSrcLcg48><<<blocks, 128, 0, st>>>(a, offset, count, out);
  else
    k_uniforms<kSrcMrg><<<blocks, 128, 0, st>>>(a, offset, count, out);
  return cudaGetLastError();
}

}  // namespace qt
