// qt_bench.cu -- the reference's micro-benchmarks on the GPU:
//   k_pi    Monte Carlo pi with partitioned streams (monte_carlo.hpp:39-77,
//           `qtree bench-rng`): the inside-count of the quarter disk is an
//           integer sum, so the estimate equals the reference's exactly for
//           any launch shape (the uniforms are bit-exact).
//   bench-nn (`qtree bench-nn`, qtree_main.cpp:162-191) reuses
//           k_serial_normals + the exact projection kernels (qt_capi.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include "qt_device.cuh"
#include "qt_internal.h"

namespace qt {

constexpr uint32_t kPiPairs = 1024;  // points per thread

__device__ __forceinline__ void add_inside(unsigned long long* out, uint64_t c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31u) == 0 && c) atomicAdd(out, static_cast<unsigned long long>(c));
}

// Block partition of a jumpable engine: stream i = serial draws
// [i per_stream, (i+1) per_stream), per_stream even, so the union is the
// serial pairs (2p, 2p+1), p < samples / 2.
template <int SRC>
__global__ void k_pi_block(const SrcArgs a, uint64_t points, unsigned long long* inside) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t p0 = t * kPiPairs;
  uint64_t c = 0;
  if (p0 < points) {
    Source<SRC> src;
    src.start(a, 2 * p0);  // draws == 1: position at serial draw 2 p0
    const uint64_t n = points - p0 < kPiPairs ? points - p0 : kPiPairs;
    for (uint64_t q = 0; q < n; ++q) {
      const double u = src.uniform(), v = src.uniform();
      c += __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)) <= 1.0;
    }
  }
  add_inside(inside, c);
}

// Block partition with XORWOW: stream i independently seeded (seed, i) with a
// 64-step burn-in (stream.hpp:146-153); one thread per stream.
__global__ void k_pi_xorwow(const SrcArgs a, uint64_t streams, uint64_t per_stream_points,
                            unsigned long long* inside) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t c = 0;
  if (i < streams) {
    Source<kSrcXorwow> src;
    src.start(a, i);
    for (uint64_t q = 0; q < per_stream_points; ++q) {
      const double u = src.uniform(), v = src.uniform();
      c += __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)) <= 1.0;
    }
  }
  add_inside(inside, c);
}

// Skip-ahead partition (stream i of s emits serial draws i, i+s, ...): stream
// i's k-th point is (serial[2ks + i], serial[2ks + s + i]). Thread = (k, run of
// kPiPairs consecutive i), walking the two serial positions in lockstep.
template <int SRC>
__global__ void k_pi_skip(const SrcArgs a, uint64_t s, uint64_t super_blocks,
                          unsigned long long* inside) {
  const uint64_t runs = (s + kPiPairs - 1) / kPiPairs;
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t c = 0;
  if (t < super_blocks * runs) {
    const uint64_t k = t / runs, i0 = (t % runs) * kPiPairs;
    const uint64_t n = s - i0 < kPiPairs ? s - i0 : kPiPairs;
    Source<SRC> A, B;
    A.start(a, 2 * k * s + i0);
    B.start(a, 2 * k * s + s + i0);
    for (uint64_t q = 0; q < n; ++q) {
      const double u = A.uniform(), v = B.uniform();
      c += __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)) <= 1.0;
    }
  }
  add_inside(inside, c);
}

cudaError_t launch_pi(int engine, int skip, const SrcArgs& a, uint64_t samples, uint64_t streams,
                      unsigned long long* inside, cudaStream_t st) {
  const uint64_t points = samples / 2;
  if (engine == kSrcXorwow) {
    const uint64_t per = points / streams;
    k_pi_xorwow<<<static_cast<uint32_t>((streams + 127) / 128), 128, 0, st>>>(a, streams, per, inside);
  } else if (!skip || streams == 1) {
    const uint64_t threads = (points + kPiPairs - 1) / kPiPairs;
    const uint32_t b = static_cast<uint32_t>((threads + 127) / 128);
    if (engine == kSrcMrg) k_pi_block<kSrcMrg><<<b, 128, 0, st>>>(a, points, inside);
    else k_pi_block<kSrcLcg48><<<b, 128, 0, st>>>(a, points, inside);
  } else {
    const uint64_t super_blocks = samples / (2 * streams);
    const uint64_t threads = super_blocks * ((streams + kPiPairs - 1) / kPiPairs);
    const uint32_t b = static_cast<uint32_t>((threads + 127) / 128);
    if (engine == kSrcMrg) k_pi_skip<kSrcMrg><<<b, 128, 0, st>>>(a, streams, super_blocks, inside);
    else k_pi_skip<kSrcLcg48><<<b, 128, 0, st>>>(a, streams, super_blocks, inside);
  }
  return cudaGetLastError();
}

__global__ void k_sum_u64(const unsigned long long* v, uint64_t n, unsigned long long* out) {
  uint64_t c = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    c += v[i];
  add_inside(out, c);
}

cudaError_t launch_sum_u64(const unsigned long long* v, uint64_t n, unsigned long long* out,
                           cudaStream_t st) {
  k_sum_u64<<<148 * 8, 256, 0, st>>>(v, n, out);
  return cudaGetLastError();
}

}  // namespace qt
