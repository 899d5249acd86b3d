// qt_lloyd.cu -- grid construction on the GPU: the
// randomized Lloyd fixed point of lloyd.hpp:59-107 (lloyd_build with the
// GaussianSampler, as build_brownian_grids / build_two_factor_grids call it,
// pipeline.hpp:27-77).
//
// Per iteration: the batch's normals come from the serial MRG32k3a stream
// (k_serial_normals, each thread jumping to a 64-pair chunk), every sample is
// projected with the exact K2 kernel (k_nearest), and the recentering keeps
// the reference's arithmetic order exactly: samples are stably radix-sorted
// by cell, so each cell's coordinate sums are accumulated by one thread in
// sample order from 0.0 (lloyd.hpp:90-96), then divided by the count. With
// the same normals (parity mode) the grid is therefore bit-identical to the
// reference's; with the in-kernel stream the normals are the device
// Box-Muller's (<= 1 ulp from glibc).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/cub.cuh>

#include "qt_device.cuh"
#include "qt_internal.h"

namespace qt {

constexpr uint32_t kPairsPerThread = 64;

// normals [first, first + count) of the serial stream (normal j = pair j/2:
// even j -> r cos, odd j -> r sin, stream.hpp:57-62,97-108), sample-major
__global__ void k_serial_normals(const SrcArgs a, uint64_t first, uint64_t count, double* out) {
  const uint64_t base = first & ~1ull;
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t n0 = base + t * 2 * kPairsPerThread;
  if (n0 >= first + count) return;
  Source<kSrcMrg> src;
  src.start(a, n0);  // a.draws == 1: uniform index == normal index at pair boundaries
  for (uint32_t q = 0; q < kPairsPerThread; ++q) {
    const uint64_t j = n0 + 2 * q;
    if (j >= first + count) break;
    const double u1 = src.uniform();
    const double u2 = src.uniform();
    double z1, z2;
    box_muller(u1, u2, z1, z2);
    if (j >= first) out[j - first] = z1;
    if (j + 1 >= first && j + 1 < first + count) out[j + 1 - first] = z2;
  }
}

// squared_distance (grid.hpp:65-72) of each sample to its center, plus the
// u32 keys / sample indices for the stable sort and the cell counts
__global__ void k_lloyd_prep(const double* X, const double* centers, const unsigned long long* cell,
                             uint64_t M, int d, double* d2, uint32_t* key, uint32_t* idx,
                             uint32_t* counts) {
  for (uint64_t m = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; m < M;
       m += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(cell[m]);
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
      const double t = __dsub_rn(X[m * d + j], centers[static_cast<uint64_t>(c) * d + j]);
      s = __dadd_rn(s, __dmul_rn(t, t));
    }
    d2[m] = s;
    key[m] = c;
    idx[m] = static_cast<uint32_t>(m);
    atomicAdd(counts + c, 1u);
  }
}

// non-empty cell i: center = (sum of its samples in sample order, from 0.0) / count
__global__ void k_lloyd_centers(const double* X, const uint32_t* sorted_idx, const uint32_t* offs,
                                const uint32_t* counts, uint64_t N, int d, double* centers) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const uint32_t n = counts[i];
  if (n == 0) return;  // empty cells keep their point (lloyd.hpp:99-103)
  const uint32_t o = offs[i];
  for (int j = 0; j < d; ++j) {
    double s = 0.0;
    for (uint32_t r = 0; r < n; ++r)
      s = __dadd_rn(s, X[static_cast<uint64_t>(sorted_idx[o + r]) * d + j]);
    centers[i * d + j] = __ddiv_rn(s, static_cast<double>(n));
  }
}

cudaError_t launch_serial_normals(const SrcArgs& a, uint64_t first, uint64_t count, double* out,
                                  cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const uint64_t pairs = (first + count - (first & ~1ull) + 1) / 2;
  const uint64_t threads = (pairs + kPairsPerThread - 1) / kPairsPerThread;
  k_serial_normals<<<static_cast<uint32_t>((threads + 127) / 128), 128, 0, st>>>(a, first, count, out);
  return cudaGetLastError();
}

// One recentering pass given the cells of M samples (see the file header).
// Scratch: d2[M], key/idx/key2/idx2[M], counts/offs[N], tmp (cub) of tmp_bytes.
cudaError_t launch_lloyd_update(const double* X, const unsigned long long* cell, uint64_t M,
                                uint64_t N, int d, double* centers, double* d2, uint32_t* key,
                                uint32_t* idx, uint32_t* key2, uint32_t* idx2, uint32_t* counts,
                                uint32_t* offs, void* tmp, size_t tmp_bytes, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(counts, 0, N * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((M + 255) / 256, 148 * 16));
  k_lloyd_prep<<<blocks ? blocks : 1, 256, 0, st>>>(X, centers, cell, M, d, d2, key, idx, counts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int bits = 1;
  while ((1ull << bits) < N) ++bits;
  size_t need = tmp_bytes;
  e = cub::DeviceRadixSort::SortPairs(tmp, need, key, key2, idx, idx2, static_cast<int>(M), 0, bits, st);
  if (e != cudaSuccess) return e;
  need = tmp_bytes;
  e = cub::DeviceScan::ExclusiveSum(tmp, need, counts, offs, static_cast<int>(N), st);
  if (e != cudaSuccess) return e;
  k_lloyd_centers<<<static_cast<uint32_t>((N + 127) / 128), 128, 0, st>>>(X, idx2, offs, counts, N,
                                                                          d, centers);
  return cudaGetLastError();
}

size_t lloyd_tmp_bytes(uint64_t M, uint64_t N) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int>(M));
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), static_cast<int>(N));
  return std::max(a, b);
}

}  // namespace qt
