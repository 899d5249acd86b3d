// RED throughput probe: every thread issues `per` no-return 64-bit (or 32-bit)
// atomic adds to pseudo-random addresses inside a region of `bytes`, optionally
// confined to a band (consecutive hits within `band` elements of a moving
// diagonal, like the sorted-cell counts of a 1-D chain). Prints REDs/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_probe tools/red_probe.cu
//   tools/red_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <bool W64>
__global__ void k_red(void* base, uint64_t elems, uint64_t band, int per, uint32_t seed, int inter) {
  uint32_t s = seed ^ (blockIdx.x * 1024u + threadIdx.x) * 2654435761u;
  uint64_t row = 0;
  const uint64_t rows = band ? elems / 512 : 0;
  for (int r = 0; r < per; ++r) {
    s = s * 1664525u + 1013904223u;
    uint64_t e;
    if (band) {  // 512-wide rows, hit within +-band/2 of the diagonal
      row = (s >> 8) % rows;
      const uint64_t col = ((row * 512) / rows + ((s >> 3) % band)) % 512;
      e = row * 512 + col;
      if (inter) {  // rows 64 apart share a sector: (i, j) -> ((i & 63) * 512 + j) * 8 + (i >> 6)
        const uint64_t blk = row / 512, i = row % 512;
        e = blk * 512 * 512 + (((i & 63) * 512 + col) << 3) + (i >> 6);
      }
    } else {
      e = ((uint64_t)s * 2654435761ull + r) % elems;
    }
    if (W64)
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"((unsigned long long*)base + e));
    else
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"((unsigned int*)base + e));
  }
}

int main() {
  void* d;
  const size_t maxb = 256ull << 20;
  cudaMalloc(&d, maxb);
  cudaMemset(d, 0, maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int per = 256;
  const int blocks = 148 * 8, threads = 256;
  const double reds = (double)per * blocks * threads;
  for (int w64 = 1; w64 >= 0; --w64)
    for (size_t mb : {8, 16, 32, 49, 64, 98})
      for (int mode : {0, 1, 2}) {
        const uint64_t band = mode ? 64 : 0;
        const int inter = mode == 2;
        const uint64_t elems = (mb << 20) / (w64 ? 8 : 4);
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(a);
          if (w64) k_red<true><<<blocks, threads>>>(d, elems, band, per, 7 + it, inter);
          else k_red<false><<<blocks, threads>>>(d, elems, band, per, 7 + it, inter);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (it) printf("u%d region %4zu MB band %3llu inter %d: %.3g REDs/s (%.2f ms)\n",
                         w64 ? 64 : 32, mb, (unsigned long long)band, inter, reds / (ms * 1e-3), ms);
        }
      }
  return 0;
}
