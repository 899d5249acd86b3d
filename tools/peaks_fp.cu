// peaks_fp.cu -- non-tensor FP64 / FP32 / INT issue peaks of this B200, the
// roofline denominators MEASURED_PEAKS.json does not carry.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks_fp tools/peaks_fp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void k_fma(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
    x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_imad(unsigned* out, int iters, unsigned a, unsigned b) {
  unsigned x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
           x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <class F>
double time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  const double ops = 2.0 * blocks * threads * (double)iters * 16 * 8;  // 2 flop per FMA
  void* out;
  cudaMalloc(&out, blocks * threads * 8);
  double t64 = time_ms([&] { k_fma<double><<<blocks, threads>>>((double*)out, iters, 0.999, 1e-3); });
  double t32 = time_ms([&] { k_fma<float><<<blocks, threads>>>((float*)out, iters, 0.999f, 1e-3f); });
  double ti = time_ms([&] { k_imad<<<blocks, threads>>>((unsigned*)out, iters, 1664525u, 1013904223u); });
  printf("{\"fp64_tflops\": %.3f, \"fp32_tflops\": %.3f, \"int32_tops\": %.3f, \"sms\": %d, "
         "\"how\": \"dependent FMA chains x8 per thread, %d blocks x %d threads, best of 5\"}\n",
         ops / t64 / 1e9, ops / t32 / 1e9, ops / ti / 1e9, sms, blocks, threads);
  return 0;
}
