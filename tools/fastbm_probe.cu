// fastbm_probe.cu -- exploration tool: error structure of FP32 (MUFU) Box-Muller
// radius / angle against the exact FP64 device Box-Muller, over ALL 2^32 MRG32k3a
// outputs. Not part of the product; the bounds it suggests are re-verified by
// qt_fast_bounds_check() in the library.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1101_3228_b200/csrc -o tools/fastbm_probe tools/fastbm_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "qt_device.cuh"

using namespace qt;

__device__ __forceinline__ float lg2a(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sina(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cosa(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrta(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpa(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float kNeg2Ln2 = -1.3862943611198906f;
// -2 ln2 * (log2(2^32) - log2(m1 + 1)) = -2 ln2 * 6.9867e-8... folded as +c0
constexpr float kC0 = -9.6853e-8f;

__device__ __forceinline__ float fast_R(uint32_t x1, int mode) {
  const uint32_t v = kM1 - x1;  // (0, m1]
  const float uf = __fmul_rn(__uint2float_rn(x1 + 1u), 0x1p-32f);
  const float wf = __fmul_rn(__uint2float_rn(v), 0x1p-32f);
  const bool A = x1 < 2147483544u;  // u < 1/2
  const float t = __fsub_rn(1.0f, wf);
  const float L = lg2a(A ? uf : t);
  const float RA = __fmaf_rn(L, kNeg2Ln2, kC0);
  const float om = __fsub_rn(1.0f, t);  // exact
  float RB;
  if (mode == 0) {
    RB = __fmul_rn(__fmul_rn(L, kNeg2Ln2), __fmul_rn(wf, rcpa(om)));
  } else {
    RB = __fmul_rn(L, kNeg2Ln2);
  }
  // -2 ln(1 - w) = 2 w (1 + w/2 + w^2/3 + ... + w^6/7), w <= 1/8
  float P = __fmaf_rn(wf, 0.14285714285714285f, 0.16666666666666666f);
  P = __fmaf_rn(wf, P, 0.2f);
  P = __fmaf_rn(wf, P, 0.25f);
  P = __fmaf_rn(wf, P, 0.3333333333333333f);
  P = __fmaf_rn(wf, P, 0.5f);
  P = __fmaf_rn(wf, P, 1.0f);
  const float RS = __fmul_rn(__fmul_rn(2.0f, wf), P);
  return A ? RA : (wf <= 0.125f ? RS : RB);
}

__device__ unsigned int g_rbin[64];   // max abs err of r per floor(log2 r~) + 40
__device__ unsigned int g_rrel[64];   // max err / r~ per bin
__device__ unsigned int g_cmax, g_smax, g_count_bad;
__device__ unsigned int g_cbin[16], g_sbin[16];
__device__ unsigned int g_alpha[8];  // max(err - beta_i r~) for beta_i = i * 0.5e-7

__device__ __forceinline__ void amax(unsigned int* p, float v) {
  atomicMax(p, __float_as_uint(v));
}

__global__ void k_probe(int mode, uint32_t start, uint32_t count) {
  __shared__ unsigned int srb[64], srr[64], scb[16], ssb[16];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) srb[i] = srr[i] = 0;
  for (int i = threadIdx.x; i < 16; i += blockDim.x) scb[i] = ssb[i] = 0;
  __syncthreads();
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < count;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = start + (uint32_t)g;
    if (x >= kM1) continue;
    // radius
    const double u = mrg_to_unit(x);
    const double r = __dsqrt_rn(__dmul_rn(-2.0, qt_log_unit(u)));
    const float rt = sqrta(fast_R(x, mode));
    const float er = (float)fabs((double)rt - r);
    int b = (rt > 0.f) ? (int)floorf(log2f(rt)) + 40 : 0;
    b = b < 0 ? 0 : (b > 63 ? 63 : b);
    atomicMax(&srb[b], __float_as_uint(er));
    if (rt > 0.f) atomicMax(&srr[b], __float_as_uint(er / rt));
    for (int i = 0; i < 8; ++i) {
      const float al = er - (float)i * 0.5e-7f * rt;
      if (al > 0.f) atomicMax(&g_alpha[i], __float_as_uint(al));
    }
    // angle
    const double a = __dmul_rn(kTwoPi, u);
    double s, c;
    qt_sincos_2pi(a, &s, &c);
    const int d = (int)(x + 1u - 2147483544u);
    const float ap = __fmul_rn(__int2float_rn(d), 1.4629180792671596e-09f);  // 2 pi / (m1+1)
    const float ct = -cosa(ap), st = -sina(ap);
    const int ab = min(15, (int)(fabsf(ap) * 4.0f));
    atomicMax(&scb[ab], __float_as_uint((float)fabs((double)ct - c)));
    atomicMax(&ssb[ab], __float_as_uint((float)fabs((double)st - s)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    if (srb[i]) atomicMax(&g_rbin[i], srb[i]);
    if (srr[i]) atomicMax(&g_rrel[i], srr[i]);
  }
  for (int i = threadIdx.x; i < 16; i += blockDim.x) {
    if (scb[i]) atomicMax(&g_cbin[i], scb[i]);
    if (ssb[i]) atomicMax(&g_sbin[i], ssb[i]);
  }
}

int main(int argc, char** argv) {
  for (int mode = 0; mode < 2; ++mode) {
    unsigned int z[64] = {0};
    cudaMemcpyToSymbol(g_rbin, z, sizeof z);
    cudaMemcpyToSymbol(g_rrel, z, sizeof z);
    cudaMemcpyToSymbol(g_cbin, z, 64);
    cudaMemcpyToSymbol(g_sbin, z, 64);
    cudaMemcpyToSymbol(g_alpha, z, 32);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_probe<<<148 * 8, 256>>>(mode, 0u, 0xFFFFFFFFu);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d: %s, %.1f ms\n", mode, cudaGetErrorString(cudaGetLastError()), ms);
    unsigned int rb[64], rr[64], cb[16], sb[16];
    cudaMemcpyFromSymbol(rb, g_rbin, sizeof rb);
    cudaMemcpyFromSymbol(rr, g_rrel, sizeof rr);
    cudaMemcpyFromSymbol(cb, g_cbin, sizeof cb);
    cudaMemcpyFromSymbol(sb, g_sbin, sizeof sb);
    for (int i = 0; i < 64; ++i)
      if (rb[i]) {
        float a, b;
        memcpy(&a, &rb[i], 4);
        memcpy(&b, &rr[i], 4);
        printf("  r~ in [2^%d, 2^%d): max abs err %.3e  max rel %.3e\n", i - 40, i - 39, a, b);
      }
    unsigned int al[8];
    cudaMemcpyFromSymbol(al, g_alpha, sizeof al);
    for (int i = 0; i < 8; ++i) {
      float a;
      memcpy(&a, &al[i], 4);
      printf("  beta %.2e -> alpha %.3e\n", i * 0.5e-7, a);
    }
    for (int i = 0; i < 16; ++i)
      if (cb[i]) {
        float a, b;
        memcpy(&a, &cb[i], 4);
        memcpy(&b, &sb[i], 4);
        printf("  |a'| in [%.2f,%.2f): cos err %.3e  sin err %.3e\n", i / 4.0, (i + 1) / 4.0, a, b);
      }
  }
  return 0;
}
