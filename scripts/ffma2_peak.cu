// FP32 paired-FMA (FFMA2, fma.rn.f32x2) throughput on the whole chip vs scalar FFMA:
// 16 independent float2 accumulator chains per thread, three register operands, and the
// broadcast form (a scalar times a float2, the register-tile GEMM pattern).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return d;
}
template <int BCAST>
__global__ void __launch_bounds__(256) k(float* out, int iters, float s0, float s1) {
  float2 a[16], b[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = make_float2(threadIdx.x * 1e-7f + i, i * 1e-3f);
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = make_float2(s0 + i * 1e-3f, s1 - i * 1e-3f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (BCAST) {
        const float x = b[i & 7].x;
        a[i] = ffma2(make_float2(x, x), b[(i + 1) & 7], a[i]);
      } else {
        a[i] = ffma2(a[i], b[i & 7], b[(i + 3) & 7]);
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc += a[i].x + a[i].y;
  if (acc == 1234.5f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}
int main() {
  float* d;
  cudaMalloc(&d, 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bc = 0; bc < 2; ++bc)
    for (int bps : {4, 8}) {
      const int iters = 20000, grid = sms * bps;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      if (bc) k<1><<<grid, 256>>>(d, 100, 1.0f, 0.5f); else k<0><<<grid, 256>>>(d, 100, 1.0f, 0.5f);
      cudaEventRecord(e0);
      if (bc) k<1><<<grid, 256>>>(d, iters, 1.0f, 0.5f); else k<0><<<grid, 256>>>(d, iters, 1.0f, 0.5f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      float cyc; cudaMemcpy(&cyc, d + 1, 4, cudaMemcpyDeviceToHost);
      double fma = (double)grid * 256 * iters * 16 * 2;   // scalar FMAs
      double clk = cyc / (ms * 1e-3);
      printf("%s FFMA2, %d blocks/SM: %.1f TFLOP/s, %.1f FMA/clk/SM at %.0f MHz\n", bc ? "broadcast" : "3-register", bps,
             2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / clk / sms, clk / 1e6);
    }
}
