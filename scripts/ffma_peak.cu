// FP32 FFMA throughput on the whole chip: register-operand FFMA (3 registers) and the
// immediate form, 16 independent accumulator chains per thread.  Reports TFLOP/s (2 FLOP/FFMA)
// and FFMA/clk/SM at the measured SM clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int IMM>
__global__ void __launch_bounds__(256) k(float* out, int iters, float s0, float s1) {
  float a[16], b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 1e-7f + i; b[i] = s0 + i * 1e-3f; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (IMM) a[i] = fmaf(a[i], 0.999f, 0.0001f);
      else a[i] = fmaf(a[i], b[i], s1);   // three register operands
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (IMM) a[i] = fmaf(a[i], 1.0001f, -0.0001f);
      else a[i] = fmaf(a[i], b[(i + 1) & 15], a[(i + 8) & 15]);
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc += a[i];
  if (acc == 1234.5f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}
int main() {
  float* d;
  cudaMalloc(&d, 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int imm = 0; imm < 2; ++imm)
    for (int bps : {4, 8}) {
      const int iters = 20000, grid = sms * bps;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      if (imm) k<1><<<grid, 256>>>(d, 100, 1.0f, 0.5f); else k<0><<<grid, 256>>>(d, 100, 1.0f, 0.5f);
      cudaEventRecord(e0);
      if (imm) k<1><<<grid, 256>>>(d, iters, 1.0f, 0.5f); else k<0><<<grid, 256>>>(d, iters, 1.0f, 0.5f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      float cyc; cudaMemcpy(&cyc, d + 1, 4, cudaMemcpyDeviceToHost);
      double ffma = (double)grid * 256 * iters * 32;
      double clk = cyc / (ms * 1e-3);   // SM cycles per second seen by block 0
      printf("%s FFMA, %d blocks/SM: %.1f TFLOP/s, %.1f FFMA/clk/SM at %.0f MHz\n", imm ? "immediate" : "3-register", bps,
             2 * ffma / (ms * 1e-3) / 1e12, ffma / (ms * 1e-3) / clk / sms, clk / 1e6);
    }
}
