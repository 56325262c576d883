// Microbenchmark: latency of a TMA bulk load (4 x 16 KB, global -> shared) on every SM,
// alone and right after the SM issued a 128 KB fp32 red.global.add flush (or plain stores).
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

__global__ void __launch_bounds__(512, 1) k(const uint8_t* src, float* dst, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  __syncthreads();
  float* base = dst + (size_t)(blockIdx.x % 16) * 32768;
  long long acc = 0;
  uint32_t ph = 0;
  for (int it = 0; it < 8; ++it) {
    if (mode == 1)
      for (int q = 0; q < 16; ++q) {
        float* p = base + (size_t)(tid >> 5) * 2048 + (tid & 31) * 64 + 4 * q;   // row-contig (kernel pattern)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    if (mode == 2)
      for (int q = 0; q < 16; ++q) {
        float* p = base + (size_t)(q * 512 + tid) * 4;
        asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    if (mode == 3)
      for (int q = 0; q < 16; ++q) {
        float* p = base + (size_t)(q * 512 + tid) * 4;   // coalesced red
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    __syncthreads();
    if (tid == 0) {
      long long t0 = clock64();
      mbar_arrive_expect_tx(&bar, 65536);
      for (int s = 0; s < 4; ++s) bulk_copy_g2s(smem_u32(smem) + s * 16384, src + (size_t)(it & 1) * 65536 + s * 16384, 16384, &bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      acc += clock64() - t0;
    }
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = acc / 8;
}

int main() {
  uint8_t* src; float* dst; long long* out;
  cudaMalloc(&src, 1 << 20); cudaMalloc(&dst, 16 * 32768 * 4 * 4); cudaMalloc(&out, 148 * 8);
  cudaMemset(src, 0, 1 << 20); cudaMemset(dst, 0, 16 * 32768 * 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const char* names[] = {"load alone", "after 128KB red row-contig", "after 128KB st coalesced", "after 128KB red coalesced"};
  for (int g : {148, 1})
    for (int m = 0; m < 4; ++m) {
      k<<<g, 512, 65536>>>(src, dst, m, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, g * 8, cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      for (int i = 0; i < g; ++i) { sum += h[i]; mx = h[i] > mx ? h[i] : mx; }
      printf("grid %3d %-28s: 64 KB bulk load latency mean %lld max %lld cycles (%s)\n", g, names[m], sum / g, mx, cudaGetErrorString(e));
    }
  return 0;
}
