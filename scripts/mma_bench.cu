// Microbenchmark: latency/throughput of back-to-back tcgen05.mma (bf16, SS operands,
// no-swizzle core-matrix layout) for different N, operand majors and accumulator chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2210_14907_b200/csrc mma_bench.cu -o mma_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

using namespace nbm::tc;

__global__ void bench(long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3F803F80u;
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (tid < 32) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase, sb = smem_u32(smem);
  uint32_t phase = 0;
  if (tid == 0) {
    // mode: 0 = 8 x N128 same D (K-major A, K-major B)
    //       1 = 16 x N64 alternating two D
    //       2 = 8 x N256 same D
    //       3 = 8 x N128 same D, A MN-major, B MN-major
    //       4 = 16 x N128 two GEMMs interleaved (different D)
    //       5 = 8 x N16 same D (MN, MN)
    //       6 = 8 x N128 same D K-major, repeated x4 (32 instr) same D
    long long t0 = clock64();
    for (int rep = 0; rep < 16; ++rep) {
      tc_fence_after();
      if (mode == 0 || mode == 6) {
        int n = mode == 6 ? 32 : 8;
        for (int s = 0; s < n; ++s)
          mma_bf16(tmem, sdesc(sb + (s & 7) * 4096, 2048, 128), sdesc(sb + 32768 + (s & 7) * 4096, 2048, 128),
                   idesc_bf16(128, 128, 0, 0), s > 0);
      } else if (mode == 1) {
        for (int s = 0; s < 8; ++s)
          for (int hlf = 0; hlf < 2; ++hlf)
            mma_bf16(tmem + 64 * hlf, sdesc(sb + s * 4096, 2048, 128), sdesc(sb + 32768 + hlf * 1024 + s * 4096, 2048, 128),
                     idesc_bf16(128, 64, 0, 0), s > 0);
      } else if (mode == 2) {
        for (int s = 0; s < 8; ++s)
          mma_bf16(tmem, sdesc(sb + s * 4096, 2048, 128), sdesc(sb + 32768 + s * 8192, 4096, 128),
                   idesc_bf16(128, 256, 0, 0), s > 0);
      } else if (mode == 3) {
        for (int s = 0; s < 8; ++s)
          mma_bf16(tmem, sdesc(sb + s * 256, 128, 2048), sdesc(sb + 32768 + s * 256, 128, 2048),
                   idesc_bf16(128, 128, 1, 1), s > 0);
      } else if (mode == 4) {
        for (int s = 0; s < 8; ++s)
          for (int g = 0; g < 2; ++g)
            mma_bf16(tmem + 128 * g, sdesc(sb + s * 4096, 2048, 128), sdesc(sb + 32768 + s * 4096, 2048, 128),
                     idesc_bf16(128, 128, 0, 0), s > 0);
      } else if (mode == 5) {
        for (int s = 0; s < 8; ++s)
          mma_bf16(tmem, sdesc(sb + s * 256, 128, 2048), sdesc(sb + 65536 + s * 256, 128, 2048),
                   idesc_bf16(128, 16, 1, 1), s > 0);
      }
      mma_commit(&bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
    long long t1 = clock64();
    out[mode] = (t1 - t0) / 16;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"8 x N128 same D (K,K)", "16 x N64 two D", "8 x N256 same D", "8 x N128 same D (MN,MN)",
                         "16 x N128 two GEMMs interleaved", "8 x N16 same D (MN,MN)", "32 x N128 same D (K,K)"};
  for (int m = 0; m < 7; ++m) {
    bench<<<1, 128, 200 * 1024>>>(d, m);
    cudaError_t e = cudaDeviceSynchronize();
    long long v = 0;
    cudaMemcpy(&v, d + m, sizeof(v), cudaMemcpyDeviceToHost);
    printf("%-36s %6lld cycles per group  (%s)\n", names[m], v, cudaGetErrorString(e));
  }
  return 0;
}
