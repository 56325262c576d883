// Microbenchmark (tooling): throughput of back-to-back pair MMAs (tcgen05.mma.cta_group::2,
// bf16, M = 256, K = 16 per instruction) in the operand layouts K3w uses, and with 128-byte
// swizzled K-major operands.  One GEMM = 16 instructions (K = 256); 8 GEMMs back to back per
// commit, 16 repetitions; prints cycles per GEMM (ideal at 8192 MAC/clk per pair: N = 256 -> 2048).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2210_14907_b200/csrc mma2_bench.cu -o mma2_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

using namespace nbm::tc;

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

__global__ void __cluster_dims__(2, 1, 1) bench(long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 192 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3F803F80u;
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (tid < 32) tmem_alloc2(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tbase, sb = (smem_u32(smem) + 1023) & ~1023u;
  const bool leader = cluster_rank() == 0;
  const uint32_t A = sb, B = sb + 65536;
  uint32_t phase = 0;
  long long t0 = 0;
  const int REP = 16, G = 8;
  for (int rep = 0; rep < REP + 1; ++rep) {
    if (rep == 1) t0 = clock64();
    if (leader && tid == 0) {
      tc_fence_after();
      for (int g = 0; g < G; ++g) {
        for (int kk = 0; kk < 16; ++kk) {
          uint64_t ad, bd;
          uint32_t id, d = tmem;
          if (mode == 0) {          // fwd: A K-major, B K-major (no swizzle)
            ad = sdesc(A + kk * 2 * 2048, 2048, 128); bd = sdesc(B + (kk & 3) * 4096 + (kk >> 2) * 0, 2048, 128);
            id = idesc_bf16(256, 256, 0, 0);
          } else if (mode == 1) {   // dH: A K-major, B MN-major
            ad = sdesc(A + kk * 2 * 2048, 2048, 128); bd = sdesc(B + (kk & 3) * 256, 128, 1024);
            id = idesc_bf16(256, 256, 0, 1);
          } else if (mode == 2) {   // dW: A MN-major, B MN-major
            ad = sdesc(A + (kk >> 3) * 32768 + (kk & 7) * 256, 128, 2048);
            bd = sdesc(B + (kk >> 3) * 32768 + (kk & 7) * 256, 128, 2048);
            id = idesc_bf16(256, 256, 1, 1); d = tmem + 256;
          } else if (mode == 3) {   // fwd, 128B swizzle K-major: rows of 64 K (128 B), 8-row atoms (1 KB)
            const int kb = kk >> 2, ki = kk & 3;   // K block of 64, 16-element step inside it
            ad = sdesc_sw128(A + kb * 16384 + ki * 32, 1024); bd = sdesc_sw128(B + (kb & 1) * 16384 + ki * 32, 1024);
            id = idesc_bf16(256, 256, 0, 0);
          } else if (mode == 4) {   // N = 128 halves (2 x 16 instructions), K-major no swizzle
            ad = sdesc(A + kk * 2 * 2048, 2048, 128); bd = sdesc(B + (kk & 3) * 4096, 2048, 128);
            id = idesc_bf16(256, 128, 0, 0);
            mma2_bf16(tmem + 128, ad, bd, id, kk > 0);
          } else if (mode == 6 || mode == 7) {   // M = 128 pairs (64 rows per CTA): two instructions per K-step
            // (rows 0-63 -> D columns [0,128), rows 64-127 -> [128,256)); A [64][256] K-major blocks
            ad = sdesc(A + kk * 2 * 1024, 1024, 128); bd = sdesc(B + kk * 2 * 2048, 2048, 128);
            id = idesc_bf16(128, 256, 0, 0);
            mma2_bf16(tmem, ad, bd, id, kk > 0);
            ad = sdesc(A + 32768 + kk * 2 * 1024, 1024, 128);
            if (mode == 7) d = tmem + 128;
          } else {                   // mode 5: fwd, A K-major 128B swizzle, B no swizzle
            const int kb = kk >> 2, ki = kk & 3;
            ad = sdesc_sw128(A + kb * 16384 + ki * 32, 1024); bd = sdesc(B + (kk & 3) * 4096, 2048, 128);
            id = idesc_bf16(256, 256, 0, 0);
          }
          mma2_bf16(d, ad, bd, id, kk > 0);
        }
      }
      mma2_commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
  }
  long long t1 = clock64();
  if (leader && tid == 0) out[mode] = (t1 - t0) / (REP * G);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (tid < 32) tmem_dealloc2(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"fwd  A K / B K (no swizzle)", "dH   A K / B MN (no swizzle)", "dW   A MN / B MN (no swizzle)",
                         "fwd  A K / B K (128B swizzle)", "fwd  N=128 x2 halves (no swizzle)",
                         "fwd  A K sw128 / B K no swizzle", "fwd  2 x M128 pair, same D (K-major)",
                         "fwd  2 x M128 pair, D halves (K-major)"};
  for (int m = 0; m < 8; ++m) {
    bench<<<2, 128, 200 * 1024>>>(d, m);
    cudaError_t e = cudaDeviceSynchronize();
    long long v = 0;
    cudaMemcpy(&v, d + m, sizeof(v), cudaMemcpyDeviceToHost);
    printf("%-40s %6lld cycles per GEMM (M256 N256 K256; ideal 2048)  %s\n", names[m], v, cudaGetErrorString(e));
  }
  return 0;
}
