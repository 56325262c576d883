// Probe (tooling) for a cluster-pipelined W = 256 design:
//   a) how many 6-CTA clusters (3 CTA pairs) of a 1-CTA/SM kernel fit on the GPU at once
//   b) the TMEM layout of a cta_group::2 M = 128 MMA (64 rows per CTA), and whether a second
//      such accumulator at lane offset 16 of the same columns works, on the pair (2, 3)
//   c) back-to-back pair M = 128, N = 256, K = 16 MMAs: cycles per instruction
//   d) shared -> peer shared bulk copies (cp.async.bulk.shared::cluster): bytes per cycle
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2210_14907_b200/csrc pair_probe.cu -o pair_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

__device__ void put(uint8_t* base, int R, int r, int k, float v) {   // K-major core layout, [R][16]
  *reinterpret_cast<__nv_bfloat16*>(base + (k / 8) * R * 16 + r * 16 + (k % 8) * 2) = __float2bfloat16(v);
}
__device__ __forceinline__ void mma2_commit_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void bulk_s2peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst_cluster), "r"(src), "r"(bytes), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}

__global__ void __cluster_dims__(6, 1, 1) __launch_bounds__(128, 1) k(float* out, long long* cyc, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, cbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank(), pair = rank >> 1, leader = (rank & 1) == 0;
  uint8_t* sA = smem;              // [64 rows][16] bf16 (2 KB) per CTA
  uint8_t* sB = smem + 4096;       // [128 n][16] bf16 (4 KB) per CTA (its N-half)
  for (int i = tid; i < 8192 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  // A[m][0] = global row + 1 (rows 64 * (rank & 1) + m), B[n][0] = global column + 1 (n + 128 (rank & 1))
  if (tid < 64) put(sA, 64, tid, 0, 64 * (rank & 1) + tid + 1);
  if (tid < 128) put(sB, 128, tid, 0, 128 * (rank & 1) + tid + 1);
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); mbar_init(&cbar, 1); mbar_fence_init(); }
  if (warp == 0) tmem_alloc2(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint16_t mask = (uint16_t)(3u << (2 * pair));
  if (mode == 0 || mode == 3) {   // b) layout: D = A B^T (M = 128 pair rows, N = 256) at lane offset 0 (pairs 0, 2) or 16 (pair 1)
    const uint32_t loff = (mode == 3 && pair == 1) ? 16u : 0u;
    if (leader && tid == 0) {
      mma2_bf16(tmem + (loff << 16), sdesc(smem_u32(sA), 64 * 16, 128), sdesc(smem_u32(sB), 128 * 16, 128),
                idesc_bf16(128, 256, 0, 0), 0);
      mma2_commit_mask(&bar, mask);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);   // columns 0..31
    float w[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 224, w);   // columns 224..255
    out[(blockIdx.x * 128 + tid) * 3 + 0] = v[0];
    out[(blockIdx.x * 128 + tid) * 3 + 1] = v[1];
    out[(blockIdx.x * 128 + tid) * 3 + 2] = w[31];
  } else if (mode == 1) {   // c) throughput of 64 pair M = 128 N = 256 instructions
    if (leader && tid == 0) {
      long long best = 1 << 30;
      uint32_t ph = 0;
      for (int rep = 0; rep < 8; ++rep) {
        const long long t0 = clock64();
        for (int i = 0; i < 64; ++i)
          mma2_bf16(tmem, sdesc(smem_u32(sA), 64 * 16, 128), sdesc(smem_u32(sB), 128 * 16, 128),
                    idesc_bf16(128, 256, 0, 0), i > 0);
        mma2_commit_mask(&bar, mask);
        mbar_wait(&bar, ph);
        ph ^= 1;
        const long long t = clock64() - t0;
        if (t < best) best = t;
      }
      cyc[blockIdx.x] = best;
    } else if (tid == 0) {
      uint32_t ph = 0;
      for (int rep = 0; rep < 8; ++rep) { mbar_wait(&bar, ph); ph ^= 1; }
    }
  } else {   // d) CTA r copies 48 KB chunks to CTA (r + 2) % 6 (a different pair), 32 times
    uint8_t* src = smem + 16384;
    uint8_t* dst = smem + 16384 + 65536;
    const uint32_t CH = 49152;
    if (tid == 0) {
      const uint32_t to = (rank + 2) % 6;
      const uint32_t dbar = mapa(smem_u32(&cbar), to), ddst = mapa(smem_u32(dst), to);
      const long long t0 = clock64();
      uint32_t ph = 0;
      for (int i = 0; i < 32; ++i) {
        // receiver side: this CTA's cbar expects CH bytes from (rank + 4) % 6
        mbar_arrive_expect_tx(&cbar, CH);
        bulk_s2peer(ddst, smem_u32(src), CH, dbar);
        mbar_wait(&cbar, ph);   // my incoming copy landed
        ph ^= 1;
      }
      cyc[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) tmem_dealloc2(tmem, 256);
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  int ncl = 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(144);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 6; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr; cfg.numAttrs = 1;
  cudaError_t e0 = cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
  printf("a) max active 6-CTA clusters (200 KB smem, 1 CTA/SM): %d (%s)\n", ncl, cudaGetErrorString(e0));
  float* d; long long* c;
  cudaMalloc(&d, 144 * 128 * 3 * sizeof(float));
  cudaMalloc(&c, 144 * sizeof(long long));
  if (which == 1) goto C;
  if (which == 2) goto D;
  {
  k<<<6, 128, 200 * 1024>>>(d, c, which == 3 ? 3 : 0);
  cudaError_t e = cudaDeviceSynchronize();
  float h[6 * 128 * 3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("b) %s; per CTA: TMEM lane -> (col0, col1, col255) for lanes 0..31 step 1 of quadrant 0 and lanes 16, 32, 48\n", cudaGetErrorString(e));
  for (int b = 0; b < 6; ++b) {
    printf(" CTA %d:", b);
    for (int l : {0, 1, 15, 16, 17, 31, 32, 47, 48, 64, 96, 111, 112, 127})
      printf(" %d:(%g,%g,%g)", l, h[(b * 128 + l) * 3], h[(b * 128 + l) * 3 + 1], h[(b * 128 + l) * 3 + 2]);
    printf("\n");
  }
  return 0;
  }
C: {
  k<<<144, 128, 200 * 1024>>>(d, c, 1);
  cudaError_t e = cudaDeviceSynchronize();
  long long hc[144];
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("c) %s; pair M128 N256 K16 x64: %lld cyc (%.1f per instr; floor 64)\n", cudaGetErrorString(e), hc[0], hc[0] / 64.0);
  return 0;
  }
D: {
  k<<<144, 128, 200 * 1024>>>(d, c, 2);
  cudaError_t e = cudaDeviceSynchronize();
  long long hc[144];
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 144; ++i) s += hc[i];
  s /= 144;
  printf("d) %s; DSMEM bulk copies 32 x 48 KB: %.0f cyc = %.1f B/cyc per CTA (all 144 CTAs sending)\n", cudaGetErrorString(e), s,
         32.0 * 49152 / s);
  }
  return 0;
}
