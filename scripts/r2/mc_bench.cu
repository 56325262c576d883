// Microbenchmark (tooling): does TMA multicast relieve the SM <-> L2 interface for K3w's weight
// slices?  All 148 SMs, clusters of 2, one 512-thread CTA per SM.  Per round each CTA receives
// 64 KB (4 x 16 KB chunks, L2-resident source) while 480 threads issue red.global.add.v4:
//   0  unicast: each CTA loads its own 4 chunks
//   1  multicast: each CTA issues 2 of the 4 chunks with .multicast::cluster to both CTAs
// Prints the per-SM received-load rate and the reduction rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2210_14907_b200/csrc mc_bench.cu -o mc_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

constexpr int CH = 16384, ROUNDS = 64, REDS = 2048;

__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k(const uint8_t* src, float* dst, int mode, int reds,
                                                                       long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full, armed, done;
  __shared__ long long tl, tr;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  if (tid == 0) { mbar_init(&full, 1); mbar_init(&armed, 1); mbar_init(&done, 1); mbar_fence_init(); }
  __syncthreads();
  cluster_sync();
  const uint8_t* my = src + (size_t)((blockIdx.x >> 1) % 32) * (1 << 20);   // the pair shares a source
  float* rd = dst + (size_t)(blockIdx.x % 16) * 65536;
  const uint32_t sb = smem_u32(smem);
  const long long t0 = clock64();
  if (warp == 0) {
    uint32_t ph = 0;
    for (int r = 0; r < ROUNDS; ++r) {
      if (tid == 0) {
        mbar_arrive_expect_tx(&full, 4 * CH);
        if (mode == 1) {   // both CTAs armed before any multicast lands: hand-shake on `armed`
          arrive_remote(&armed, rank ^ 1u);
          mbar_wait(&armed, ph);
        }
        if (mode == 0) {
          for (int c = 0; c < 4; ++c) bulk_copy_g2s(sb + c * CH, my + (size_t)((r * 4 + c) % 64) * CH, CH, &full);
        } else {
          for (int c = (int)rank; c < 4; c += 2) bulk_g2s_mc(sb + c * CH, my + (size_t)((r * 4 + c) % 64) * CH, CH, &full, 3);
        }
      }
      mbar_wait(&full, ph);
      if (mode == 1 && tid == 0) {   // the peer has also received this round before either re-arms
        arrive_remote(&done, rank ^ 1u);
        mbar_wait(&done, ph);
      }
      __syncwarp();
      ph ^= 1;
    }
    if (tid == 0) tl = clock64() - t0;
  } else {
    const int t = tid - 32;
    for (int i = 0; i < reds; ++i) {
      float* p = rd + ((size_t)(i % 128) * 480 + t) * 4;
      asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.0f), "f"(1.0f), "f"(1.0f), "f"(1.0f) : "memory");
    }
    __threadfence();
    asm volatile("bar.sync 1, 480;");
    if (t == 0) tr = clock64() - t0;
  }
  __syncthreads();
  if (tid == 0) { out[2 * blockIdx.x] = tl; out[2 * blockIdx.x + 1] = tr; }
  cluster_sync();
}

int main() {
  uint8_t* src; float* dst; long long* out;
  cudaMalloc(&src, 64 << 20); cudaMalloc(&dst, 16 * 65536 * 16);
  cudaMemset(src, 0, 64 << 20); cudaMemset(dst, 0, 16 * 65536 * 16);
  cudaMalloc(&out, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int reds : {0, REDS})
    for (int m = 0; m < 2; ++m)
      for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 512, 80 * 1024>>>(src, dst, m, reds, out);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[296];
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        double l = 0, r = 0;
        for (int b = 0; b < 148; ++b) { l += h[2 * b]; r += h[2 * b + 1]; }
        l /= 148; r /= 148;
        if (rep == 1)
          printf("%-10s reds %-5d: received loads %7.1f B/clk per SM | reductions %6.1f B/clk  %s\n",
                 m ? "multicast" : "unicast", reds, ROUNDS * 4.0 * CH / l, reds ? 480.0 * reds * 16 / r : 0.0,
                 cudaGetErrorString(e));
      }
  return 0;
}
