// Microbenchmark (tooling): the single-CTA tcgen05 costs that pace K3t's serial tile chain.
//   A  issue cost: R back-to-back cta_group::1 bf16 MMAs (M = 128, N = 16/64/128, K = 16) by one
//      thread -- cycles until the issuing thread is free again, and until the commit arrives
//   B  round trip: one GEMM of K = 64 / 128 (4 / 8 instructions) + commit + wait, repeated
//   C  TMEM -> registers: tcgen05.ld.32x32b.x32 + wait::ld by 4 / 8 / 16 warps over 512 columns
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2210_14907_b200/csrc tc_issue_bench.cu -o tc_issue_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

// the MMA issued by one elected lane of a converged warp (the predicate from elect.sync inside
// the asm, operands warp-uniform): no per-instruction waterfall loop around UTCHMMA
__device__ __forceinline__ void mma_bf16_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 rx;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync rx|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      ".reg .b32 rx;\n"
      "elect.sync rx|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(512, 1) k(long long* out, int mode, int arg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3F803F80u;
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase, sb = smem_u32(smem);
  uint32_t phase = 0;
  if (mode == 0 || mode == 1) {   // A: issue cost of R instructions of N = arg
    const int R = mode == 0 ? 64 : 8;
    if (tid == 0) {
      const uint32_t id = idesc_bf16(128, arg, 0, 0);
      long long best_issue = 1 << 30, best_done = 1 << 30;
      for (int rep = 0; rep < 8; ++rep) {
        const long long t0 = clock64();
        for (int i = 0; i < R; ++i)
          mma_bf16(tmem, sdesc(sb + (i & 3) * 4096, 2048, 128), sdesc(sb + 65536 + (i & 3) * 4096, 2048, 128), id,
                   i > 0);
        const long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        const long long t2 = clock64();
        if (t1 - t0 < best_issue) best_issue = t1 - t0;
        if (t2 - t0 < best_done) best_done = t2 - t0;
      }
      out[0] = best_issue;
      out[1] = best_done;
    }
  } else if (mode == 4 || mode == 5) {   // A': the same R instructions issued by a converged warp 0
    const int R = mode == 4 ? 64 : 8;
    if (warp == 0) {
      const uint32_t id = idesc_bf16(128, arg, 0, 0);
      long long best_issue = 1 << 30, best_done = 1 << 30;
      const uint64_t a0 = sdesc(sb, 2048, 128), b0 = sdesc(sb + 65536, 2048, 128);
      for (int rep = 0; rep < 8; ++rep) {
        __syncwarp();
        const long long t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < R; ++i)
          mma_bf16_warp(tmem, a0 + (uint64_t)((i & 3) * 256), b0 + (uint64_t)((i & 3) * 256), id, i > 0);
        const long long t1 = clock64();
        mma_commit_warp(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        const long long t2 = clock64();
        if (t1 - t0 < best_issue) best_issue = t1 - t0;
        if (t2 - t0 < best_done) best_done = t2 - t0;
      }
      if (tid == 0) {
        out[0] = best_issue;
        out[1] = best_done;
      }
    }
  } else if (mode == 2) {   // B: round trip of one K = 16 * arg GEMM, N = 128
    if (tid == 0) {
      const uint32_t id = idesc_bf16(128, 128, 0, 0);
      long long best = 1 << 30;
      for (int rep = 0; rep < 16; ++rep) {
        const long long t0 = clock64();
        tc_fence_after();
        for (int i = 0; i < arg; ++i)
          mma_bf16(tmem, sdesc(sb + i * 4096, 2048, 128), sdesc(sb + 65536 + (i & 3) * 4096, 2048, 128), id, i > 0);
        mma_commit(&bar);
        mbar_wait(&bar, phase);
        phase ^= 1;
        const long long t2 = clock64();
        if (t2 - t0 < best) best = t2 - t0;
      }
      out[0] = best;
      out[1] = 0;
    }
  } else {   // C: TMEM loads by `arg` warps: each warp reads its lane quadrant, all 512 columns, 8 times
    __syncthreads();
    const long long t0 = clock64();
    float acc = 0.f;
    if (warp < arg) {
      const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
      const int nq = arg / 4;                        // warps sharing a quadrant split the columns
      const int c0 = (warp >> 2) * (512 / nq), c1 = c0 + 512 / nq;
      for (int rep = 0; rep < 8; ++rep)
        for (int c = c0; c < c1; c += 32) {
          float v[32];
          tmem_ld32(tmem + lane_base + c, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) acc += v[j];
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) { out[0] = t1 - t0; out[1] = 0; }
    if (acc == 12345.f) out[2] = 1;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  long long h[2];
  for (int n : {16, 64, 128, 256}) {
    for (int m : {0, 1, 4, 5}) {
      k<<<1, 512, 160 * 1024>>>(d, m, n);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const int R = (m == 0 || m == 4) ? 64 : 8;
      printf("A%s %2d MMAs M128 N%-3d K16: issue %6lld cyc (%5.1f/instr)  done %6lld cyc (%5.1f/instr; floor %d)  %s\n", m >= 4 ? "'" : " ", R,
             n, h[0], (double)h[0] / R, h[1], (double)h[1] / R, 128 * n / 256, cudaGetErrorString(e));
    }
  }
  for (int kk : {1, 4, 8}) {
    k<<<1, 512, 160 * 1024>>>(d, 2, kk);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("B  round trip M128 N128 K%-3d: %6lld cyc  %s\n", 16 * kk, h[0], cudaGetErrorString(e));
  }
  for (int w : {4, 8, 16}) {
    k<<<1, 512, 160 * 1024>>>(d, 3, w);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = 8.0 * 128 * 512 * 4;
    printf("C  TMEM ld by %2d warps: %7lld cyc for %.0f KB = %5.1f B/cyc  %s\n", w, h[0], bytes / 1024, bytes / h[0],
           cudaGetErrorString(e));
  }
  return 0;
}
