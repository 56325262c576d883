// Microbenchmark: throughput of flushing 128 KB fp32 partials from each CTA into L2 with
// red.global.add.v4.f32, plain st.global.v4, TMA bulk reduce (smem->global .add.f32) and
// TMA bulk store, for different grid sizes and replica counts.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

__global__ void __launch_bounds__(512, 1) k(float* dst, int nrep, int mode, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  float* base = dst + (size_t)(blockIdx.x % nrep) * 32768;
  for (int i = tid; i < 32768; i += 512) reinterpret_cast<float*>(smem)[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      for (int q = 0; q < 16; ++q) {
        float* p = base + (size_t)tid * 64 + 4 * q;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else if (mode == 1) {
      for (int q = 0; q < 16; ++q) {
        float* p = base + (size_t)(q * 512 + tid) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else if (mode == 2) {
      for (int q = 0; q < 16; ++q) {
        float* p = base + (size_t)(q * 512 + tid) * 4;
        asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
      }
    } else if (mode == 3) {
      if (tid == 0) {
        for (int s = 0; s < 4; ++s) bulk_reduce_add_f32(base + s * 8192, smem_u32(smem) + s * 32768, 32768);
        bulk_commit();
        bulk_wait_read0();
      }
      __syncthreads();
    } else if (mode == 4) {
      if (tid == 0) {
        for (int s = 0; s < 4; ++s)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + s * 8192),
                       "r"(smem_u32(smem) + s * 32768), "r"(32768) : "memory");
        bulk_commit();
        bulk_wait_read0();
      }
      __syncthreads();
    } else if (mode == 5) {   // bulk reduce issued by 4 threads (one per 32 KB piece)
      if (tid < 128 && (tid & 31) == 0) {
        int s = tid >> 5;
        bulk_reduce_add_f32(base + s * 8192, smem_u32(smem) + s * 32768, 32768);
        bulk_commit();
        bulk_wait_read0();
      }
      __syncthreads();
    } else if (mode == 6) {   // bulk reduce in 4 KB pieces by 32 threads
      if (tid < 32) {
        for (int s = 0; s < 32; s += 32) {}
        bulk_reduce_add_f32(base + tid * 1024, smem_u32(smem) + tid * 4096, 4096);
        bulk_commit();
        bulk_wait_read0();
      }
      __syncthreads();
    }
  }
  if (tid == 0) bulk_wait0();
}

int main() {
  float* d;
  cudaMalloc(&d, (size_t)148 * 32768 * 4);
  cudaMemset(d, 0, (size_t)148 * 32768 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const char* names[] = {"red.v4 row-contig (thread=64 floats)", "red.v4 coalesced", "st.v4 coalesced",
                         "bulk reduce 4x32KB (1 thr)", "bulk store 4x32KB", "bulk reduce 4 thr", "bulk reduce 32x4KB"};
  int grids[] = {148, 16, 1};
  int reps[] = {148, 16};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int m = 0; m < 7; ++m)
    for (int g : grids)
      for (int r : reps) {
        if (r > g && r != 148) continue;
        int nr = r > g ? g : r;
        const int iters = 64;
        k<<<g, 512, 131072>>>(d, nr, m, 4);
        cudaEventRecord(a);
        k<<<g, 512, 131072>>>(d, nr, m, iters);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double bytes = (double)g * iters * 131072;
        double us_per_flush = ms * 1e3 / iters;
        printf("%-40s grid %3d rep %3d: %7.2f us per 128KB flush (%5.0f cyc @1.9GHz), agg %6.2f TB/s  %s\n", names[m], g, nr,
               us_per_flush, us_per_flush * 1900, bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
      }
  return 0;
}
