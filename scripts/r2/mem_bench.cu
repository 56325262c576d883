// Microbenchmark (tooling): the SM <-> L2 interface under the traffic mix of K3w, on all 148 SMs
// (one 512-thread CTA per SM, data L2-resident).  Cycles per KB for:
//   0  TMA bulk loads (16 KB chunks, 4-deep ring)                     alone
//   1  TMA bulk stores (16 KB chunks, smem -> global)                  alone
//   2  red.global.add.v4.f32 by 480 threads                            alone
//   3  st.global.v4 by 480 threads                                     alone
//   4  TMA loads by warp 0 while 480 threads issue reductions          (load rate, red rate)
//   5  TMA loads while TMA stores of the same CTA run (both by warp 0) (combined)
//   6  TMA loads while 480 threads issue plain stores
//   7  TMA bulk reductions (cp.reduce.async.bulk .add.f32, 16 KB chunks, smem -> global)  alone
//   8  TMA loads while the same warp issues TMA bulk reductions           (combined)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2210_14907_b200/csrc mem_bench.cu -o mem_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

constexpr int CH = 16384, STAGES = 4;
constexpr int LOADS = 256;      // 4 MB of loads per CTA
constexpr int REDS = 2048;      // per thread: 2048 x 16 B = 32 KB -> 15 MB per CTA (480 threads)

__global__ void __launch_bounds__(512, 1) k(const uint8_t* src, float* dst, uint8_t* sdst, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES];
  __shared__ long long tl, tr;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const uint8_t* my = src + (size_t)(blockIdx.x % 32) * (1 << 20);   // 32 MB of L2-resident source
  uint8_t* myd = sdst + (size_t)blockIdx.x * (1 << 20);
  float* rd = dst + (size_t)(blockIdx.x % 16) * 65536;                // 16 replicas x 256 KB
  const uint32_t sb = smem_u32(smem);
  __syncthreads();
  const long long t0 = clock64();
  if (warp == 0) {
    if (tid == 0) {
      uint32_t ph[STAGES] = {0, 0, 0, 0};
      if (mode == 0 || mode == 4 || mode == 5 || mode == 6 || mode == 8) {
        for (int i = 0; i < LOADS; ++i) {
          const int s = i % STAGES;
          if (i >= STAGES) { mbar_wait(&full[s], ph[s]); ph[s] ^= 1; }
          mbar_arrive_expect_tx(&full[s], CH);
          bulk_copy_g2s(sb + s * CH, my + (size_t)(i % 64) * CH, CH, &full[s]);
          if (mode == 5) {   // interleave a 16 KB store from the other half of smem
            bulk_copy_s2g(myd + (size_t)(i % 64) * CH, sb + 65536 + (i % 4) * CH, CH);
            bulk_commit();
          }
          if (mode == 8) {   // interleave a 16 KB bulk reduction
            bulk_reduce_add_f32(dst + (size_t)(blockIdx.x % 16) * 65536 + (size_t)(i % 16) * (CH / 4),
                                sb + 65536 + (i % 4) * CH, CH);
            bulk_commit();
          }
        }
        for (int s = 0; s < STAGES; ++s) { mbar_wait(&full[s], ph[s]); ph[s] ^= 1; }
        if (mode == 5 || mode == 8) bulk_wait0();
      } else if (mode == 7) {
        float* rdst = dst + (size_t)(blockIdx.x % 16) * 65536;
        for (int i = 0; i < LOADS; ++i) {
          bulk_reduce_add_f32(rdst + (size_t)(i % 16) * (CH / 4), sb + (i % 4) * CH, CH);
          bulk_commit();
        }
        bulk_wait0();
      } else if (mode == 1) {
        for (int i = 0; i < LOADS; ++i) {
          bulk_copy_s2g(myd + (size_t)(i % 64) * CH, sb + (i % 4) * CH, CH);
          bulk_commit();
        }
        bulk_wait0();
      }
      tl = clock64() - t0;
    }
  } else if (mode == 2 || mode == 3 || mode == 4 || mode == 6) {
    const int t = tid - 32;
    for (int i = 0; i < REDS; ++i) {
      float* p = rd + ((size_t)(i % 128) * 480 + t) * 4;
      if (mode == 2 || mode == 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.0f), "f"(1.0f), "f"(1.0f), "f"(1.0f) : "memory");
      else
        asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.0f), "f"(1.0f), "f"(1.0f), "f"(1.0f) : "memory");
    }
    __threadfence();
    asm volatile("bar.sync 1, 480;");
    if (t == 0) tr = clock64() - t0;
  }
  __syncthreads();
  if (tid == 0) { out[2 * blockIdx.x] = tl; out[2 * blockIdx.x + 1] = tr; }
}

int main() {
  uint8_t *src, *sdst; float* dst; long long* out;
  cudaMalloc(&src, 64 << 20); cudaMalloc(&sdst, (size_t)148 << 20); cudaMalloc(&dst, 16 * 65536 * 4 * 4);
  cudaMemset(src, 0, 64 << 20); cudaMemset(dst, 0, 16 * 65536 * 16);
  cudaMalloc(&out, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const char* names[] = {"TMA loads alone", "TMA stores alone", "red.v4 alone", "st.v4 alone",
                         "TMA loads + red.v4", "TMA loads + TMA stores", "TMA loads + st.v4",
                         "TMA bulk reduce alone", "TMA loads + TMA bulk reduce"};
  for (int m = 0; m < 9; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(out, 0, 2 * 148 * sizeof(long long));
      k<<<148, 512, 160 * 1024>>>(src, dst, sdst, m, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[296];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      double l = 0, r = 0;
      for (int b = 0; b < 148; ++b) { l += h[2 * b]; r += h[2 * b + 1]; }
      l /= 148; r /= 148;
      const double lkb = LOADS * 16.0 * ((m == 5 || m == 8) ? 2 : 1), rkb = 480.0 * REDS * 16 / 1024;
      if (rep == 1)
        printf("%-26s load/store %8.0f cyc = %6.1f B/clk | red/st %8.0f cyc = %6.1f B/clk  %s\n", names[m], l,
               l > 0 ? lkb * 1024 / l : 0.0, r, r > 0 ? rkb * 1024 / r : 0.0, cudaGetErrorString(e));
    }
  }
  return 0;
}
