// Microbenchmark: CTA-pair (cluster of 2) shared-memory exchange bandwidth.
//  mode 0: cp.async.bulk shared::cta -> shared::cluster (peer), 64 KB per CTA per iteration (4 x 16 KB)
//  mode 1: ld.shared::cluster.v4 by all 512 threads from the peer's smem (64 KB), sum into a register
//  mode 2: st.shared::cluster.v4 by all 512 threads into the peer's smem (64 KB)
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t cta) { uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k(int mode, int iters, long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x;
  for (int i = tid; i < 32768; i += 512) reinterpret_cast<float*>(smem)[i] = 1.0f;
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  csync();
  const uint32_t peer = rank ^ 1u;
  const uint32_t src = su32(smem), dst = mapa(su32(smem) + 65536, peer), pbar = mapa(su32(&bar), peer);
  float acc = 0.f;
  uint32_t ph = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(65536) : "memory");
      }
      csync();   // both expect_tx posted before any copy lands
      if (tid == 0) {
        for (int s = 0; s < 4; ++s)
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + s * 16384), "r"(src + s * 16384), "r"(16384), "r"(pbar) : "memory");
        mbar_wait(su32(&bar), ph);
      }
      ph ^= 1;
      __syncthreads();
    } else if (mode == 1) {
      const uint32_t ps = mapa(src, peer);
      for (int q = 0; q < 8; ++q) {
        float a, b, c, d;
        asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(ps + (q * 512 + tid) * 16));
        acc += a + b + c + d;
      }
      __syncthreads();
    } else {
      for (int q = 0; q < 8; ++q)
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(dst + (q * 512 + tid) * 16), "f"(acc + q) : "memory");
      csync();
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
}
int main() {
  long long* d; float* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  const char* nm[] = {"bulk push 64KB", "ld.shared::cluster.v4 64KB", "st.shared::cluster.v4 64KB"};
  for (int m = 0; m < 3; ++m)
    for (int g : {2, 148}) {
      int iters = 200;
      k<<<g, 512, 140000>>>(m, 10, d, s);
      k<<<g, 512, 140000>>>(m, iters, d, s);
      long long h[148];
      cudaError_t e = cudaMemcpy(h, d, g * 8, cudaMemcpyDeviceToHost);
      double c = (double)h[0] / iters;
      printf("%-28s grid %3d: %8.0f cyc per 64 KB per CTA = %6.1f B/cyc/SM  %s\n", nm[m], g, c, 65536.0 / c, cudaGetErrorString(e));
    }
}
