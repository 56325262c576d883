// Validation of the CTA-pair (cta_group::2) tcgen05 path used by K3w: M = 256 rows split
// over the two CTAs of a cluster, B split by N halves, TMEM allocated with cta_group::2,
// completion multicast to both CTAs; weight halves loaded by each CTA with a bulk copy and
// forwarded to the leader's barrier by a remote arrive.  Also checks the MN-major (dW)
// operand form.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2210_14907_b200/csrc pair_test.cu -o pair_test
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
using namespace nbm::tc;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_remote_leader(uint64_t* bar) {
  uint32_t a = smem_u32(bar), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(0));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "h"((unsigned short)3) : "memory");
}

// mode 0 (K-major, forward-like): D[m][n] = sum_k A[m][k] B[n][k]; CTA r holds A rows
//   [128r, 128r+128) and B rows (n) [128r, 128r+128), both K-major core layout.
// mode 1 (MN-major, dW-like): same math, but both operands stored MN-major:
//   element (m, k) at (m/8)*K*16 + k*16 + (m%8)*2 ... i.e. [k rows][m cols] activation layout.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_pair(const __nv_bfloat16* A, const uint16_t* Bpk, int K, float* D, int reps, long long* cyc, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bfull, bdone;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_rank();
  const uint32_t sA = smem_u32(smem), sB = sA + 128 * K * 2;
  for (int e = tid; e < 128 * K; e += 128) {
    const int m = e / K, k = e % K;
    const uint32_t off = mode == 0 ? (uint32_t)((k / 8) * 2048 + m * 16 + (k % 8) * 2)
                                   : (uint32_t)((m / 8) * K * 16 + k * 16 + (m % 8) * 2);
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = A[(size_t)(rank * 128 + m) * K + k];
  }
  if (tid == 0) {
    mbar_init(&bfull, rank == 0 ? 2 : 1);
    mbar_init(&bdone, 1);
    mbar_fence_init();
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t bytes = 128 * K * 2;
    mbar_arrive_expect_tx(&bfull, bytes);
    bulk_copy_g2s(sB, Bpk + (size_t)rank * 128 * K, bytes, &bfull);
    if (rank == 1) {
      mbar_wait(&bfull, 0);
      arrive_remote_leader(&bfull);
    }
  }
  const uint32_t idesc = idesc_bf16(256, 256, mode, mode);
  long long t0 = clock64();
  uint32_t ph = 0;
  for (int r = 0; r < reps; ++r) {
    if (rank == 0 && tid == 0) {
      if (r == 0) mbar_wait(&bfull, 0);
      tc_fence_after();
      for (int kk = 0; kk < K / 16; ++kk) {
        uint64_t ad, bd;
        if (mode == 0) {
          ad = sdesc(sA + kk * 2 * 2048, 2048, 128);
          bd = sdesc(sB + kk * 2 * 2048, 2048, 128);
        } else {   // MN-major: LBO = K-direction core stride (128), SBO = 8-column stride (K*16)
          ad = sdesc(sA + kk * 256, 128, K * 16);
          bd = sdesc(sB + kk * 256, 128, K * 16);
        }
        mma2(tmem, ad, bd, idesc, kk > 0);
      }
      commit2(&bdone);
    }
    mbar_wait(&bdone, ph);
    ph ^= 1;
    tc_fence_after();
  }
  long long t1 = clock64();
  if (tid == 0 && rank == 0) *cyc = (t1 - t0) / reps;
  for (int c = 0; c < 256; c += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(tid / 32 * 32) << 16) + c, v);
    for (int j = 0; j < 32; ++j) D[(size_t)(rank * 128 + tid) * 256 + c + j] = v[j];
  }
  tc_fence_before();
  cluster_sync_all();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

int main() {
  const int K = 256;
  std::vector<__nv_bfloat16> A(256 * K), B(256 * K);
  std::vector<float> Af(256 * K), Bf(256 * K);
  srand(1);
  for (int i = 0; i < 256 * K; ++i) {
    A[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); Af[i] = __bfloat162float(A[i]);
    B[i] = __float2bfloat16((rand() % 13 - 6) / 4.0f); Bf[i] = __bfloat162float(B[i]);
  }
  __nv_bfloat16* dA; uint16_t* dB; float* dD; long long* dc;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 256 * 256 * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 2 * 128 * K * 2;
  cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad = 0;
  for (int mode = 0; mode < 2; ++mode) {
    std::vector<uint16_t> Bp(256 * K);
    for (int n = 0; n < 256; ++n)
      for (int k = 0; k < K; ++k) {
        const int h = n / 128, nn = n % 128;
        uint16_t bits;
        memcpy(&bits, &B[n * K + k], 2);
        const size_t off = mode == 0 ? (size_t)(k / 8) * 1024 + nn * 8 + (k % 8) : (size_t)(nn / 8) * K * 8 + k * 8 + (nn % 8);
        Bp[(size_t)h * 128 * K + off] = bits;
      }
    cudaMemcpy(dB, Bp.data(), Bp.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 256 * 256 * 4);
    k_pair<<<2, 128, smem>>>(dA, dB, K, dD, 64, dc, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(256 * 256);
    long long cyc = 0;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < 256; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)Af[m * K + k] * Bf[n * K + k];
        maxerr = fmax(maxerr, fabs(s - D[m * 256 + n]));
      }
    printf("mode %d (%s): %s  max |D - ref| = %g   cycles per M256xN256xK%d = %lld (%.1f per K16 MMA)\n", mode,
           mode ? "MN-major" : "K-major", cudaGetErrorString(e), maxerr, K, cyc, (double)cyc / (K / 16));
    bad |= !(maxerr < 1e-3) || e != cudaSuccess;
  }
  return bad;
}
