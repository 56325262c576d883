// tc_epi.cuh -- register-level helpers shared by the tcgen05 kernels' epilogues (K3t, K3h):
// bf16 packing, the MUFU activations, vector shared-memory access and the warp transpose-sum.
#pragma once
#include <stdint.h>

#include "tc_ptx.cuh"   // check_smem (bounds-checked builds)

namespace nbm {
namespace epi {

// core-matrix (8 rows x 16 B) layout of an [R][C] bf16 tile: element (r, c) at
// (c/8)*R*16 + r*16 + (c%8)*2 bytes.
__device__ __forceinline__ uint32_t core_off(int R, int r, int c8) { return (uint32_t)(c8 * R * 16 + r * 16); }

// two fp32 -> packed bf16x2 (RNE), one cvt.rn.bf16x2.f32 (F2FP) instruction; a -> low half
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// bf16 path activation: MUFU tanh.approx.f32 (max relative error 2^-10.99, below the bf16
// operand rounding; the fp32 configs use the accurate tanhf, G15).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// logistic via one MUFU op: sg(z) = 0.5 + 0.5 tanh(z / 2)
__device__ __forceinline__ float sigmoid_fast(float z) { return fmaf(0.5f, tanh_fast(0.5f * z), 0.5f); }

// lane j of the warp receives the sum over the warp's 32 rows of v[j] (fixed butterfly)
__device__ __forceinline__ float warp_transpose_sum(float (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? v[i] : v[i + s];
      const float keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// half-warp version: lanes 16*side + j hold 32 values of row j (16 rows per half-warp); after
// the butterfly, lane 16*side + j holds the sum over the half-warp's 16 rows of v[j] (first
// return) and of v[16 + j] (second)
__device__ __forceinline__ void warp_transpose_sum16(float (&v)[32], int lane, float& s0, float& s1) {
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < s; ++i) {
        const float send = up ? v[16 * b + i] : v[16 * b + i + s];
        const float keep = up ? v[16 * b + i + s] : v[16 * b + i];
        v[16 * b + i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
  }
  s0 = v[0];
  s1 = v[16];
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  tc::check_smem(addr, 16);
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void ld_shared_v4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  tc::check_smem(addr, 16);
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr) : "memory");
}

}  // namespace epi
}  // namespace nbm
