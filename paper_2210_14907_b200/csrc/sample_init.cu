// sample_init.cu -- K1 point sampler, Xavier init and K4a Adam.
//
// K1 ("random collocation points"; G9):
// Philox4x32-10, key = seed, counter = (2i + j, step, stream); interior points are
// uniform integers on the 2^-24 lattice of [-1+h, 1-h]^3 converted exactly to fp32,
// boundary points pick a face uniformly.  Pure integer arithmetic -> bit-exact.
// One thread per point; the 12-byte AoS output is written through shared memory so
// each warp stores 384 contiguous bytes (coalesced).
#include "nbm_internal.cuh"

namespace nbm {

__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint4 philox_ctr(uint64_t seed, uint64_t counter, uint32_t w2,
                                            uint32_t stream) {
  return philox10(make_uint4((uint32_t)counter, (uint32_t)(counter >> 32), w2, stream),
                  (uint32_t)seed, (uint32_t)(seed >> 32));
}

__global__ void __launch_bounds__(256) k_sample(int kind, uint64_t seed, uint32_t step_arg,
                                                const int64_t* __restrict__ step_dev, int64_t first,
                                                int64_t n, int64_t H, float* __restrict__ pts) {
  __shared__ float stage[256 * 3];
  const uint32_t step = step_dev ? (uint32_t)*step_dev : step_arg;   // device counter: graph replay
  int64_t base = (int64_t)blockIdx.x * 256;
  int64_t i = base + threadIdx.x;
  float x[3] = {0.f, 0.f, 0.f};
  if (i < n) {
    uint64_t gi = (uint64_t)(first + i);
    uint4 a = philox_ctr(seed, 2 * gi, step, (uint32_t)kind);
    uint4 b = philox_ctr(seed, 2 * gi + 1, step, (uint32_t)kind);
    uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const int64_t L = kLattice;
    if (kind == NBM_POINTS_INTERIOR) {
      uint64_t M1 = (uint64_t)(2 * (L - H)) + 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        uint64_t W = (uint64_t)w[2 * c] | ((uint64_t)w[2 * c + 1] << 32);
        int64_t m = (int64_t)__umul64hi(W, M1);
        x[c] = (float)(m - (L - H)) * 0x1p-24f;
      }
    } else {
      uint32_t f = __umulhi(w[6], 6u);
      int axis = (int)(f >> 1);
      int slot = 0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (c == axis) {
          x[c] = (f & 1u) ? -1.0f : 1.0f;
        } else {
          uint64_t W = (uint64_t)w[2 * slot] | ((uint64_t)w[2 * slot + 1] << 32);
          int64_t m = (int64_t)__umul64hi(W, (uint64_t)(2 * L) + 1);
          x[c] = (float)(m - L) * 0x1p-24f;
          ++slot;
        }
      }
    }
  }
  stage[3 * threadIdx.x + 0] = x[0];
  stage[3 * threadIdx.x + 1] = x[1];
  stage[3 * threadIdx.x + 2] = x[2];
  __syncthreads();
  int64_t lim = (n - base) * 3;
  for (int t = threadIdx.x; t < 256 * 3; t += 256)
    if (t < lim) pts[base * 3 + t] = stage[t];
}

cudaError_t launch_sample(int kind, uint64_t seed, uint64_t step, const int64_t* step_dev, int64_t first,
                          int64_t n, int64_t H, float* pts, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  k_sample<<<(unsigned)blocks, 256, 0, s>>>(kind, seed, (uint32_t)step, step_dev, first, n, H, pts);
  return cudaGetLastError();
}

// ---- Xavier / Glorot-uniform init (G11) ----
struct InitTable {
  int n;
  int sine;                        // sine nets: +-sqrt(6/fan_in), else Glorot (G11)
  int64_t off[2 * kMaxLayers];     // theta offset of the layer block
  int64_t ebase[2 * kMaxLayers];   // running weight-element index at the block start
  int fi[2 * kMaxLayers], fo[2 * kMaxLayers];
};

__global__ void k_init(InitTable t, int64_t P, uint64_t seed, float* __restrict__ theta) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  int l = 0;
  while (l + 1 < t.n && i >= t.off[l + 1]) ++l;
  int64_t r = i - t.off[l];
  int64_t nw = (int64_t)t.fi[l] * t.fo[l];
  if (r >= nw) { theta[i] = 0.0f; return; }          // bias
  uint64_t e = (uint64_t)(t.ebase[l] + r);
  uint4 w = philox_ctr(seed, e >> 2, 0u, 2u);
  uint32_t word = (e & 3) == 0 ? w.x : (e & 3) == 1 ? w.y : (e & 3) == 2 ? w.z : w.w;
  float u = (float)(word >> 8) * 0x1p-24f;
  float amp = __fsqrt_rn(__fdiv_rn(6.0f, (float)(t.sine ? t.fi[l] : t.fi[l] + t.fo[l])));
  theta[i] = __fmul_rn(amp, __fsub_rn(__fmul_rn(2.0f, u), 1.0f));
}

cudaError_t launch_init_params(const ArchInfo& a, uint64_t seed, float* theta, cudaStream_t s) {
  InitTable t{};
  int64_t off = 0, e = 0;
  int k = 0;
  for (int net = 0; net < a.n_nets; ++net)
    for (int l = 1; l < a.n_layers; ++l, ++k) {
      t.off[k] = off;
      t.ebase[k] = e;
      t.fi[k] = a.sizes[l - 1];
      t.fo[k] = a.sizes[l];
      off += (int64_t)t.fi[k] * t.fo[k] + t.fo[k];
      e += (int64_t)t.fi[k] * t.fo[k];
    }
  t.n = k;
  t.sine = a.act == NBM_ACT_SINE ? 1 : 0;
  k_init<<<(unsigned)((off + 255) / 256), 256, 0, s>>>(t, off, seed, theta);
  return cudaGetLastError();
}

// ---- K4a Adam (G19).  Each op is one IEEE fp32 rounding in the written order. ----
__global__ void k_adam(int64_t P, float* __restrict__ th, float* __restrict__ m,
                       float* __restrict__ v, const float* __restrict__ g, float lr, float b1,
                       float b2, float eps, float bc1, float bc2, const float* __restrict__ bc_dev) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  if (bc_dev) {   // bias corrections of the device step counter (k_adam_prep)
    bc1 = bc_dev[0];
    bc2 = bc_dev[1];
  }
  float ob1 = __fsub_rn(1.0f, b1), ob2 = __fsub_rn(1.0f, b2);
  float gi = g[i];
  float mi = __fadd_rn(__fmul_rn(b1, m[i]), __fmul_rn(ob1, gi));
  float vi = __fadd_rn(__fmul_rn(b2, v[i]), __fmul_rn(ob2, __fmul_rn(gi, gi)));
  m[i] = mi;
  v[i] = vi;
  float mh = __fdiv_rn(mi, bc1), vh = __fdiv_rn(vi, bc2);
  float den = __fadd_rn(__fsqrt_rn(vh), eps);
  th[i] = __fsub_rn(th[i], __fdiv_rn(__fmul_rn(lr, mh), den));
}

cudaError_t launch_adam(int64_t P, float* theta, float* m, float* v, const float* g, float lr,
                        float b1, float b2, float eps, float bc1, float bc2, cudaStream_t s) {
  if (P <= 0) return cudaSuccess;
  k_adam<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(P, theta, m, v, g, lr, b1, b2, eps, bc1, bc2, nullptr);
  return cudaGetLastError();
}

// Device-counter variant (CUDA-graph replay): t = *t_dev + 1 (1-based step), the same fp32 bias
// corrections as the host path (1 - b^t in fp64, rounded once), then *t_dev = t.
__global__ void k_adam_prep(int64_t* __restrict__ t_dev, float b1, float b2, float* __restrict__ bc) {
  const int64_t t = *t_dev + 1;
  bc[0] = (float)(1.0 - pow((double)b1, (double)t));
  bc[1] = (float)(1.0 - pow((double)b2, (double)t));
  *t_dev = t;
}

cudaError_t launch_adam_dev(int64_t P, float* theta, float* m, float* v, const float* g, float lr, float b1,
                            float b2, float eps, int64_t* t_dev, float* bc, cudaStream_t s) {
  k_adam_prep<<<1, 1, 0, s>>>(t_dev, b1, b2, bc);
  if (P <= 0) return cudaGetLastError();
  k_adam<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(P, theta, m, v, g, lr, b1, b2, eps, 1.0f, 1.0f, bc);
  return cudaGetLastError();
}

}  // namespace nbm
