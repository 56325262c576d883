// stab.cuh -- the stable stencil form's per-element maps (G27),
// shared by the tensor-core kernels K3t (mlp_tc.cu) and K3w (mlp_w256.cu).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace nbm {
namespace stab {

__device__ __forceinline__ float stab_tanh(float x) {   // MUFU tanh.approx.f32 (max rel. error 2^-10.99)
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- stable stencil evaluation (G27): difference propagation ----
// Row roles on a stencil tile (point k at rows 8k..8k+7, one lane octet of a warp): 0 the
// centre activation a, 1..3 the first differences P_d = a(x + h e_d) - a(x), 4..6 the second
// differences Q_d = a(x + h e_d) + a(x - h e_d) - 2 a(x), 7 padding (zero).
// tanh(d) - d: odd Taylor series to d^7 below 1/4 (truncation < 2e-5 relative, under the bf16
// rounding of the rows), MUFU tanh above (rare: |d| is O(h) on the difference rows).  Both are
// computed and selected: a branch per element would serialise the unrolled column loop
__device__ __forceinline__ float tanh_minus_id(float d) {
  const float d2 = d * d;
  const float s = fmaf(d2, fmaf(d2, -17.0f / 315.0f, 2.0f / 15.0f), -1.0f / 3.0f) * (d * d2);
  return fabsf(d) < 0.25f ? s : stab_tanh(d) - d;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// g(d) = tanh(z + d) - tanh(z) - (1 - t^2) d = s2 [(tanh d - d) - t tanh(d) d] / (1 + t tanh d)
// with s2 = 1 - t^2 (tanh addition theorem)
__device__ __forceinline__ float stab_g(float t, float s2, float d) {
  const float s = tanh_minus_id(d), x = t * (d + s);
  return s2 * fmaf(-x, d, s) * rcp_approx(1.0f + x);
}
// Role masks of a lane (0/1): the maps below are written branch-free (a select chain per element
// compiles to branches, which serialise the unrolled column loop and guard every shuffle)
struct StabRole {
  int base, pl, partner;
  float cC, cP, cQ, cPQ;
  __device__ __forceinline__ explicit StabRole(int lane) {
    const int jr = lane & 7;
    const bool isP = jr >= 1 && jr < 4, isQ = jr >= 4 && jr < 7;
    base = lane & ~7;
    pl = base + (isQ ? jr - 3 : jr);                         // the P_d lane of this row's axis
    partner = base + (isP ? jr + 3 : isQ ? jr - 3 : jr);     // P_d <-> Q_d
    cC = jr == 0 ? 1.0f : 0.0f;
    cP = isP ? 1.0f : 0.0f;
    cQ = isQ ? 1.0f : 0.0f;
    cPQ = cP + cQ;
  }
};
// forward map of one 32-column chunk: v = the row's pre-activation without bias (z - b for the
// centre, p_d, D_d); bl = the layer's bias.  a = tanh z, P = (1 - t^2) p + g(p),
// Q = (1 - t^2) D + g(p) + g(D - p).  t from MUFU tanh.approx as on the direct path: its
// 2^-11 error moves 1 - t^2 of saturated units by ~2^-10 absolute, below the bf16 rounding
// of the rows (the GPU results agree with the exact-tanh emulation, test_gpu_stable)
// (N = 32 columns, or 16 where register pressure demands it)
template <int N>
__device__ __forceinline__ void stab_fwd(float (&v)[N], const float* bl, int lane) {
  const StabRole R(lane);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float t = stab_tanh(__shfl_sync(0xffffffffu, v[j] + bl[j], R.base));
    const float s2 = fmaf(-t, t, 1.0f);
    const float pv = __shfl_sync(0xffffffffu, v[j], R.pl);
    const float g = stab_g(t, s2, fmaf(-R.cQ, pv, R.cPQ * v[j]));   // p, D - p; 0 on centre / pad
    const float gp = __shfl_sync(0xffffffffu, g, R.pl);
    v[j] = fmaf(R.cC, t, fmaf(R.cQ, gp, R.cPQ * fmaf(s2, v[j], g)));
  }
}
// backward map: v = upstream gradients of the row (g_a, g_P or g_Q), hq = the row's activation
// copy (t, P or Q).  With M = Q - P:  g_z = g_a (1 - t^2) - sum_d [g_P P (2t + P)
// + g_Q (2tQ + P^2 + M^2)],  g_p = g_P (1 - (t + P)^2) + g_Q (M - P)(2t + M + P),
// g_D = g_Q (1 - (t + M)^2)   (oracle/stable_stencil.py, pinned against the plain gradient)
template <int N>
__device__ __forceinline__ void stab_bwd(float (&v)[N], const float (&hq)[N], int lane) {
  const StabRole R(lane);
  const uint32_t qm = R.cQ != 0.0f ? 0xffffffffu : 0u;   // bit select (LOP3), not a branch
  auto sel = [qm](float a, float b) { return __uint_as_float((__float_as_uint(a) & qm) | (__float_as_uint(b) & ~qm)); };
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float t = __shfl_sync(0xffffffffu, hq[j], R.base);
    const float ho = __shfl_sync(0xffffffffu, hq[j], R.partner);
    const float go = __shfl_sync(0xffffffffu, v[j], R.partner);
    const float pv = sel(ho, hq[j]), qv = sel(hq[j], ho);
    const float gP = sel(go, v[j]), gQ = sel(v[j], go);
    const float m = qv - pv, t2 = t + t;
    const float cp = gP * pv * (t2 + pv), cq = gQ * fmaf(t2, qv, fmaf(pv, pv, m * m));
    float c = fmaf(R.cP, cp, R.cQ * cq);
    c += __shfl_xor_sync(0xffffffffu, c, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    const float tp = t + pv, tm = t + m;
    const float oC = fmaf(v[j], fmaf(-t, t, 1.0f), -c);
    const float oP = fmaf(gP, fmaf(-tp, tp, 1.0f), gQ * (m - pv) * (t2 + m + pv));
    const float oQ = gQ * fmaf(-tm, tm, 1.0f);
    v[j] = fmaf(R.cC, oC, fmaf(R.cP, oP, R.cQ * oQ));
  }
}

// ---- fp32 kernels (K3f, K3fw): one thread per (point, column) of a stencil tile in shared memory, rows 8k..8k+7 = centre, P_x, P_y, P_z, Q_x, Q_y, Q_z, pad (fp32-accurate
// maps: tanhf, the series of tanh d - d to d^11 below 1/4, IEEE division) ----
__device__ __forceinline__ float tanh_minus_id_f32(float d) {
  const float d2 = d * d;
  const float s = fmaf(d2, fmaf(d2, fmaf(d2, fmaf(d2, -1382.0f / 155925.0f, 62.0f / 2835.0f), -17.0f / 315.0f),
                                2.0f / 15.0f), -1.0f / 3.0f) * (d * d2);
  return s;   // |d| < 1/4 (stab_g_f32 branches above the cut)
}
// g(d) = tanh(z + d) - t - s2 d (t = tanh z, s2 = 1 - t^2) without cancellation.  Below the
// cut the tanh addition theorem form s2 [(tanh d - d) - t tanh(d) d] / (1 + x), x = t tanh d:
// there |x| <= |tanh d| < 1/4, so 1 + x lies in [0.75, 1.25] and the approximate division
// (reciprocal within 1 ulp) keeps g within 2 ulp.  At |d| >= 1/4 (rare) 1 + x can approach 0
// for saturated units, so g is formed directly, where nothing cancels at that size of d.
__device__ __forceinline__ float stab_g_f32(float z, float t, float s2, float d) {
  if (fabsf(d) >= 0.25f) return tanhf(z + d) - t - s2 * d;   // rare (a branch: tanhf is long)
  const float s = tanh_minus_id_f32(d), x = t * (d + s);
  return __fdividef(s2 * fmaf(-x, d, s), 1.0f + x);
}
// in place: z (bias included), p_d, D_d -> t = tanh z, P_d, Q_d
template <int W, int LDA, int NPTS, int NTHR>
__device__ void fwd_pass_f32(float* __restrict__ H, int tid) {
  for (int it = tid; it < NPTS * W; it += NTHR) {
    float* h = H + (it / W) * 8 * LDA + it % W;
    const float z = h[0], t = tanhf(z);
    const float s2 = (1.0f - t) * (1.0f + t);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float p = h[(1 + d) * LDA], D = h[(4 + d) * LDA];
      const float gp = stab_g_f32(z, t, s2, p), gm = stab_g_f32(z, t, s2, D - p);
      h[(1 + d) * LDA] = fmaf(s2, p, gp);
      h[(4 + d) * LDA] = fmaf(s2, D, gp) + gm;
    }
    h[0] = t;
    h[7 * LDA] = 0.0f;
  }
}
// G of the point's rows from the upstream gradients R (g_a, g_P, g_Q; R = null: the output
// layer's ub_row wo_col) and the activations H (t, P, Q), written over H
template <int W, int LDA, int NPTS, int NTHR>
__device__ void bwd_pass_f32(const float* __restrict__ R, float* __restrict__ H, const float* __restrict__ ub,
                             const float* __restrict__ wo, int tid) {
  for (int it = tid; it < NPTS * W; it += NTHR) {
    const int k = it / W, col = it % W;
    float* h = H + k * 8 * LDA + col;
    auto up = [&](int j) { return R ? R[(k * 8 + j) * LDA + col] : ub[k * 8 + j] * wo[col]; };
    const float t = h[0], t2 = t + t;
    float gz = up(0) * ((1.0f - t) * (1.0f + t));
    float gp[3], gd[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float P = h[(1 + d) * LDA], Q = h[(4 + d) * LDA], M = Q - P;
      const float gP = up(1 + d), gQ = up(4 + d);
      gz -= gP * P * (t2 + P) + gQ * fmaf(t2, Q, fmaf(P, P, M * M));
      const float tp = t + P, tm = t + M;
      gp[d] = fmaf(gP, (1.0f - tp) * (1.0f + tp), gQ * (M - P) * (t2 + M + P));
      gd[d] = gQ * ((1.0f - tm) * (1.0f + tm));
    }
    h[0] = gz;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      h[(1 + d) * LDA] = gp[d];
      h[(4 + d) * LDA] = gd[d];
    }
    h[7 * LDA] = 0.0f;
  }
}

}  // namespace stab
}  // namespace nbm
