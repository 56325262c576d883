// mlp_fp32w.cu -- K3fw: the fused fp32 MLP forward -> residual epilogue -> backward kernel
// for wide hidden layers (W = 128, 256; config 5 in fp32, G15: IEEE fp32 with an accurate
// tanhf).  Same per-tile algorithm as K3f (mlp_fp32.cu), re-shaped for
// widths whose weights (64-256 KB per matrix) and dW (as much per layer) do not fit on chip:
//   * tiles of R rows (R = 32 at W = 256: 4 stencil points x 7 = 28 rows; R = 64 at W = 128:
//     9 points = 63 rows), all activations h_1..h_NH of the tile in shared memory;
//   * hidden weights streamed from an L2-resident fp32 image in K-slices of 32 rows through a
//     2-deep cp.async ring (forward: W_l^T [i][o], dH: W_l [o][i]; both read as [k][n]); the
//     first slice of the next GEMM is in flight during the current one;
//   * GEMMs register-tiled 8 rows x 4 columns per thread (A broadcast, B float4 per lane);
//   * dW_l = G_l^T h_{l-1} over the tile's rows in 8 x 4 blocks, flushed per tile with
//     red.global.add.v4.f32 into one of `nrep` gradient replicas (this width's FFMA time per
//     tile is ~75 us, so the per-tile flush is ~10 GB/s per SM); the small gradients (layer 1,
//     biases, output layer) accumulate in shared memory and are flushed once per CTA.
// The replica sum (K4r, k_reduce_rep) runs in fixed replica order; the order of the L2
// reductions is not fixed, so this path is deterministic within tolerance only (G21).
#include <math.h>

#include "nbm_internal.cuh"
#include "stab.cuh"
#include "tc_ptx.cuh"   // NBM_CHECK (bounds-checked builds)

namespace nbm {

namespace {

constexpr int kThr = 256;   // 8 warps
constexpr int KS = 32;      // K-slice depth of the streamed weights

template <int W, int NH>
struct FW {
  static constexpr int CG = W / 128;          // warps across the columns (32 lanes x 4 columns)
  static constexpr int RG = 8 / CG;           // row groups of 8 rows
  static constexpr int R = RG * 8;            // tile rows
  static constexpr int PT = (R - 1) / 7;      // stencil points per tile
  static constexpr int NS = W / KS;           // slices per GEMM
  static constexpr int NHH = NH - 1;
  static constexpr int TPR = kThr / R;        // threads per row (output layer)
  // shared memory carve (floats)
  static constexpr int oAct = 0;                        // [NH][R][W]
  static constexpr int oSl = oAct + NH * R * W;         // [2][KS][W]
  static constexpr int oW1 = oSl + 2 * KS * W;          // [W][3]
  static constexpr int oB = oW1 + 3 * W;                // [NH][W]
  static constexpr int oWo = oB + NH * W;               // [W] + bo
  static constexpr int oX = oWo + W + 4;                // [R][4]
  static constexpr int oU = oX + 4 * R;                 // [R]
  static constexpr int oUb = oU + R;                    // [R]
  static constexpr int oAux = oUb + R;                  // [R]
  static constexpr int oItem = oAux + R;                // int [R]
  static constexpr int oAW1 = oItem + R;                // [W][3]  accumulated gradients
  static constexpr int oAB = oAW1 + 3 * W;              // [NH][W]
  static constexpr int oAWo = oAB + NH * W;             // [W] + bo
  static constexpr int oRed = oAWo + W + 4;             // [4][kThr] reduction scratch
  static constexpr int total = oRed + 4 * kThr;
  static constexpr size_t bytes = sizeof(float) * total;
  static_assert(bytes <= 232448, "shared memory");
  static_assert(R * 4 * TPR == 4 * kThr, "output-layer mapping");
  // theta offsets within one network (G17)
  static constexpr int64_t tW1 = 0, tB1 = 3 * W;
  __host__ __device__ static constexpr int64_t tWl(int l) { return 4 * W + (int64_t)(l - 2) * (W * W + W); }
  __host__ __device__ static constexpr int64_t tBl(int l) { return tWl(l) + W * W; }
  static constexpr int64_t tWo = 4 * W + (int64_t)NHH * (W * W + W);
  static constexpr int64_t tBo = tWo + W;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

}  // namespace

// STAB: stencil tiles in the stable difference form (G27; training pass): R / 8 points per tile
template <int W, int NH, bool TRAIN, bool STAB = false>
__global__ void __launch_bounds__(kThr, 1) k_mlp_fp32w(const MlpParams prm, const float* __restrict__ wimg,
                                                        float* __restrict__ rep, int nrep) {
  using L = FW<W, NH>;
  static_assert(!STAB || TRAIN, "stable form: training pass");
  constexpr int R = L::R, NS = L::NS, NHH = L::NHH;
  constexpr int PT = STAB ? R / 8 : L::PT;   // stencil points per tile
  extern __shared__ __align__(16) float sm[];
  float* sAct = sm + L::oAct;
  float* sSl = sm + L::oSl;
  float* sW1 = sm + L::oW1;
  float* sBias = sm + L::oB;
  float* sWo = sm + L::oWo;
  float* sX = sm + L::oX;
  float* sU = sm + L::oU;
  float* sUb = sm + L::oUb;
  float* sAux = sm + L::oAux;
  int* sItem = reinterpret_cast<int*>(sm + L::oItem);
  float* sAW1 = sm + L::oAW1;
  float* sAB = sm + L::oAB;
  float* sAWo = sm + L::oAWo;
  float* sRed = sm + L::oRed;
  __shared__ int segTiles[kNumSeg], segCnt[kNumSeg], segStart[kNumSeg];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = (warp / L::CG) * 8, c0 = ((warp % L::CG) * 32 + lane) * 4;   // GEMM block
  if (tid < kNumSeg) {
    const int c = prm.counts[prm.cnt_slot[tid]];
    segCnt[tid] = c;
    segStart[tid] = prm.start_slot[tid] >= 0 ? prm.counts[prm.start_slot[tid]] : 0;
    const int per = prm.seg.kind[tid] == kSegStencil ? PT : R;
    segTiles[tid] = (c + per - 1) / per;
  }
  __syncthreads();
  int firstTile[kNumSeg + 1];
  int total = 0;
#pragma unroll
  for (int s = 0; s < kNumSeg; ++s) { firstTile[s] = total; total += segTiles[s]; }
  firstTile[kNumSeg] = total;
  const int G = gridDim.x, cta = blockIdx.x;
  const int t0 = (int)((int64_t)total * cta / G), t1 = (int)((int64_t)total * (cta + 1) / G);
  float* myRep = rep + (int64_t)(cta % nrep) * 2 * prm.p_stride;
  NBM_CHECK((int64_t)(cta % nrep + 1) * 2 * prm.p_stride <= prm.rep_len);

  // ---- weight stream: slices of [KS][W] through a 2-deep ring ----
  const uint32_t slBase = (uint32_t)__cvta_generic_to_shared(sSl);
  int cur = 0;                    // ring slot holding (or receiving) the current slice
  const float* primed = nullptr;  // image whose slice 0 is in flight into slot `cur`
  auto issue = [&](const float* img, int s, int slot) {
    const float* src = img + (int64_t)s * KS * W;
    const uint32_t dst = slBase + (uint32_t)(slot * KS * W * 4);
#pragma unroll
    for (int q = tid; q < KS * W / 4; q += kThr) cp_async16(dst + q * 16, src + 4 * q);
  };
  auto img_of = [&](int net, int l, int dir) -> const float* {   // dir 0: W_l^T [i][o], 1: W_l [o][i]
    return wimg + (((int64_t)net * NHH + (l - 2)) * 2 + dir) * W * W;
  };
  // acc[8][4] = A[r0..r0+7][:] * B[:][c0..c0+3], A [R][W] in shared memory, B streamed from img
  auto gemm = [&](const float* A, const float* img, const float* next, float (&acc)[8][4]) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = 0.0f;
    if (primed != img) {
      if (primed) {   // a different image's first slice is in flight into `cur`: drain it
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
      }
      issue(img, 0, cur);
      cp_commit();
    }
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
      if (s + 1 < NS) issue(img, s + 1, cur ^ 1);
      else if (next) issue(next, 0, cur ^ 1);
      cp_commit();
      cp_wait1();
      __syncthreads();
      const float* ws = sSl + cur * KS * W;
#pragma unroll 2
      for (int k = 0; k < KS; k += 4) {
        float4 a[8], w[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4*>(A + (r0 + i) * W + s * KS + k);
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const float4*>(ws + (k + q) * W + c0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float av[4] = {a[i].x, a[i].y, a[i].z, a[i].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[i][0] = fmaf(av[q], w[q].x, acc[i][0]);
            acc[i][1] = fmaf(av[q], w[q].y, acc[i][1]);
            acc[i][2] = fmaf(av[q], w[q].z, acc[i][2]);
            acc[i][3] = fmaf(av[q], w[q].w, acc[i][3]);
          }
        }
      }
      __syncthreads();
      cur ^= 1;
    }
    primed = next;
  };
  // column sums over the tile's rows (fixed order): acc[col] += sum_r X[r][col] * (wr ? wr[r] : 1)
  auto colsum = [&](const float* X, const float* wr, float* accv, bool centre_only = false) {
    constexpr int parts = kThr / W > 0 ? kThr / W : 1;
    const int col = tid % W, part = tid / W;
    if (part < parts) {
      float s = 0.0f;
      for (int r = part * (R / parts); r < (part + 1) * (R / parts); ++r)
        if (!centre_only || (r & 7) == 0) s = wr ? fmaf(wr[r], X[r * W + col], s) : s + X[r * W + col];
      sRed[part * W + col] = s;
    }
    __syncthreads();
    if (tid < W) {
      float t = 0.0f;
      for (int p = 0; p < parts; ++p) t += sRed[p * W + tid];
      accv[tid] += t;
    }
    __syncthreads();
  };
  // dW_l[o][i] += sum_r G[r][o] H[r][i] over the tile, flushed into the replica
  auto dw_flush = [&](const float* Gs, const float* Hs, int l, int net) {
    float* out = myRep + (int64_t)net * prm.p_stride + L::tWl(l);
#pragma unroll 1
    for (int q = warp; q < (W / 8) * L::CG; q += 8) {
      const int ob = (q / L::CG) * 8, ic = ((q % L::CG) * 32 + lane) * 4;
      float d[8][4];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) d[a][c] = 0.0f;
#pragma unroll 4
      for (int r = 0; r < R; ++r) {
        const float4 g0 = *reinterpret_cast<const float4*>(Gs + r * W + ob);
        const float4 g1 = *reinterpret_cast<const float4*>(Gs + r * W + ob + 4);
        const float4 h = *reinterpret_cast<const float4*>(Hs + r * W + ic);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          d[a][0] = fmaf(gv[a], h.x, d[a][0]);
          d[a][1] = fmaf(gv[a], h.y, d[a][1]);
          d[a][2] = fmaf(gv[a], h.z, d[a][2]);
          d[a][3] = fmaf(gv[a], h.w, d[a][3]);
        }
      }
#pragma unroll
      for (int a = 0; a < 8; ++a) red4(out + (int64_t)(ob + a) * W + ic, d[a][0], d[a][1], d[a][2], d[a][3]);
    }
  };
  auto zero_small = [&]() {
    for (int i = tid; i < 3 * W + NH * W + W + 4; i += kThr) sAW1[i] = 0.0f;   // AW1, AB, AWo contiguous
  };
  auto flush_small = [&](int net) {
    float* out = myRep + (int64_t)net * prm.p_stride;
    for (int i = tid; i < 3 * W; i += kThr) atomicAdd(out + L::tW1 + i, sAW1[i]);
    for (int i = tid; i < W; i += kThr) {
      atomicAdd(out + L::tB1 + i, sAB[i]);
      for (int l = 2; l <= NH; ++l) atomicAdd(out + L::tBl(l) + i, sAB[(l - 1) * W + i]);
      atomicAdd(out + L::tWo + i, sAWo[i]);
    }
    if (tid == 0) atomicAdd(out + L::tBo, sAWo[W]);
  };
  auto load_net = [&](int net) {
    const float* th = prm.theta + (int64_t)net * prm.p_net;
    for (int i = tid; i < 3 * W; i += kThr) sW1[i] = th[L::tW1 + i];
    for (int i = tid; i < W; i += kThr) {
      sBias[i] = th[L::tB1 + i];
      for (int l = 2; l <= NH; ++l) sBias[(l - 1) * W + i] = th[L::tBl(l) + i];
      sWo[i] = th[L::tWo + i];
    }
    if (tid == 0) sWo[W] = th[L::tBo];
  };
  auto net_of_tile = [&](int t) {
    int s = 0;
    while (t >= firstTile[s + 1]) ++s;
    return prm.seg.net[s];
  };

  double lossAcc = 0.0;
  int curNet = -1;
  int seg = 0;
  for (int t = t0; t < t1; ++t) {
    while (t >= firstTile[seg + 1]) ++seg;
    const int kind = prm.seg.kind[seg], net = prm.seg.net[seg];
    const int per = kind == kSegStencil ? PT : R;
    const int first = (t - firstTile[seg]) * per;
    const int nvalid = min(per, segCnt[seg] - first);
    const int nextNet = t + 1 < t1 ? net_of_tile(t + 1) : -1;
    const bool stab = STAB && kind == kSegStencil;   // block-uniform
    if (net != curNet) {
      __syncthreads();
      if (TRAIN && curNet >= 0) flush_small(curNet);
      __syncthreads();
      load_net(net);
      if (TRAIN) zero_small();
      curNet = net;
    }
    // ---- gather the tile's items and rows (x, aux) ----
    const int* items = prm.seg.items[seg] + segStart[seg];
    if (tid < per) {
      const int it = tid < nvalid ? item_at(prm.seg, seg, items, first + tid) : -1;
      sItem[tid] = it;
      float a = 0.0f;
      if (it >= 0) a = prm.aux_by_item[seg] ? prm.seg.aux[seg][it] : prm.seg.aux[seg][segStart[seg] + first + tid];
      sAux[tid] = a;
    }
    __syncthreads();
    if (tid < R) {
      float x0 = 0.0f, x1 = 0.0f, x2 = 0.0f;
      if (stab) {   // row 8k + jr: x, h e_1..3 (P_d), 0 (Q_d, pad)
        const int k = tid >> 3, jr = tid & 7;
        if (k < nvalid && jr == 0) {
          const float* src = prm.seg.src[seg] + 3 * (int64_t)sItem[k];
          x0 = src[0]; x1 = src[1]; x2 = src[2];
        } else if (k < nvalid && jr < 4) {
          if (jr == 1) x0 = prm.h; else if (jr == 2) x1 = prm.h; else x2 = prm.h;
        }
      } else if (kind == kSegStencil) {
        const int j = tid / PT, p = tid - j * PT;
        if (j < 7 && p < nvalid) {
          const float* src = prm.seg.src[seg] + 3 * (int64_t)sItem[p];
          x0 = src[0]; x1 = src[1]; x2 = src[2];
          if (j > 0) {   // arms +x, -x, +y, -y, +z, -z (exact on the lattice)
            const float hs = (j & 1) ? prm.h : -prm.h;
            if (j <= 2) x0 = __fadd_rn(x0, hs); else if (j <= 4) x1 = __fadd_rn(x1, hs); else x2 = __fadd_rn(x2, hs);
          }
        }
      } else if (tid < nvalid) {
        const float* src = prm.seg.src[seg] + 3 * (int64_t)sItem[tid];
        x0 = src[0]; x1 = src[1]; x2 = src[2];
      }
      sX[4 * tid] = x0; sX[4 * tid + 1] = x1; sX[4 * tid + 2] = x2;
    }
    __syncthreads();
    // ---- layer 1 (K = 3) ----
    for (int e = tid; e < R * W; e += kThr) {
      const int r = e / W, n = e % W;
      const float b = (!stab || (r & 7) == 0) ? sBias[n] : 0.0f;   // stable form: bias on the centre rows
      const float z = fmaf(sW1[3 * n + 2], sX[4 * r + 2], fmaf(sW1[3 * n + 1], sX[4 * r + 1], fmaf(sW1[3 * n], sX[4 * r], b)));
      sAct[e] = (STAB && stab) ? z : tanhf(z);
    }
    __syncthreads();
    if (STAB && stab) {
      stab::fwd_pass_f32<W, W, R / 8, kThr>(sAct, tid);
      __syncthreads();
    }
    // ---- hidden layers: h_l = tanh(h_{l-1} W_l^T + b_l) ----
#pragma unroll 1
    for (int l = 2; l <= NH; ++l) {
      const float* next = l < NH ? img_of(net, l + 1, 0) : TRAIN ? img_of(net, NH, 1)
                                                                : (nextNet >= 0 ? img_of(nextNet, 2, 0) : nullptr);
      float acc[8][4];
      gemm(sAct + (l - 2) * R * W, img_of(net, l, 0), next, acc);
      const float4 bv = *reinterpret_cast<const float4*>(sBias + (l - 1) * W + c0);
      float* out = sAct + (l - 1) * R * W;
      if (STAB && stab) {   // raw pre-activations (bias on the centre rows), then the stable map
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float m = ((r0 + i) & 7) == 0 ? 1.0f : 0.0f;
          *reinterpret_cast<float4*>(out + (r0 + i) * W + c0) =
              make_float4(fmaf(m, bv.x, acc[i][0]), fmaf(m, bv.y, acc[i][1]), fmaf(m, bv.z, acc[i][2]), fmaf(m, bv.w, acc[i][3]));
        }
        __syncthreads();
        stab::fwd_pass_f32<W, W, R / 8, kThr>(out, tid);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(out + (r0 + i) * W + c0) =
              make_float4(tanhf(acc[i][0] + bv.x), tanhf(acc[i][1] + bv.y), tanhf(acc[i][2] + bv.z), tanhf(acc[i][3] + bv.w));
      }
      __syncthreads();
    }
    // ---- output layer u = wo . h_NH + bo ----
    float* hTop = sAct + (NH - 1) * R * W;
    {
      const int r = tid / L::TPR, q = tid % L::TPR;
      constexpr int span = W / L::TPR;
      float s = 0.0f;
      for (int k = q * span; k < (q + 1) * span; ++k) s = fmaf(sWo[k], hTop[r * W + k], s);
#pragma unroll
      for (int o = 1; o < L::TPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (q == 0) sU[r] = (!stab || (r & 7) == 0) ? s + sWo[W] : s;   // differences carry no output bias
    }
    __syncthreads();
    if (!TRAIN) {
      if (tid < nvalid) prm.u_out[sItem[tid]] = sU[tid];
      __syncthreads();
      continue;
    }
    // ---- residual epilogue -> cotangents (S4) ----
    if (STAB && stab) {   // r = c_c u + c_hat sum_d DU_d - b/d (G27); cotangents c_c 2r/N, c_hat 2r/N (Q_d)
      if (tid < R) {
        const int k = tid >> 3, jr = tid & 7;
        float ub = 0.0f;
        if (k < nvalid) {
          const float chat = prm.seg.chat[seg], cc = prm.seg.ccen[seg];
          const float du = (sU[8 * k + 4] + sU[8 * k + 5]) + sU[8 * k + 6];
          const float r = fmaf(cc, sU[8 * k], chat * du) - sAux[k];
          if (jr == 0) lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;
          const float rc = prm.two_over_n * r;
          ub = jr == 0 ? rc * cc : (jr >= 4 && jr < 7) ? rc * chat : 0.0f;
        }
        sUb[tid] = ub;
      }
    } else if (kind == kSegStencil) {
      if (tid < PT) {
        float r = 0.0f;
        float cj[6];   // arm coefficients c_j / d: uniform (constant beta) or per point (variable mu)
#pragma unroll
        for (int j = 0; j < 6; ++j) cj[j] = prm.seg.chat[seg];
        if (prm.pcoef && tid < nvalid) {
          const float* pc = prm.pcoef + 6 * (int64_t)sItem[tid];
#pragma unroll
          for (int j = 0; j < 6; ++j) cj[j] = pc[j];
        }
        if (tid < nvalid) {
          float acc = sU[tid];
#pragma unroll
          for (int j = 1; j < 7; ++j) acc = fmaf(cj[j - 1], sU[j * PT + tid], acc);
          r = acc - sAux[tid];
          lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;   // r^2 / N
        }
        const float rc = prm.two_over_n * r;
        sUb[tid] = rc;
#pragma unroll
        for (int j = 1; j < 7; ++j) sUb[j * PT + tid] = rc * cj[j - 1];
      } else if (tid >= 7 * PT && tid < R) {
        sUb[tid] = 0.0f;
      }
    } else if (tid < R) {
      float ub = 0.0f;
      if (tid < nvalid) {
        if (kind == kSegBRows) {
          const float e = sU[tid] - sAux[tid];
          ub = prm.seg.a[seg] * e;
          lossAcc += 0.5 * (double)prm.seg.a[seg] * (double)e * (double)e;
        } else {
          ub = sAux[tid];
        }
      }
      sUb[tid] = ub;
    }
    __syncthreads();
    // ---- backward (S5): output layer, then G_NH = ub wo (1 - h_NH^2) in place ----
    colsum(hTop, sUb, sAWo);   // dwo += sum_r ub h_NH
    if (tid < 32) {
      float b = 0.0f;
      for (int r = tid; r < R; r += 32)
        if (!stab || (r & 7) == 0) b += sUb[r];
#pragma unroll
      for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
      if (tid == 0) sAWo[W] += b;
    }
    if (STAB && stab) {
      __syncthreads();   // dwo has read h_NH
      stab::bwd_pass_f32<W, W, R / 8, kThr>(nullptr, hTop, sUb, sWo, tid);
    } else {
      for (int e = tid; e < R * W; e += kThr) {
        const int r = e / W, n = e % W;
        const float hv = hTop[e];
        hTop[e] = sUb[r] * sWo[n] * (1.0f - hv * hv);
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int l = NH; l >= 2; --l) {   // G_l in act[l-1], h_{l-1} in act[l-2]
      float* Gl = sAct + (l - 1) * R * W;
      float* Hp = sAct + (l - 2) * R * W;
      dw_flush(Gl, Hp, l, net);
      colsum(Gl, nullptr, sAB + (l - 1) * W, STAB && stab);   // db_l (contains __syncthreads)
      const float* next = l > 2 ? img_of(net, l - 1, 1) : (nextNet >= 0 ? img_of(nextNet, 2, 0) : nullptr);
      float acc[8][4];
      gemm(Gl, img_of(net, l, 1), next, acc);   // (G_l W_l)[r][i]
      if (STAB && stab) {   // the products over the consumed G_l, then the backward map -> Hp
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(Gl + (r0 + i) * W + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        __syncthreads();
        stab::bwd_pass_f32<W, W, R / 8, kThr>(Gl, Hp, nullptr, nullptr, tid);
        __syncthreads();
        continue;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float* p = Hp + (r0 + i) * W + c0;
        const float4 hv = *reinterpret_cast<const float4*>(p);
        *reinterpret_cast<float4*>(p) = make_float4(acc[i][0] * (1.0f - hv.x * hv.x), acc[i][1] * (1.0f - hv.y * hv.y),
                                                    acc[i][2] * (1.0f - hv.z * hv.z), acc[i][3] * (1.0f - hv.w * hv.w));
      }
      __syncthreads();
    }
    {  // layer 1: dW1[n][c] += sum_r G1[r][n] x[r][c]; db1 += sum_r G1[r][n]
      for (int n = tid; n < W; n += kThr) {
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, sb = 0.f;
        for (int r = 0; r < R; ++r) {
          const float g = sAct[r * W + n];
          s0 = fmaf(g, sX[4 * r], s0);
          s1 = fmaf(g, sX[4 * r + 1], s1);
          s2 = fmaf(g, sX[4 * r + 2], s2);
          if (!stab || (r & 7) == 0) sb += g;
        }
        sAW1[3 * n] += s0;
        sAW1[3 * n + 1] += s1;
        sAW1[3 * n + 2] += s2;
        sAB[n] += sb;
      }
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (!TRAIN) return;
  __syncthreads();
  if (curNet >= 0) flush_small(curNet);
  for (int o = 16; o; o >>= 1) lossAcc += __shfl_xor_sync(0xffffffffu, lossAcc, o);
  __shared__ double wl[kThr / 32];
  if (lane == 0) wl[warp] = lossAcc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThr / 32; ++w) s += wl[w];
    prm.lpart[cta] = s;
  }
}

template <int W, int NH, bool TRAIN, bool STAB = false>
static cudaError_t launch_fw_t(const MlpParams& p, const float* wimg, float* rep, int nrep, int grid, cudaStream_t s) {
  using L = FW<W, NH>;
  auto kern = k_mlp_fp32w<W, NH, TRAIN, STAB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, (const void*)kern, (int)L::bytes); e != cudaSuccess) return e;
  kern<<<grid, kThr, L::bytes, s>>>(p, wimg, rep, nrep);
  return cudaGetLastError();
}

int mlp_fp32w_supported(int width, int n_hidden) {
  return (width == 128 || width == 256) && n_hidden >= 2 && n_hidden <= 4;
}

cudaError_t launch_mlp_fp32w(int width, int n_hidden, bool train, bool stable, const MlpParams& p, const float* wimg,
                             float* rep, int nrep, int grid, cudaStream_t s) {
  if (nrep < 1) return cudaErrorInvalidValue;
  if (stable && train) {
#define NBM_FW_SCASES(WW)                                                          \
  switch (n_hidden) {                                                              \
    case 2: return launch_fw_t<WW, 2, true, true>(p, wimg, rep, nrep, grid, s);    \
    case 3: return launch_fw_t<WW, 3, true, true>(p, wimg, rep, nrep, grid, s);    \
    case 4: return launch_fw_t<WW, 4, true, true>(p, wimg, rep, nrep, grid, s);    \
  }
    if (width == 256) { NBM_FW_SCASES(256) }
    if (width == 128) { NBM_FW_SCASES(128) }
#undef NBM_FW_SCASES
    return cudaErrorInvalidValue;
  }
#define NBM_FW_CASES(WW)                                                                              \
  switch (n_hidden) {                                                                                 \
    case 2: return train ? launch_fw_t<WW, 2, true>(p, wimg, rep, nrep, grid, s)                      \
                         : launch_fw_t<WW, 2, false>(p, wimg, rep, nrep, grid, s);                    \
    case 3: return train ? launch_fw_t<WW, 3, true>(p, wimg, rep, nrep, grid, s)                      \
                         : launch_fw_t<WW, 3, false>(p, wimg, rep, nrep, grid, s);                    \
    case 4: return train ? launch_fw_t<WW, 4, true>(p, wimg, rep, nrep, grid, s)                      \
                         : launch_fw_t<WW, 4, false>(p, wimg, rep, nrep, grid, s);                    \
  }
  if (width == 256) { NBM_FW_CASES(256) }
  if (width == 128) { NBM_FW_CASES(128) }
#undef NBM_FW_CASES
  return cudaErrorInvalidValue;
}

// fp32 weight images of the hidden layers, 16-B aligned: [net][l][dir][W*W],
// dir 0 = W_l^T ([i][o], forward K-slices), dir 1 = W_l ([o][i], dH K-slices)
__global__ void k_pack_fp32w(const float* __restrict__ theta, int64_t p_net, int W, int nhh, int n_nets,
                             float* __restrict__ img) {
  const int64_t total = (int64_t)n_nets * nhh * W * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / ((int64_t)W * W);
    const int net = (int)(m / nhh), l = (int)(m % nhh) + 2;
    const int r = (int)(e % ((int64_t)W * W)), o = r / W, i = r % W;
    const float v = theta[(int64_t)net * p_net + 4 * W + (int64_t)(l - 2) * ((int64_t)W * W + W) + r];
    img[(m * 2 + 0) * W * W + (int64_t)i * W + o] = v;
    img[(m * 2 + 1) * W * W + r] = v;
  }
}

cudaError_t launch_pack_fp32w(const ArchInfo& a, const float* theta, float* img, cudaStream_t s) {
  const int nhh = a.n_hidden - 1;
  if (nhh <= 0) return cudaSuccess;
  k_pack_fp32w<<<148 * 4, 256, 0, s>>>(theta, a.p_net, a.width, nhh, a.n_nets, img);
  return cudaGetLastError();
}

}  // namespace nbm
