// mlp_fp32.cu -- K3f: the fused MLP forward -> residual epilogue -> backward -> dW
// kernel in IEEE fp32 on the CUDA cores (configs 1, 2, 5-fp32; G15).
//
// One CTA (256 threads) processes a contiguous range of 128-row tiles of the
// segment table:
//   * stencil tile: 18 uncrossed points x 7 stencil vertices (126 rows, arm-major:
//     row = j*18 + p), all on one network ("neural networks can be evaluated
//     over vertices of any discretization stencils"; P:60 one network per side);
//   * row tile: 128 independent evaluations with an affine cotangent (boundary rows:
//     u_bar = a (u - g); crossed rows: u_bar given by the crossed pass).
// Per tile: layer 1 (K=3) -> hidden GEMMs (register-tiled FFMA from shared memory)
// -> output layer -> epilogue r = u0 + chat sum_j u_j - rhs_hat (r = M^-1 A u - M^-1 b,
// P:60), u_bar = (2/N) r chat_j -> backward GEMMs.  The hidden x hidden dW
// accumulate in registers across all the CTA's tiles and the small
// layers' grads in shared memory; each CTA writes one fp32 partial per network that
// K4r sums in fixed CTA order (deterministic, G21).
#include <math.h>

#include "nbm_internal.cuh"
#include "stab.cuh"
#include "tc_ptx.cuh"   // NBM_CHECK (bounds-checked builds)

namespace nbm {

// activation of the fp32 kernel: accurate tanhf (G15); NBM_F32_TANH_APPROX (timing experiments
// only, not a supported build) swaps in MUFU tanh.approx
#ifdef NBM_F32_TANH_APPROX
__device__ __forceinline__ float f32_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#else
__device__ __forceinline__ float f32_tanh(float x) { return tanhf(x); }
#endif

#ifndef NBM_F32_TILE
#define NBM_F32_TILE 64
#endif
// 64-row tiles with 256 threads run two CTAs per SM, so one CTA's barriers and load latencies
// overlap the other's FFMA work; 128-row tiles with 512 threads run one.
constexpr int kB = NBM_F32_TILE;     // rows per tile
constexpr int kPT = (kB - 1) / 7;    // points per stencil tile (9 -> 63 rows; 18 -> 126 rows)
constexpr int kThreads = 4 * kB;     // 8 or 16 warps
constexpr int kCtasPerSm = kB == 64 ? 2 : 1;
constexpr int kRT = kB / 32;         // GEMM rows per thread
constexpr int kHalves = kThreads / 256;   // dW row groups (summed at the flush)



template <int N> struct VecT;
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<4> { using T = float4; };

__device__ __forceinline__ void ldv(const float* p, float (&v)[4]) {
  float4 t = *reinterpret_cast<const float4*>(p);
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void ldv(const float* p, float (&v)[2]) {
  float2 t = *reinterpret_cast<const float2*>(p);
  v[0] = t.x; v[1] = t.y;
}
__device__ __forceinline__ void ldv(const float* p, float (&v)[1]) { v[0] = *p; }
__device__ __forceinline__ void ldv(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void stv(float* p, const float (&v)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void stv(float* p, const float (&v)[1]) { *p = v[0]; }
__device__ __forceinline__ void stv(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void stv(float* p, const float (&v)[2]) {
  *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
}

template <int W, int NH, bool SINE = false>
struct Layout {
  static constexpr int LDA = W + 4;              // padded row stride of activations
  static constexpr int LDW = W + 4;              // padded row stride of hidden weights
  static constexpr int TC = W / (kThreads / 32);   // GEMM columns per thread (rows: kRT)
  static constexpr int DB = W / 16;              // dW block per thread: DB x DB (16 x 16 blocks)
  static constexpr int NHH = NH - 1;             // hidden x hidden layers
  // shared-memory carve (floats)
  static constexpr int oW1 = 0;                          // [W][3]
  static constexpr int oB = oW1 + 4 * W;                 // [NH][W]
  static constexpr int oWh = oB + NH * W;                // [NHH][W][LDW]
  static constexpr int oWo = oWh + (NHH > 0 ? NHH : 0) * W * LDW;   // [W] + bo
  static constexpr int oAct = oWo + W + 4;               // [NH][kB][LDA]
  static constexpr int oX = oAct + NH * kB * LDA;        // [kB][4]
  static constexpr int oU = oX + 4 * kB;                 // [kB]
  static constexpr int oUb = oU + kB;                    // [kB]
  static constexpr int oRed = oUb + kB;                  // [4][256]
  static constexpr int oAW1 = oRed + 4 * kThreads;       // [W][3]
  static constexpr int oAB = oAW1 + 4 * W;               // [NH][W]
  static constexpr int oAWo = oAB + NH * W;              // [W] + bo
  static constexpr int oAux = oAWo + W + 4;              // [kB]
  static constexpr int oItem = oAux + kB;                // int [kB]
  static constexpr int oCos = (oItem + kB + 16 + 3) & ~3;   // sine: [NH][kB][LDA] cos(z_l) for act'
  static constexpr int total = oCos + (SINE ? NH * kB * LDA : 0);
  static constexpr size_t bytes = sizeof(float) * total;
  static_assert(bytes <= 232448, "shared memory");
  // theta offsets within one network (G17)
  static constexpr int64_t tW1 = 0, tB1 = 3 * W;
  __host__ __device__ static constexpr int64_t tWl(int l) { return 4 * W + (int64_t)(l - 2) * (W * W + W); }
  __host__ __device__ static constexpr int64_t tBl(int l) { return tWl(l) + W * W; }
  static constexpr int64_t tWo = 4 * W + (int64_t)NHH * (W * W + W);
  static constexpr int64_t tBo = tWo + W;
  static constexpr int64_t pnet = tBo + 1;
};

// Hout[b][n] = tanh(sum_k Hin[b][k] W[n][k] + bias[n]); thread = 8 rows x TC cols.
// raw (stable form, G27): Hout = the pre-activation, the bias on the centre rows (8k) only
template <int W, int NH, bool SINE = false>
__device__ __forceinline__ void fwd_gemm(const float* __restrict__ Hin, float* __restrict__ Hout,
                                         const float* __restrict__ Ws, const float* __restrict__ bias,
                                         int tid, float* __restrict__ CosOut = nullptr, bool raw = false) {
  using L = Layout<W, NH>;
  constexpr int TC = L::TC;
  const int tr = tid & 31, tc = tid >> 5;
  float acc[kRT][TC];
#pragma unroll
  for (int i = 0; i < kRT; ++i)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[i][c] = 0.0f;
#pragma unroll 4
  for (int k = 0; k < W; k += 4) {
    float a[kRT][4], w[TC][4];
#pragma unroll
    for (int i = 0; i < kRT; ++i) ldv(Hin + (tr + 32 * i) * L::LDA + k, a[i]);
#pragma unroll
    for (int c = 0; c < TC; ++c) ldv(Ws + (tc * TC + c) * L::LDW + k, w[c]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < kRT; ++i)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[i][c] = fmaf(a[i][q], w[c][q], acc[i][c]);
  }
  float bv[TC];
#pragma unroll
  for (int c = 0; c < TC; ++c) bv[c] = bias[tc * TC + c];
#pragma unroll
  for (int i = 0; i < kRT; ++i) {
    float o[TC], oc[TC];
#pragma unroll
    for (int c = 0; c < TC; ++c) {
      if (SINE) sincosf(acc[i][c] + bv[c], &o[c], &oc[c]);   // P:68 sine units; cos kept for act'
      else if (raw) o[c] = (tr & 7) == 0 ? acc[i][c] + bv[c] : acc[i][c];
      else o[c] = f32_tanh(acc[i][c] + bv[c]);
    }
    stv(Hout + (tr + 32 * i) * L::LDA + tc * TC, o);
    if (SINE) stv(CosOut + (tr + 32 * i) * L::LDA + tc * TC, oc);
  }
}

// In place: H[b][i] <- (sum_o G[b][o] W[o][i]) * (1 - H[b][i]^2)   (delta_{l-1}, tanh')
// raw (stable form, G27): the products sum_o G W are written over G itself (after a barrier:
// every thread has read G) for the stable backward map, H is left unchanged
template <int W, int NH, bool SINE = false>
__device__ __forceinline__ void bwd_gemm(float* __restrict__ G, float* __restrict__ H,
                                         const float* __restrict__ Ws, int tid,
                                         const float* __restrict__ Cs = nullptr, bool raw = false) {
  using L = Layout<W, NH>;
  constexpr int TC = L::TC;
  const int tr = tid & 31, tc = tid >> 5;
  float acc[kRT][TC];
#pragma unroll
  for (int i = 0; i < kRT; ++i)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[i][c] = 0.0f;
#pragma unroll 4
  for (int o = 0; o < W; o += 4) {
    float g[kRT][4], w[4][TC];
#pragma unroll
    for (int i = 0; i < kRT; ++i) ldv(G + (tr + 32 * i) * L::LDA + o, g[i]);
#pragma unroll
    for (int q = 0; q < 4; ++q) ldv(Ws + (o + q) * L::LDW + tc * TC, w[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int i = 0; i < kRT; ++i)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[i][c] = fmaf(g[i][q], w[q][c], acc[i][c]);
  }
  if (raw) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRT; ++i) stv(G + (tr + 32 * i) * L::LDA + tc * TC, acc[i]);
    return;
  }
#pragma unroll
  for (int i = 0; i < kRT; ++i) {
    float hv[TC], o[TC];
    float* p = H + (tr + 32 * i) * L::LDA + tc * TC;
    if (SINE) ldv(Cs + (tr + 32 * i) * L::LDA + tc * TC, hv);   // act' = cos(z)
    else ldv(p, hv);
#pragma unroll
    for (int c = 0; c < TC; ++c) o[c] = SINE ? acc[i][c] * hv[c] : acc[i][c] * (1.0f - hv[c] * hv[c]);
    stv(p, o);
  }
}

// dW[o][i] += sum_b G[b][o] H[b][i] over this thread's half of the rows; thread owns a
// DB x DB block (registers); the two halves are summed at the flush.
template <int W, int NH>
__device__ __forceinline__ void dw_gemm(const float* __restrict__ G, const float* __restrict__ H,
                                        float (&dW)[Layout<W, NH>::DB * Layout<W, NH>::DB], int tid) {
  using L = Layout<W, NH>;
  constexpr int DB = L::DB;
  const int t = tid & 255, half = tid >> 8;
  const int to = t >> 4, ti = t & 15;
#pragma unroll 4
  for (int b = half * (kB / kHalves); b < (half + 1) * (kB / kHalves); ++b) {
    float g[DB], hv[DB];
    ldv(G + b * L::LDA + to * DB, g);
    ldv(H + b * L::LDA + ti * DB, hv);
#pragma unroll
    for (int a = 0; a < DB; ++a)
#pragma unroll
      for (int c = 0; c < DB; ++c) dW[a * DB + c] = fmaf(g[a], hv[c], dW[a * DB + c]);
  }
}

// acc[col] += sum_b X[b][col] (fixed order: contiguous row ranges, then parts in order)
template <int W, int NH>
__device__ __forceinline__ void colsum(const float* __restrict__ X, float* __restrict__ acc,
                                       float* __restrict__ red, int tid, bool centre_only = false) {
  using L = Layout<W, NH>;
  constexpr int parts = kThreads / W, per = kB / parts;
  const int col = tid % W, part = tid / W;
  float s = 0.0f;
  for (int r = part * per; r < (part + 1) * per; ++r)
    if (!centre_only || (r & 7) == 0) s += X[r * L::LDA + col];
  red[part * W + col] = s;
  __syncthreads();
  if (tid < W) {
    float t = 0.0f;
    for (int p = 0; p < parts; ++p) t += red[p * W + tid];
    acc[tid] += t;
  }
  __syncthreads();
}

// W is the kernel width (16, 32, 64); the network's real width wr <= W (prm.width_real) is
// embedded with zero weights and biases in the padded units (their activations are 0 for tanh
// and sine, their deltas 0), and only real parameters are read and written.
// STAB: stencil tiles in the stable difference form (G27; tanh, training pass)
template <int W, int NH, int ACT, bool TRAIN, bool STAB = false>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_mlp_fp32(const MlpParams prm) {
  static_assert(kB % 32 == 0, "tile rows");
  static_assert(!STAB || (ACT == NBM_ACT_TANH && TRAIN), "stable form: tanh training pass");
  constexpr int TPT = STAB ? kB / 8 : kPT;   // stencil points per tile
  constexpr bool SINE = ACT == NBM_ACT_SINE;
  using L = Layout<W, NH, SINE>;
  constexpr int NHH = L::NHH;
  constexpr int DB = L::DB;
  extern __shared__ __align__(16) float sm[];
  float* sW1 = sm + L::oW1;
  float* sBias = sm + L::oB;
  float* sWh = sm + L::oWh;
  float* sWo = sm + L::oWo;
  float* sAct = sm + L::oAct;
  float* sX = sm + L::oX;
  float* sU = sm + L::oU;
  float* sUb = sm + L::oUb;
  float* sRed = sm + L::oRed;
  float* sAW1 = sm + L::oAW1;
  float* sAB = sm + L::oAB;
  float* sAWo = sm + L::oAWo;
  float* sAux = sm + L::oAux;
  int* sItem = reinterpret_cast<int*>(sm + L::oItem);
  float* sCos = sm + L::oCos;   // sine: cos(z_l), layer l at (l-1) kB LDA
  __shared__ int segTiles[kNumSeg + 1], segCnt[kNumSeg], segStart[kNumSeg];

  const int tid = threadIdx.x;
  // theta offsets of the real network (G17) with real width wr
  const int wr = prm.width_real > 0 ? prm.width_real : W;
  const int64_t tW1 = 0, tB1 = 3 * wr;
  auto tWl = [&](int l) -> int64_t { return 4 * wr + (int64_t)(l - 2) * (wr * wr + wr); };
  auto tBl = [&](int l) -> int64_t { return tWl(l) + (int64_t)wr * wr; };
  const int64_t tWo = 4 * wr + (int64_t)NHH * (wr * wr + wr), tBo = tWo + wr;
  if (tid < kNumSeg) {
    int c = prm.counts[prm.cnt_slot[tid]];
    segCnt[tid] = c;
    segStart[tid] = prm.start_slot[tid] >= 0 ? prm.counts[prm.start_slot[tid]] : 0;
    int per = prm.seg.kind[tid] == kSegStencil ? TPT : kB;
    segTiles[tid] = (c + per - 1) / per;
  }
  __syncthreads();
  int total = 0;
  int firstTile[kNumSeg + 1];
#pragma unroll
  for (int s = 0; s < kNumSeg; ++s) { firstTile[s] = total; total += segTiles[s]; }
  firstTile[kNumSeg] = total;
  const int G = gridDim.x, cta = blockIdx.x;
  const int t0 = (int)((int64_t)total * cta / G), t1 = (int)((int64_t)total * (cta + 1) / G);

  float dWh[NHH > 0 ? NHH : 1][DB * DB];
  double lossAcc = 0.0;
  int curNet = -1;
  bool touched[2] = {false, false};

  auto zero_acc = [&]() {
#pragma unroll
    for (int l = 0; l < (NHH > 0 ? NHH : 1); ++l)
#pragma unroll
      for (int e = 0; e < DB * DB; ++e) dWh[l][e] = 0.0f;
    for (int i = tid; i < 4 * W + NH * W + W + 4; i += kThreads) sAW1[i] = 0.0f;   // AW1, AB, AWo contiguous
  };
  auto flush = [&](int net) {
    float* out = prm.part + ((int64_t)net * G + cta) * prm.p_stride;
    NBM_CHECK(((int64_t)net * G + cta + 1) * prm.p_stride <= prm.part_len);
    const int t = tid & 255, half = tid >> 8;
    const int to = t >> 4, ti = t & 15;
    float* scr = sAct;   // free between tiles: [256][NHH][DB*DB] partials of the second row-half
    if (half == 1) {
#pragma unroll
      for (int l = 0; l < NHH; ++l)
#pragma unroll
        for (int e = 0; e < DB * DB; ++e) scr[(t * (NHH > 0 ? NHH : 1) + l) * DB * DB + e] = dWh[l][e];
    }
    __syncthreads();
    if (half == 0) {
#pragma unroll
      for (int l = 0; l < NHH; ++l)
#pragma unroll
        for (int a = 0; a < DB; ++a) {
          const int o = to * DB + a;
#pragma unroll
          for (int c = 0; c < DB; ++c) {
            const int i = ti * DB + c;
            if (o < wr && i < wr)
              out[tWl(l + 2) + (int64_t)o * wr + i] =
                  dWh[l][a * DB + c] +
                  (kHalves == 2 ? scr[(t * (NHH > 0 ? NHH : 1) + l) * DB * DB + a * DB + c] : 0.0f);
          }
        }
    }
    for (int i = tid; i < 3 * wr; i += kThreads) out[tW1 + i] = sAW1[i];
    for (int i = tid; i < wr; i += kThreads) {
      out[tB1 + i] = sAB[i];
      for (int l = 2; l <= NH; ++l) out[tBl(l) + i] = sAB[(l - 1) * W + i];
      out[tWo + i] = sAWo[i];
    }
    if (tid == 0) out[tBo] = sAWo[W];
    touched[net] = true;
  };
  auto load_net = [&](int net) {
    const float* th = prm.theta + (int64_t)net * prm.p_net;
    for (int i = tid; i < 3 * W; i += kThreads) sW1[i] = i < 3 * wr ? th[tW1 + i] : 0.0f;
    for (int i = tid; i < W; i += kThreads) {
      const bool real = i < wr;
      sBias[i] = real ? th[tB1 + i] : 0.0f;
      for (int l = 2; l <= NH; ++l) sBias[(l - 1) * W + i] = real ? th[tBl(l) + i] : 0.0f;
      sWo[i] = real ? th[tWo + i] : 0.0f;
    }
    if (tid == 0) sWo[W] = th[tBo];
    for (int l = 0; l < NHH; ++l)
      for (int i = tid; i < W * W; i += kThreads) {
        const int o = i / W, c = i % W;
        sWh[l * W * L::LDW + o * L::LDW + c] = (o < wr && c < wr) ? th[tWl(l + 2) + (int64_t)o * wr + c] : 0.0f;
      }
  };

  int seg = 0;
  for (int t = t0; t < t1; ++t) {
    while (t >= firstTile[seg + 1]) ++seg;
    const int kind = prm.seg.kind[seg], net = prm.seg.net[seg];
    const int lt = t - firstTile[seg];
    const int per = kind == kSegStencil ? TPT : kB;
    const int first = lt * per;
    const int nvalid = min(per, segCnt[seg] - first);
    const bool stab = STAB && kind == kSegStencil;   // block-uniform
    if (net != curNet) {
      __syncthreads();
      if (TRAIN && curNet >= 0) flush(curNet);
      __syncthreads();
      load_net(net);
      if (TRAIN) zero_acc();
      curNet = net;
    }
    // ---- gather the tile's items and rows (x, aux) ----
    const int* items = prm.seg.items[seg] + segStart[seg];
    if (tid < per) {
      int it = tid < nvalid ? item_at(prm.seg, seg, items, first + tid) : -1;
      sItem[tid] = it;
      float a = 0.0f;
      if (it >= 0) a = prm.aux_by_item[seg] ? prm.seg.aux[seg][it] : prm.seg.aux[seg][segStart[seg] + first + tid];
      sAux[tid] = a;
    }
    __syncthreads();
    if (tid < kB) {
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
        const int j = tid / kPT, p = tid - j * kPT;
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
      sX[4 * tid + 0] = x0; sX[4 * tid + 1] = x1; sX[4 * tid + 2] = x2;
    }
    __syncthreads();
    // ---- layer 1 (K = 3) on CUDA cores ----
    {
      const int col = tid % W, r0 = tid / W;
      constexpr int step = kThreads / W;
      const float w0 = sW1[3 * col], w1 = sW1[3 * col + 1], w2 = sW1[3 * col + 2], bb = sBias[col];
      for (int r = r0; r < kB; r += step) {
        float z = fmaf(w2, sX[4 * r + 2], fmaf(w1, sX[4 * r + 1], fmaf(w0, sX[4 * r], (!stab || (r & 7) == 0) ? bb : 0.0f)));
        if (SINE) sincosf(z, &sAct[r * L::LDA + col], &sCos[r * L::LDA + col]);
        else if (STAB && stab) sAct[r * L::LDA + col] = z;
        else sAct[r * L::LDA + col] = f32_tanh(z);
      }
    }
    __syncthreads();
    if (STAB && stab) {
      stab::fwd_pass_f32<W, L::LDA, kB / 8, kThreads>(sAct, tid);
      __syncthreads();
    }
    // ---- hidden GEMMs ----
#pragma unroll
    for (int l = 0; l < NHH; ++l) {
      fwd_gemm<W, NH, SINE>(sAct + l * kB * L::LDA, sAct + (l + 1) * kB * L::LDA, sWh + l * W * L::LDW,
                            sBias + (l + 1) * W, tid, sCos + (l + 1) * kB * L::LDA, STAB && stab);
      __syncthreads();
      if (STAB && stab) {
        stab::fwd_pass_f32<W, L::LDA, kB / 8, kThreads>(sAct + (l + 1) * kB * L::LDA, tid);
        __syncthreads();
      }
    }
    // ---- output layer u = wo . h_NH + bo ----
    float* hTop = sAct + (NH - 1) * kB * L::LDA;
    {
      const int r = tid >> 2, qq = tid & 3;
      float s = 0.0f;
      for (int k = qq * (W / 4); k < (qq + 1) * (W / 4); ++k) s = fmaf(sWo[k], hTop[r * L::LDA + k], s);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (qq == 0) sU[r] = (!stab || (r & 7) == 0) ? s + sWo[W] : s;   // differences carry no output bias
    }
    __syncthreads();
    if (!TRAIN) {
      if (tid < nvalid) prm.u_out[sItem[tid]] = sU[tid];
      __syncthreads();
      continue;
    }
    // ---- residual epilogue -> cotangents (S4) ----
    if (STAB && stab) {   // r = c_c u + c_hat sum_d DU_d - b/d (G27); cotangents c_c 2r/N, c_hat 2r/N (Q_d)
      if (tid < kB) {
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
      if (tid < kPT) {
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
          for (int j = 1; j < 7; ++j) acc = fmaf(cj[j - 1], sU[j * kPT + tid], acc);
          r = acc - sAux[tid];
          lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;   // r^2 / N
        }
        const float rc = prm.two_over_n * r;
        sUb[tid] = rc;
#pragma unroll
        for (int j = 1; j < 7; ++j) sUb[j * kPT + tid] = rc * cj[j - 1];
      } else if (tid >= 7 * kPT && tid < kB) {
        sUb[tid] = 0.0f;
      }
    } else if (tid < kB) {
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
    // ---- backward (S5) ----
    {  // output layer: dWo += sum_b ub h_NH, dbo += sum_b ub; then G_NH in place
      const int col = tid % W, part = tid / W;
      constexpr int parts = kThreads / W, per = kB / parts;
      float s = 0.0f;
      for (int r = part * per; r < (part + 1) * per; ++r) s = fmaf(sUb[r], hTop[r * L::LDA + col], s);
      sRed[part * W + col] = s;
      if (tid < 32) {
        float b = 0.0f;
        for (int r = tid; r < kB; r += 32)
          if (!stab || (r & 7) == 0) b += sUb[r];
        for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        if (tid == 0) sAWo[W] += b;
      }
      __syncthreads();
      if (tid < W) {
        float t = 0.0f;
        for (int p = 0; p < parts; ++p) t += sRed[p * W + tid];
        sAWo[tid] += t;
      }
      const float wo = sWo[col];
      if (STAB && stab) {
        __syncthreads();   // dWo has read h_NH
        stab::bwd_pass_f32<W, L::LDA, kB / 8, kThreads>(nullptr, hTop, sUb, sWo, tid);
      } else {
        for (int r = part; r < kB; r += parts) {
          float hv = hTop[r * L::LDA + col];
          const float ad = SINE ? sCos[(NH - 1) * kB * L::LDA + r * L::LDA + col] : 1.0f - hv * hv;
          hTop[r * L::LDA + col] = sUb[r] * wo * ad;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int l = NHH - 1; l >= 0; --l) {   // hidden layer (l+2): G in act[l+1], h in act[l]
      float* Gl = sAct + (l + 1) * kB * L::LDA;
      float* Hp = sAct + l * kB * L::LDA;
      dw_gemm<W, NH>(Gl, Hp, dWh[l], tid);
      colsum<W, NH>(Gl, sAB + (l + 1) * W, sRed, tid, STAB && stab);   // db (contains __syncthreads)
      bwd_gemm<W, NH, SINE>(Gl, Hp, sWh + l * W * L::LDW, tid, sCos + l * kB * L::LDA, STAB && stab);
      __syncthreads();
      if (STAB && stab) {   // G_{l+1} W_{l+1} (now in Gl) through the backward map of layer l+1 -> Hp
        stab::bwd_pass_f32<W, L::LDA, kB / 8, kThreads>(Gl, Hp, nullptr, nullptr, tid);
        __syncthreads();
      }
    }
    {  // layer 1: dW1[n][c] += sum_b G1[b][n] x[b][c]; db1 += sum_b G1[b][n]
      const int col = tid % W, part = tid / W;
      constexpr int parts = kThreads / W, per = kB / parts;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, sb = 0.f;
      for (int r = part * per; r < (part + 1) * per; ++r) {
        const float g = sAct[r * L::LDA + col];
        s0 = fmaf(g, sX[4 * r], s0);
        s1 = fmaf(g, sX[4 * r + 1], s1);
        s2 = fmaf(g, sX[4 * r + 2], s2);
        if (!stab || (r & 7) == 0) sb += g;
      }
      sRed[(0 * parts + part) * W + col] = s0;
      sRed[(1 * parts + part) * W + col] = s1;
      sRed[(2 * parts + part) * W + col] = s2;
      sRed[(3 * parts + part) * W + col] = sb;
      __syncthreads();
      if (tid < W) {
        float t0v = 0.f, t1v = 0.f, t2v = 0.f, tb = 0.f;
        for (int p = 0; p < parts; ++p) {
          t0v += sRed[(0 * parts + p) * W + tid];
          t1v += sRed[(1 * parts + p) * W + tid];
          t2v += sRed[(2 * parts + p) * W + tid];
          tb += sRed[(3 * parts + p) * W + tid];
        }
        sAW1[3 * tid] += t0v;
        sAW1[3 * tid + 1] += t1v;
        sAW1[3 * tid + 2] += t2v;
        sAB[tid] += tb;
      }
      __syncthreads();
    }
  }
  if (!TRAIN) return;
  __syncthreads();
  if (curNet >= 0) flush(curNet);
  if (tid < 2) prm.touched[tid * G + cta] = touched[tid] ? 1 : 0;
  // CTA loss: fixed-order block reduction of the per-thread partials
  for (int o = 16; o; o >>= 1) lossAcc += __shfl_xor_sync(0xffffffffu, lossAcc, o);
  __shared__ double wl[kThreads / 32];
  if ((tid & 31) == 0) wl[tid >> 5] = lossAcc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += wl[w];
    prm.lpart[cta] = s;
  }
}

template <int W, int NH, int ACT, bool TRAIN, bool STAB = false>
static cudaError_t launch_t(const MlpParams& p, int grid, cudaStream_t s) {
  using L = Layout<W, NH, ACT == NBM_ACT_SINE>;
  auto kern = k_mlp_fp32<W, NH, ACT, TRAIN, STAB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, (const void*)kern, (int)L::bytes); e != cudaSuccess) return e;
  kern<<<grid * kCtasPerSm, kThreads, L::bytes, s>>>(p);
  return cudaGetLastError();
}

int mlp_fp32_ctas_per_sm() { return kCtasPerSm; }

// kernel width for a real hidden width (the smallest of 16 / 32 / 64 that holds it)
static int kernel_width(int width) { return width <= 16 ? 16 : width <= 32 ? 32 : 64; }

int mlp_fp32_supported(int width, int n_hidden, int act) {
  if (width < 1 || n_hidden < 1) return 0;
  if (act == NBM_ACT_TANH) return (width <= 32 && n_hidden <= 5) || (width <= 64 && n_hidden <= 4);
  if (act == NBM_ACT_SINE) return width <= 32 && n_hidden <= 5;
  return 0;
}

template <int ACT, bool TRAIN>
static cudaError_t dispatch(int W, int NH, const MlpParams& p, int grid, cudaStream_t s) {
#define NBM_F32_CASES(WW)                                  \
  switch (NH) {                                            \
    case 1: return launch_t<WW, 1, ACT, TRAIN>(p, grid, s); \
    case 2: return launch_t<WW, 2, ACT, TRAIN>(p, grid, s); \
    case 3: return launch_t<WW, 3, ACT, TRAIN>(p, grid, s); \
    case 4: return launch_t<WW, 4, ACT, TRAIN>(p, grid, s); \
    case 5: return launch_t<WW, 5, ACT, TRAIN>(p, grid, s); \
  }
  if (W == 16) { NBM_F32_CASES(16) }
  if (W == 32) { NBM_F32_CASES(32) }
  if constexpr (ACT == NBM_ACT_TANH) {
    if (W == 64) {
      switch (NH) {
        case 1: return launch_t<64, 1, ACT, TRAIN>(p, grid, s);
        case 2: return launch_t<64, 2, ACT, TRAIN>(p, grid, s);
        case 3: return launch_t<64, 3, ACT, TRAIN>(p, grid, s);
        case 4: return launch_t<64, 4, ACT, TRAIN>(p, grid, s);
      }
    }
  }
#undef NBM_F32_CASES
  return cudaErrorInvalidValue;
}

// the stable form (G27): tanh training pass
static cudaError_t dispatch_stab(int W, int NH, const MlpParams& p, int grid, cudaStream_t s) {
  constexpr int T = NBM_ACT_TANH;
#define NBM_F32_SCASES(WW)                                        \
  switch (NH) {                                                   \
    case 1: return launch_t<WW, 1, T, true, true>(p, grid, s);    \
    case 2: return launch_t<WW, 2, T, true, true>(p, grid, s);    \
    case 3: return launch_t<WW, 3, T, true, true>(p, grid, s);    \
    case 4: return launch_t<WW, 4, T, true, true>(p, grid, s);    \
  }
  if (W == 16) {
    if (NH == 5) return launch_t<16, 5, T, true, true>(p, grid, s);
    NBM_F32_SCASES(16)
  }
  if (W == 32) {
    if (NH == 5) return launch_t<32, 5, T, true, true>(p, grid, s);
    NBM_F32_SCASES(32)
  }
  if (W == 64) { NBM_F32_SCASES(64) }
#undef NBM_F32_SCASES
  return cudaErrorInvalidValue;
}

cudaError_t launch_mlp_fp32(int width, int n_hidden, int act, bool train, bool stable, const MlpParams& p, int grid,
                            cudaStream_t s) {
  MlpParams q = p;
  q.width_real = width;
  const int W = kernel_width(width);
  if (stable && train) {
    if (act != NBM_ACT_TANH || p.pcoef) return cudaErrorInvalidValue;
    return dispatch_stab(W, n_hidden, q, grid, s);
  }
  if (act == NBM_ACT_SINE)
    return train ? dispatch<NBM_ACT_SINE, true>(W, n_hidden, q, grid, s) : dispatch<NBM_ACT_SINE, false>(W, n_hidden, q, grid, s);
  return train ? dispatch<NBM_ACT_TANH, true>(W, n_hidden, q, grid, s) : dispatch<NBM_ACT_TANH, false>(W, n_hidden, q, grid, s);
}

}  // namespace nbm
