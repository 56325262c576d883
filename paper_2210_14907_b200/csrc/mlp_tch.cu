// mlp_tch.cu -- K3h: the bf16 tcgen05 training kernel (fused MLP forward -> residual epilogue
// -> backward -> dW) with two 64-row half-tiles in flight per CTA, config
// 5-w128 (tanh, direct stencil form, 3-4 hidden layers).  Same arithmetic as K3t (mlp_tc.cu, DESIGN.md
// G16); the difference is the schedule.
//
// K3t walks one 128-row tile at a time: every stage of the chain (GEMM round trip, then a
// MUFU-bound epilogue over the whole CTA) waits for the previous one, so the tensor core idles
// during the epilogues and the epilogue warps idle during the GEMMs (K3t trace).
// A second 128-row tile in flight would need a second W-column TMEM accumulator, and at W = 128
// with 4 hidden layers TMEM is full (accumulator 128 + dW_2..4 384 columns).  K3h instead splits
// the CTA into two independent halves, each walking its own 64-row half-tiles with M = 64 MMAs:
// a cta_group::1 M = 64 accumulator occupies 16 lanes of each 32-lane quadrant, at lane offset 0
// or 16 of the same columns (measured, scripts/r2/m64_probe.cu), so the two halves' working
// accumulators share the W columns and TMEM stays at W + (NH-1) W.  While one half runs its
// epilogue, the other's GEMM runs; each half synchronises on its own named barrier and its own
// MMA mbarriers, and one converged warp per half issues that half's MMAs.
//
// Per half-tile (64 rows: 9 stencil points x 7 vertices + 1 pad row, or 64 independent rows):
//   layer 1 (K = 3, CUDA cores) -> bf16 h1;  l = 2..NH: acc = h_{l-1} W_l^T (M = 64, N = W)
//   -> tanh -> bf16 h_l;  u = wo . h_NH + bo;  residual epilogue (cotangents 2 r c_j / N);
//   G_NH = ub wo (1 - h_NH^2);  l = NH..2: acc = G_l W_l (M = 64), dW_l += G_l^T h_{l-1}
//   (M = W = 128 o-rows, N = W, K = 64: both halves accumulate into the same TMEM dW_l, zeroed
//   per network, their dW MMAs issued in half-tile order);  G_{l-1} = acc (1 - h~^2) in place
//   of h_{l-1}; h1 is recomputed (K = 3) for dW_2, its buffer having held G_NH.
//   Tail: [db_1, dW_1 (x, y, z as hi/lo bf16 planes) | db_l] = A_l G_l^T as M = 64 MMAs into the
//   half's own accumulator lanes (A_1 = [1, x_hi, x_lo, ...] rows, A_l = a ones row per layer,
//   MN-major; rows >= 16 of A are never read back), collected into fp32 shared accumulators.
// Half 1 starts after half 0's first hidden GEMM of each network run (named barrier 3) and the
// stagger persists; started together the halves ran in lock step and K3h was slower than K3t.
// Warps: 2 halves x 4 lane quadrants x W/64 column groups.  Thread (half, quad, cg, lane):
// row 16 quad + lane%16 of its half-tile, columns 64 cg + 32 (lane/16) .. +31 (the 16x32bx2
// TMEM access shape).  Rounding points: as K3t (GEMM operands bf16 RNE, tanh.approx,
// tanh' from the bf16 operand copy for layers 1..NH-1, exact fp32 for layer NH).
#include <cuda_bf16.h>
#include <math.h>

#include <atomic>

#include "nbm_internal.cuh"
#include "tc_epi.cuh"
#include "tc_ptx.cuh"

namespace nbm {

namespace {

using namespace epi;

constexpr int kHR = 64;   // rows per half-tile (MMA M of the row GEMMs)
constexpr int kHP = 9;    // stencil points per half-tile (63 rows + 1 pad row)

template <int W, int NH>
struct HLayout {
  static constexpr int NHH = NH - 1;
  static constexpr int NWH = W / 16;                     // warps per half
  static constexpr int THREADS = 2 * NWH * 32;
  static constexpr int NBUF = NH - 1 > 2 ? NH - 1 : 2;   // activation buffers per half
  static constexpr int CH = W / 32;                      // 32-column chunks per row
  static constexpr int NTR = NH + 5;                     // tail rows kept: [1, x_hi, x_lo, y_hi, y_lo, z_hi, z_lo] + db_2..db_{NH-1}
  static constexpr int NTP = NTR | 1;                    // their stride per unit o (odd: the 16 row-lanes of a collect hit 16 banks)
  static constexpr uint32_t ACT = kHR * W * 2;           // one bf16 half-tile activation buffer
  static constexpr uint32_t WMAT = W * W * 2;            // one bf16 weight matrix
  static constexpr uint32_t TAILA = 16 * kHR * 2;        // one tail A operand: [16][64] bf16, MN-major
  static constexpr uint32_t oAct = 0;                    // [half][NBUF]
  static constexpr uint32_t oWh = oAct + 2 * NBUF * ACT;  // W_2..W_NH (core-matrix, [o][i])
  static constexpr uint32_t oTailX = oWh + NHH * WMAT;    // [half] A_1 = [1, x, y, z split] rows
  static constexpr uint32_t oTailO = oTailX + 2 * TAILA;  // [NH-2] A_l: ones in row 7 + (l-2)
  static constexpr uint32_t oTailPad = oTailO + (NH - 2) * TAILA;   // the M-groups 2..7 of the last
                                                                    // A operand read past it
  static constexpr uint32_t oTacc = oTailPad + 1024;     // fp32 [half][W][NTP] tail accumulators
  static constexpr uint32_t oW1 = oTacc + 4 * 2 * NTP * W;   // fp32 [W][3]
  static constexpr uint32_t oBias = oW1 + 4 * 3 * W;     // fp32 [NH][W]
  static constexpr uint32_t oWo = oBias + 4 * NH * W;    // fp32 [W] + bo
  static constexpr uint32_t oHalf = oWo + 4 * (W + 4);   // per-half scalars
  static constexpr uint32_t hX = 0, hUp = 4 * 4 * kHR, hU = hUp + 4 * CH * kHR, hUb = hU + 4 * kHR,
                            hAux = hUb + 4 * kHR, hItem = hAux + 4 * kHR, HALF = hItem + 4 * kHR;
  static constexpr uint32_t oBar = oHalf + 2 * HALF;     // bar[2], dwbar[2], tmem base, dW turns
  static constexpr uint32_t bytes = oBar + 64 + 4 * 8;
  static constexpr uint32_t TMEM_COLS = (W * NH <= 128) ? 128 : (W * NH <= 256) ? 256 : 512;
  // CTAs per SM: must agree with mlp_tc_ctas_per_sm (the host sizes the partial slots with it)
  static constexpr int MINB = W * NH <= 256 ? 2 : 1;
  static_assert(bytes <= (MINB == 2 ? 113u * 1024u : 232448u), "shared memory");
  static_assert(4u * 2 * 4 * 2 * W + 64 <= 2u * NBUF * ACT, "flush scratch");
  // theta offsets within one network (G17)
  static constexpr int64_t tW1 = 0, tB1 = 3 * W;
  __host__ __device__ static constexpr int64_t tWl(int l) { return 4 * W + (int64_t)(l - 2) * (W * W + W); }
  __host__ __device__ static constexpr int64_t tBl(int l) { return tWl(l) + W * W; }
  static constexpr int64_t tWo = 4 * W + (int64_t)NHH * (W * W + W);
  static constexpr int64_t tBo = tWo + W;
};

// one thread's 32 columns (chunk c) of half-tile row r <-> the bf16 core-matrix buffer (R = 64)
__device__ __forceinline__ void store_row32(uint32_t buf, int r, int c, const float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    st_shared_v4(buf + core_off(kHR, r, c * 4 + q), pack_bf16(h[8 * q], h[8 * q + 1]), pack_bf16(h[8 * q + 2], h[8 * q + 3]),
                 pack_bf16(h[8 * q + 4], h[8 * q + 5]), pack_bf16(h[8 * q + 6], h[8 * q + 7]));
}
__device__ __forceinline__ void load_row32(uint32_t buf, int r, int c, float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
    ld_shared_v4(buf + core_off(kHR, r, c * 4 + q), w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[8 * q + 2 * e] = bf_lo(w[e]);
      h[8 * q + 2 * e + 1] = bf_hi(w[e]);
    }
  }
}
__device__ __forceinline__ void half_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// the two halves are started half a chain apart: half 1 waits (named barrier 3) until half 0's
// first half-tile of a run reaches this point of its chain (0: no offset; 1: after the first
// hidden GEMM's epilogue; 2: after the forward pass)
#ifndef NBM_TCH_OFFSET
#define NBM_TCH_OFFSET 1
#endif
// element (m, k) of a tail A operand ([16 m][64 k] bf16, MN-major core matrices: 8 k-rows x
// 8 m (16 B) each, k-core stride 256 B, m-group stride 128 B): a row's [1, x, y, z] entries
// m = 0..7 are one 16-byte store
__device__ __forceinline__ uint32_t tail_off(int m, int k) {
  return (uint32_t)((k >> 3) * 256 + (m >> 3) * 128 + (k & 7) * 16 + (m & 7) * 2);
}

}  // namespace

#ifdef NBM_TC_TRACE
__device__ long long g_tch_trace[2][8][32];   // CTA 0: [half][half-tile][point] clock64
#define TRH(k)                                                                          \
  do {                                                                                  \
    if (blockIdx.x == 0 && th == 0 && ntile < 8) g_tch_trace[half][ntile][k] = clock64(); \
  } while (0)
#else
#define TRH(k) \
  do {         \
  } while (0)
#endif

template <int W, int NH>
__global__ void __launch_bounds__(HLayout<W, NH>::THREADS, HLayout<W, NH>::MINB) k_mlp_tch(const MlpParams prm) {
  using L = HLayout<W, NH>;
  constexpr int NWH = L::NWH, HT = NWH * 32, CH = L::CH, NTR = L::NTR, NTP = L::NTP;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = tc::smem_u32(smem);
  float* sW1 = reinterpret_cast<float*>(smem + L::oW1);
  float* sBias = reinterpret_cast<float*>(smem + L::oBias);
  float* sWo = reinterpret_cast<float*>(smem + L::oWo);
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(smem + L::oBar + 32);
  // dW turns: dW_l MMAs of a run are issued in half-tile order (rs, rs+1, rs+2, ...: the halves
  // alternate), so the fp32 accumulation order in TMEM, and the result, is deterministic
  volatile int* sTurn = reinterpret_cast<volatile int*>(smem + L::oBar + 64);
  __shared__ int segTiles[kNumSeg], segCnt[kNumSeg], segStart[kNumSeg];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = warp / NWH, wh = warp % NWH, quad = wh & 3, cg = wh >> 2;
  const int r16 = lane & 15, side = lane >> 4;
  const int th = tid - half * HT;                         // thread index within the half
  const int row = quad * 16 + r16;                        // half-tile row
  const int chunk = cg * 2 + side;                        // 32-column chunk
  const int ccol = chunk * 32;
  const bool iw = wh == 0;                                // the half's MMA-issuing warp
  const int hbar_id = 1 + half;
  uint8_t* hs = smem + L::oHalf + half * L::HALF;
  float* sX = reinterpret_cast<float*>(hs + L::hX);
  float* sUp = reinterpret_cast<float*>(hs + L::hUp);
  float* sU = reinterpret_cast<float*>(hs + L::hU);
  float* sUb = reinterpret_cast<float*>(hs + L::hUb);
  float* sAux = reinterpret_cast<float*>(hs + L::hAux);
  int* sItem = reinterpret_cast<int*>(hs + L::hItem);
  float* sTacc = reinterpret_cast<float*>(smem + L::oTacc) + half * NTP * W;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::oBar) + half;        // acc MMAs of this half
  uint64_t* dwbar = reinterpret_cast<uint64_t*>(smem + L::oBar + 16) + half;  // dW MMAs of this half

  if (tid < kNumSeg) {
    const int c = prm.counts[prm.cnt_slot[tid]];
    segCnt[tid] = c;
    segStart[tid] = prm.start_slot[tid] >= 0 ? prm.counts[prm.start_slot[tid]] : 0;
    const int per = prm.seg.kind[tid] == kSegStencil ? kHP : kHR;
    segTiles[tid] = (c + per - 1) / per;
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) tc::mbar_init(reinterpret_cast<uint64_t*>(smem + L::oBar) + i, 1);
    tc::mbar_fence_init();
  }
  {  // constant tail operands (ones rows of db_2..db_{NH-1}), zeroed per-half operands and slack
    uint32_t* z = reinterpret_cast<uint32_t*>(smem + L::oTailX);
    for (int i = tid; i < (int)((2 + (NH - 2)) * L::TAILA + 1024) / 4; i += L::THREADS) z[i] = 0u;
  }
  if (warp == 0) tc::tmem_alloc(sTmem, L::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *sTmem;
  for (int l = 2; l <= NH - 1; ++l)
    for (int k = tid; k < kHR; k += L::THREADS)
      *reinterpret_cast<__nv_bfloat16*>(smem + L::oTailO + (l - 2) * L::TAILA + tail_off(7 + (l - 2), k)) =
          __float2bfloat16(1.0f);

  int firstTile[kNumSeg + 1];
  int total = 0;
#pragma unroll
  for (int s = 0; s < kNumSeg; ++s) { firstTile[s] = total; total += segTiles[s]; }
  firstTile[kNumSeg] = total;
  const int G = gridDim.x, cta = blockIdx.x;
  const int t0 = (int)((int64_t)total * cta / G), t1 = (int)((int64_t)total * (cta + 1) / G);

  constexpr uint32_t LBO_ACT = kHR * 16, LBO_W = W * 16;
  const uint32_t aAct = sbase + L::oAct + half * L::NBUF * L::ACT, aWh = sbase + L::oWh;
  const uint32_t aTailX = sbase + L::oTailX + half * L::TAILA, aTailO = sbase + L::oTailO;
  auto buf = [&](int i) -> uint32_t { return aAct + i * L::ACT; };
  auto wmat = [&](int l) -> uint32_t { return aWh + (l - 2) * L::WMAT; };
  constexpr uint32_t ID_FWD = tc::idesc_bf16(kHR, W, 0, 0);    // A K-major, B K-major
  constexpr uint32_t ID_DH = tc::idesc_bf16(kHR, W, 0, 1);     // A K-major, B MN-major
  constexpr uint32_t ID_DW = tc::idesc_bf16(128, W, 1, 1);     // M = o (padded to 128), both MN-major
  constexpr uint32_t ID_TAIL = tc::idesc_bf16(kHR, W, 1, 1);   // M = tail rows (MN-major), N = o
  const uint32_t tAcc = tmem + ((uint32_t)(half * 16) << 16);                      // MMA D of this half
  const uint32_t tMine = tmem + ((uint32_t)(quad * 32 + half * 16) << 16) + (uint32_t)(cg * 64);   // my rows / columns
  uint32_t phase = 0, dwphase = 0;

  // transposed gradients (lane 16 side + j: columns ccol + j and ccol + 16 + j over the
  // half-warp's 16 rows): wo, b_NH; output bias (cg = 0 warps, side 0 lanes)
  float gWo[2] = {0.0f, 0.0f}, gBN[2] = {0.0f, 0.0f}, gbo = 0.0f;
  double lossAcc = 0.0;
  int curNet = -1;
  bool touched[2] = {false, false};
  bool tailPending = false;
  int ntile = 0;   // half-tiles this half has processed (trace index)

  // MMAs (the half's issuing warp, one elected lane); descriptors advance by the K step
  auto gemm = [&](uint32_t d, uint32_t a0, uint32_t a_step, uint32_t a_lbo, uint32_t a_sbo, uint32_t b0,
                  uint32_t b_step, uint32_t b_lbo, uint32_t b_sbo, uint32_t idesc, int ksteps, bool acc) {
    const uint64_t ad = tc::sdesc(a0, a_lbo, a_sbo), bd = tc::sdesc(b0, b_lbo, b_sbo);
#pragma unroll 4
    for (int s = 0; s < ksteps; ++s)
      tc::mma_bf16_w(d, ad + (uint64_t)((s * a_step) >> 4), bd + (uint64_t)((s * b_step) >> 4), idesc,
                     (acc || s > 0) ? 1u : 0u);
  };
  auto wait_acc = [&]() {
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::tc_fence_after();
  };
  auto hsync = [&]() { half_bar(hbar_id, HT); };

  auto flush = [&](int net) {   // whole CTA
    float* out = prm.part + ((int64_t)net * G + cta) * prm.p_stride;
    NBM_CHECK(((int64_t)net * G + cta + 1) * prm.p_stride <= prm.part_len);
    tc::tc_fence_after();
    {  // dW_l[o][i] from TMEM (o = lane)
      const int q = warp & 3, j = warp >> 2, o = q * 32 + lane;
#pragma unroll 1
      for (int l = 2; l <= NH; ++l)
        for (int cb = j; cb < W / 32; cb += L::THREADS / 128) {
          float v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(W * (l - 1) + cb * 32), v);
          if (o < W) {
            float4* dst = reinterpret_cast<float4*>(out + L::tWl(l) + (int64_t)o * W + cb * 32);
#pragma unroll
            for (int e = 0; e < 8; ++e) dst[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
          }
        }
    }
    const float* T0 = reinterpret_cast<const float*>(smem + L::oTacc);
    const float* T1 = T0 + NTP * W;
    for (int o = tid; o < W; o += L::THREADS) {   // tail reductions: halves in fixed order
      const float* a = T0 + o * NTP;
      const float* b = T1 + o * NTP;
      out[L::tB1 + o] = a[0] + b[0];
#pragma unroll
      for (int c = 0; c < 3; ++c) out[L::tW1 + 3 * o + c] = (a[1 + 2 * c] + a[2 + 2 * c]) + (b[1 + 2 * c] + b[2 + 2 * c]);
      for (int l = 2; l <= NH - 1; ++l) out[L::tBl(l) + o] = a[5 + l] + b[5 + l];
    }
    // transposed gradients: [half][quad][2][W] + [half][quad] bo, summed in (half, quad) order
    float* scr = reinterpret_cast<float*>(smem + L::oAct);
    __syncthreads();
    {
      float* s = scr + (half * 4 + quad) * 2 * W;
      s[ccol + r16] = gBN[0];
      s[ccol + 16 + r16] = gBN[1];
      s[W + ccol + r16] = gWo[0];
      s[W + ccol + 16 + r16] = gWo[1];
      if (cg == 0 && lane == 0) scr[16 * W + half * 4 + quad] = gbo;
    }
    __syncthreads();
    for (int i = tid; i < 2 * W; i += L::THREADS) {
      const int v = i / W, col = i % W;
      float s = 0.0f;
      for (int k = 0; k < 8; ++k) s += scr[k * 2 * W + v * W + col];
      out[(v == 0 ? L::tBl(NH) : L::tWo) + col] = s;
    }
    if (tid == 0) {
      float s = 0.0f;
      for (int k = 0; k < 8; ++k) s += scr[16 * W + k];
      out[L::tBo] = s;
    }
    __syncthreads();
    touched[net] = true;
  };

  auto load_net = [&](int net) {   // whole CTA; the dW columns are zeroed (both halves accumulate)
    const float* th = prm.theta + (int64_t)net * prm.p_net;
    for (int i = tid; i < 3 * W; i += L::THREADS) sW1[i] = th[L::tW1 + i];
    for (int i = tid; i < W; i += L::THREADS) {
      sBias[i] = th[L::tB1 + i];
      for (int l = 2; l <= NH; ++l) sBias[(l - 1) * W + i] = th[L::tBl(l) + i];
      sWo[i] = th[L::tWo + i];
    }
    if (tid == 0) sWo[W] = th[L::tBo];
    for (int l = 0; l < L::NHH; ++l) {   // hidden weights -> bf16 core-matrix layout [o][i]
      const float* Wl = th + L::tWl(l + 2);
      for (int q = tid; q < W * (W / 8); q += L::THREADS) {
        const int o = q / (W / 8), c8 = q % (W / 8);
        const float* src = Wl + (int64_t)o * W + c8 * 8;   // net+ theta is not 16-B aligned
        float r[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = src[e];
        st_shared_v4(aWh + l * L::WMAT + core_off(W, o, c8), pack_bf16(r[0], r[1]), pack_bf16(r[2], r[3]),
                     pack_bf16(r[4], r[5]), pack_bf16(r[6], r[7]));
      }
    }
    tc::fence_proxy_async_smem();
    float* T = reinterpret_cast<float*>(smem + L::oTacc);
    for (int i = tid; i < 2 * NTP * W; i += L::THREADS) T[i] = 0.0f;
    {
      float z[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = 0.0f;
      const int q = warp & 3, j = warp >> 2;
      for (int cb = j; cb < (NH - 1) * W / 32; cb += L::THREADS / 128)
        tc::tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(W + cb * 32), z);
    }
    gWo[0] = gWo[1] = gBN[0] = gBN[1] = gbo = 0.0f;
    if (tid < 8) sTurn[tid] = 0;
  };

  // layer 1 for this thread's 32 columns: h = tanh(W1 x + b1)
  auto layer1 = [&](float x0, float x1, float x2, float (&h)[32]) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = ccol + j;
      h[j] = tanh_fast(fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, fmaf(sW1[3 * n], x0, sBias[n]))));
    }
  };

  // global loads of one half-tile for thread th < 64: item slot th (index + aux) and the
  // coordinates of row th (stencil arm generated on the fly); issued one half-tile ahead
  struct Fetch { int item; float aux, x0, x1, x2; };
  auto fetch = [&](int tt, int tend) -> Fetch {
    Fetch f{-1, 0.0f, 0.0f, 0.0f, 0.0f};
    if (tt >= tend || th >= kHR) return f;
    int sg = 0;
    while (tt >= firstTile[sg + 1]) ++sg;
    const int knd = prm.seg.kind[sg];
    const int pr = knd == kSegStencil ? kHP : kHR;
    const int fst = (tt - firstTile[sg]) * pr;
    const int nv = min(pr, segCnt[sg] - fst);
    const int* its = prm.seg.items[sg] + segStart[sg];
    if (th < pr && th < nv) {
      f.item = item_at(prm.seg, sg, its, fst + th);
      f.aux = prm.aux_by_item[sg] ? prm.seg.aux[sg][f.item] : prm.seg.aux[sg][segStart[sg] + fst + th];
    }
    if (knd == kSegStencil) {
      const int j = th / kHP, p = th - j * kHP;
      if (j < 7 && p < nv) {
        const float* src = prm.seg.src[sg] + 3 * (int64_t)item_at(prm.seg, sg, its, fst + p);
        f.x0 = src[0]; f.x1 = src[1]; f.x2 = src[2];
        if (j > 0) {   // arms +x, -x, +y, -y, +z, -z (exact on the lattice)
          const float hs = (j & 1) ? prm.h : -prm.h;
          if (j <= 2) f.x0 = __fadd_rn(f.x0, hs); else if (j <= 4) f.x1 = __fadd_rn(f.x1, hs); else f.x2 = __fadd_rn(f.x2, hs);
        }
      }
    } else if (th < nv) {
      const float* src = prm.seg.src[sg] + 3 * (int64_t)item_at(prm.seg, sg, its, fst + th);
      f.x0 = src[0]; f.x1 = src[1]; f.x2 = src[2];
    }
    return f;
  };

  // the tail reductions of the half's last half-tile: accumulator rows 0..15 (quadrant-0 lanes)
  auto tail_collect = [&]() {
    wait_acc();
    if (quad == 0) {   // rows 0..NTR-1 of the tail accumulator: [1, x_hi, x_lo, y_hi, y_lo, z_hi, z_lo, db_2..]
      float v[32];
      tc::tmem_ld16x2(tMine, v);
      if (r16 < NTR) {
        float* t = sTacc + ccol * NTP + r16;
#pragma unroll
        for (int j = 0; j < 32; ++j) t[j * NTP] += v[j];
      }
    }
    tailPending = false;
  };

  // ---- network runs: contiguous tile ranges of one network (net- segments precede net+) ----
  int seg = 0;
  for (int rs = t0; rs < t1;) {
    while (rs >= firstTile[seg + 1]) ++seg;
    const int net = prm.seg.net[seg];
    int re = rs, sg = seg;
    while (re < t1) {
      while (re >= firstTile[sg + 1]) ++sg;
      if (prm.seg.net[sg] != net) break;
      re = min(t1, firstTile[sg + 1]);
    }
    if (net != curNet) {
      if (curNet >= 0) flush(curNet);
      load_net(net);
      curNet = net;
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
    }
    // ---- this half's half-tiles of the run: rs + half, rs + half + 2, ... ----
    const bool stagger = NBM_TCH_OFFSET > 0 && re - rs >= 2;   // half 1 has work in this run
    bool pendingGo = stagger && half == 0;
    if (stagger && half == 1) half_bar(3, HT + 32);
    Fetch cur = fetch(rs + half, re);
    int hseg = seg;
    int seq = half;   // this half-tile's position in the run (the dW turn it takes)
#pragma unroll 1
    for (int t = rs + half; t < re; t += 2) {
      while (t >= firstTile[hseg + 1]) ++hseg;
      const int kind = prm.seg.kind[hseg];
      const int lt = t - firstTile[hseg];
      const int per = kind == kSegStencil ? kHP : kHR;
      const int nvalid = min(per, segCnt[hseg] - lt * per);
      if (th < kHR) {
        if (th < per) {
          sItem[th] = cur.item;
          sAux[th] = cur.aux;
        }
        *reinterpret_cast<float4*>(sX + 4 * th) = make_float4(cur.x0, cur.x1, cur.x2, 0.0f);
      }
      hsync();
      TRH(0);
      const float x0 = sX[4 * row], x1 = sX[4 * row + 1], x2 = sX[4 * row + 2];
      {  // layer 1 -> bf16 h1 (buffer 0; the previous half-tile's tail MMAs may still read it)
        float h[32];
        layer1(x0, x1, x2, h);
        if (tailPending) tail_collect();
        store_row32(buf(0), row, chunk, h);
      }
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      hsync();
      TRH(1);
      // ---- hidden layers 2..NH ----
#pragma unroll 1
      for (int l = 2; l <= NH; ++l) {
        if (iw) {
          tc::tc_fence_after();
          gemm(tAcc, buf(l - 2), 2 * LBO_ACT, LBO_ACT, 128, wmat(l), 2 * LBO_W, LBO_W, 128, ID_FWD, W / 16, false);
          tc::mma_commit_w(bar);
        }
        wait_acc();
        TRH(2 + 2 * (l - 2));
        float v[32];
        tc::tmem_ld16x2(tMine, v);
        const float* bl = sBias + (l - 1) * W + ccol;
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = tanh_fast(v[j] + bl[j]);
        if (l < NH) {
          store_row32(buf(l - 1), row, chunk, v);
          tc::fence_proxy_async_smem();
        } else {
          float up = 0.0f;
#pragma unroll
          for (int j = 0; j < 32; ++j) up = fmaf(sWo[ccol + j], v[j], up);
          sUp[chunk * kHR + row] = up;
          tc::tmem_st16x2(tMine, v);   // fp32 h_NH for the backward
        }
        tc::tc_fence_before();
        hsync();
        TRH(3 + 2 * (l - 2));
        if (pendingGo && (NBM_TCH_OFFSET == 1 || l == NH)) {   // release half 1 (see NBM_TCH_OFFSET)
          if (iw) bar_arrive(3, HT + 32);
          pendingGo = false;
        }
      }
      if (th < kHR) {
        float u = sUp[th];
#pragma unroll
        for (int c = 1; c < CH; ++c) u += sUp[c * kHR + th];
        sU[th] = u + sWo[W];
      }
      hsync();
      TRH(8);
      // ---- residual epilogue -> cotangents (S4) ----
      if (kind == kSegStencil) {
        if (th < kHP) {
          float r = 0.0f;
          float cj[6];   // arm coefficients c_j / d: uniform (constant beta) or per point (variable mu)
#pragma unroll
          for (int j = 0; j < 6; ++j) cj[j] = prm.seg.chat[hseg];
          if (prm.pcoef && th < nvalid) {
            const float* pc = prm.pcoef + 6 * (int64_t)sItem[th];
#pragma unroll
            for (int j = 0; j < 6; ++j) cj[j] = pc[j];
          }
          if (th < nvalid) {
            float acc = sU[th];
#pragma unroll
            for (int j = 1; j < 7; ++j) acc = fmaf(cj[j - 1], sU[j * kHP + th], acc);
            r = acc - sAux[th];
            lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;
          }
          const float rc = prm.two_over_n * r;
          sUb[th] = rc;
#pragma unroll
          for (int j = 1; j < 7; ++j) sUb[j * kHP + th] = rc * cj[j - 1];
        } else if (th >= 7 * kHP && th < kHR) {
          sUb[th] = 0.0f;
        }
      } else if (th < kHR) {
        float ub = 0.0f;
        if (th < nvalid) {
          if (kind == kSegBRows) {
            const float e = sU[th] - sAux[th];
            ub = prm.seg.a[hseg] * e;
            lossAcc += 0.5 * (double)prm.seg.a[hseg] * (double)e * (double)e;
          } else {
            ub = sAux[th];
          }
        }
        sUb[th] = ub;
      }
      hsync();
      TRH(9);
      const float ub = sUb[row];
      if (cg == 0) {   // output bias: side-0 lanes carry the row sums
        float b = side == 0 ? ub : 0.0f;
#pragma unroll
        for (int o = 8; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
        gbo += b;
      }
      // ---- output layer backward: dwo += ub h_NH; G_NH = ub wo (1 - h_NH^2) -> bf16 ----
      const uint32_t gbufNH = (NH == 2) ? buf(1) : buf(0);
      {
        float hv[32], v[32];
        tc::tmem_ld16x2(tMine, hv);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] = hv[j] * ub;
          hv[j] = (1.0f - hv[j] * hv[j]) * (ub * sWo[ccol + j]);
        }
        float s0, s1;
        warp_transpose_sum16(v, lane, s0, s1);
        gWo[0] += s0;
        gWo[1] += s1;
        store_row32(gbufNH, row, chunk, hv);
        warp_transpose_sum16(hv, lane, s0, s1);
        gBN[0] += s0;
        gBN[1] += s1;
      }
      tc::tc_fence_before();
      tc::fence_proxy_async_smem();
      hsync();
      TRH(10);
      // ---- hidden layers backward ----
      Fetch nxt;
#pragma unroll 1
      for (int l = NH; l >= 2; --l) {
        const uint32_t gbuf = (l == NH) ? gbufNH : buf(l - 1);   // G_l
        const uint32_t hbuf = buf(l - 2);                        // h_{l-1}
        if (iw) {
          tc::tc_fence_after();
          // acc = G_l W_l: A = G (K-major), B = W_l (N = i, K = o: MN-major)
          gemm(tAcc, gbuf, 2 * LBO_ACT, LBO_ACT, 128, wmat(l), 256, 128, LBO_W, ID_DH, W / 16, false);
          tc::mma_commit_w(bar);
          // dW_l += G_l^T h_{l-1}: A = G (M = o, MN-major), B = h (N = i, MN-major), K = rows
          {   // a broken turn order would hang the GPU: trap after ~10 s instead
            const long long w0 = clock64();
            while (sTurn[l] != seq)
              if (clock64() - w0 > 20000000000ll) __trap();
          }
          gemm(tmem + (uint32_t)(W * (l - 1)), gbuf, 256, 128, LBO_ACT, hbuf, 256, 128, LBO_ACT, ID_DW, kHR / 16, true);
          tc::mma_commit_w(dwbar);
          __syncwarp();
          if (lane == 0) sTurn[l] = seq + 1;
        }
        if (l == NH) nxt = fetch(t + 2, re);   // the next half-tile's loads, under the MMAs
        wait_acc();
        TRH(11 + 2 * (NH - l));
        float v[32], hq[32];
        tc::tmem_ld16x2(tMine, v);
        load_row32(hbuf, row, chunk, hq);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= 1.0f - hq[j] * hq[j];
        tc::mbar_wait(dwbar, dwphase);   // dW_l has read h_{l-1} (and G_l)
        dwphase ^= 1;
        store_row32(hbuf, row, chunk, v);   // G_{l-1} in place: h_{l-1} is consumed
        if (l - 1 == 2 && NH >= 3) {   // h1 again for dW_2 (buffer 0's G_NH is consumed)
          float h[32];
          layer1(x0, x1, x2, h);
          store_row32(buf(0), row, chunk, h);
        }
        if (l == 2 && chunk == 0) {   // tail operand A_1 column `row`: [1, x_hi, x_lo, y_hi, y_lo, z_hi, z_lo, 0]
          const float xh = __bfloat162float(__float2bfloat16_rn(x0)), yh = __bfloat162float(__float2bfloat16_rn(x1)),
                      zh = __bfloat162float(__float2bfloat16_rn(x2));
          st_shared_v4(aTailX + tail_off(0, row), pack_bf16(1.0f, xh), pack_bf16(x0 - xh, yh), pack_bf16(x1 - yh, zh),
                       pack_bf16(x2 - zh, 0.0f));
        }
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        hsync();
        TRH(12 + 2 * (NH - l));
      }
      // ---- tail: [db_1, dW_1 | db_l] = A_1 G_1^T + sum_l A_l G_l^T into the half's accumulator ----
      if (iw) {
        tc::tc_fence_after();
        gemm(tAcc, aTailX, 512, 256, 128, buf(0), 256, 128, LBO_ACT, ID_TAIL, kHR / 16, false);   // A: lbo = k-core, sbo = m-group
        for (int l = 2; l <= NH - 1; ++l)
          gemm(tAcc, aTailO + (l - 2) * L::TAILA, 512, 256, 128, buf(l - 1), 256, 128, LBO_ACT, ID_TAIL, kHR / 16, true);
        tc::mma_commit_w(bar);
      }
      tailPending = true;   // collected under the next half-tile's gather and layer 1
      TRH(20);
      ++ntile;
      seq += 2;
      cur = nxt;
    }
    if (tailPending) tail_collect();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    rs = re;
  }
  if (curNet >= 0) flush(curNet);
  if (tid < 2) prm.touched[tid * G + cta] = touched[tid] ? 1 : 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) lossAcc += __shfl_xor_sync(0xffffffffu, lossAcc, o);
  __shared__ double wl[32];
  if (lane == 0) wl[warp] = lossAcc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < L::THREADS / 32; ++w) s += wl[w];
    prm.lpart[cta] = s;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, L::TMEM_COLS);
}

#ifdef NBM_TC_TRACE
extern "C" int nbm_debug_tch_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_tch_trace, sizeof(g_tch_trace));
}
#endif

template <int W, int NH>
static cudaError_t launch_tch_t(const MlpParams& p, int grid, cudaStream_t s) {
  using L = HLayout<W, NH>;
  auto kern = k_mlp_tch<W, NH>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, (const void*)kern, (int)L::bytes); e != cudaSuccess) return e;
  kern<<<grid * L::MINB, L::THREADS, L::bytes, s>>>(p);
  return cudaGetLastError();
}

// W = 128 only: at W = 64 K3t already runs two CTAs (two 128-row tiles) per SM, and K3h measured
// the same time there (8.1 vs 8.0 ms per c5-w64 launch)
int mlp_tch_supported(int width, int n_hidden, int act) {
  return act == NBM_ACT_TANH && width == 128 && n_hidden >= 3 && n_hidden <= 4;
}

cudaError_t launch_mlp_tch(int width, int n_hidden, const MlpParams& p, int grid, cudaStream_t s) {
  if (width == 128) {
    switch (n_hidden) {
      case 3: return launch_tch_t<128, 3>(p, grid, s);
      case 4: return launch_tch_t<128, 4>(p, grid, s);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace nbm
