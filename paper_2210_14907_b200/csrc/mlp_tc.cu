// mlp_tc.cu -- K3t: the fused MLP forward -> residual epilogue -> backward -> dW kernel
// with the hidden x hidden GEMMs on the 5th-generation tensor cores (tcgen05, bf16 in,
// fp32 accumulate in TMEM), configs 3 / 5-w64 (SURVEY 8a S3-S5, 7.3 hard parts 3-5); the
// config 5-w128 training pass runs K3h (mlp_tch.cu), the two-half-tile schedule of this kernel.
//
// One CTA per SM (two at W = 64) walks a contiguous range of 128-row tiles (18 stencil points x 7
// vertices, or 128 independent rows).  4 * W/32 warps: warp w owns rows 32*(w%4)..+31
// (its TMEM lane quadrant) and columns 32*(w/4)..+31 of every activation, so the
// epilogues are spread over 16 warps at W = 128.  Per tile, for NH hidden layers:
//   layer 1 (K = 3) on the CUDA cores -> bf16 h1 (shared memory, core-matrix layout)
//   for l = 2..NH: tcgen05.mma  acc = h_{l-1} W_l^T   (M=128, N=W, K=W) -> epilogue
//       (tcgen05.ld -> bias, tanh -> bf16 operand for the next GEMM)
//   output layer u = wo . h_NH + bo (per-chunk partials) -> residual epilogue
//   (r = M^-1 A u - M^-1 b; cotangents 2 r chat_j / N)
//   backward: G_NH = u_bar wo (1 - h_NH^2);  for l = NH..2:
//       tcgen05.mma  dW_l += G_l^T h_{l-1}   (M=W (64: the M = 64 lane layout), N=W, K=128; dW stays in TMEM for all
//                                             the CTA's tiles and is written out once)
//       tcgen05.mma  acc   = G_l W_l          (M=128, N=W, K=W)
//       epilogue G_{l-1} = acc * (1 - h~_{l-1}^2) -> bf16 operand
//   tile tail: tcgen05.mma  [db_2..db_{NH-1} | db_1, dW_1] = G_l^T [1 | 1, x, y, z]
//       (M=W, N=16, K=128) into the free working accumulator; output-layer and b_NH
//       gradients: warp transpose-reductions into registers.
// TMEM columns: [0,W) working accumulator, [W(l-1), W l) dW_l  (W * NH <= 512).
// Shared memory (W=128, NH=4): 3 bf16 hidden weight matrices + 3 bf16 activation
// buffers = 192 KB.  h1 is recomputed (K = 3) for dW_2 instead of being kept, unless one more
// activation buffer fits (XBUF) and holds G_NH.  The MMAs are issued by warp 0, converged
// (elect.sync); the SiLU kernel streams its weights through one TMA stage.
// Rounding points (G16): GEMM operands bf16 (RNE), accumulators and everything
// else fp32; tanh' = 1 - h~^2 from the bf16 operand copy for hidden layers 1..NH-1,
// exact fp32 for layer NH; activation = hardware tanh.approx.f32.
#include <cuda_bf16.h>
#include <math.h>

#include "nbm_internal.cuh"
#include "stab.cuh"
#include "tc_ptx.cuh"
#include "tc_epi.cuh"

namespace nbm {

namespace {

using namespace epi;

constexpr int kTB = 128;   // rows per tile (= MMA M = TMEM lanes)
constexpr int kTPT = 18;   // stencil points per tile
constexpr int kTPTS = 16;  // stencil points per tile of the stable form (G27): 8 rows per point

// P = 1: bf16 operands (G16).  P = 3: fp32-accurate GEMMs for the fp32 configs -- every operand
// is split exactly into three bf16 planes x = x1 + x2 + x3 (x1 = bf16(x), x2 = bf16(x - x1),
// x3 = bf16(x - x1 - x2)) and each GEMM sums the six plane products with i + j <= 2 (the three
// dropped ones are below 2^-24 relative), fp32 accumulation in TMEM (PREC_FP32X, G26).
// STG: columns of the fp32 staging tile of the shared-memory stable maps (0: none)
template <int W, int NH, int ACT, int P = 1, int STG = 0>
struct TcLayout {
  static_assert(P == 1 || (P == 3 && ACT == NBM_ACT_TANH), "plane split: tanh");
  static constexpr bool SILU = ACT == NBM_ACT_SILU;
  // weights streamed (TMA bulk) to make room: for SiLU's act' buffers, and for the three-plane
  // split at four hidden layers (three 48 KB activation buffers)
  static constexpr bool STREAM = SILU || (P == 3 && NH >= 4);
  static constexpr int NHH = NH - 1;
  static constexpr int NWRES = STREAM ? 1 : NHH;           // weight matrices held in shared memory
  static constexpr int NWRES_() { return STREAM ? 1 : NHH; }
  static constexpr int NDER = SILU ? (NH - 2 > 0 ? NH - 2 : 0) : 0;   // bf16 act' buffers, layers 2..NH-1
  static constexpr int CH = W / 32;                        // 32-column chunks per row
  static constexpr int THREADS = 128 * CH;                 // 4 lane quadrants x CH chunks
  static constexpr int NT = NH + 2;                        // tensor-core reduced gradient vectors
  static constexpr uint32_t ACT_BYTES = kTB * W * 2;       // one bf16 activation plane
  static constexpr uint32_t WMAT_BYTES = W * W * 2;        // one bf16 weight plane
  static constexpr uint32_t ABUF = P * ACT_BYTES;          // one activation buffer (P planes)
  static constexpr uint32_t WBUF = P * WMAT_BYTES;         // one weight matrix (P planes)
  static constexpr uint32_t TMEM_COLS = (W * NH <= 128) ? 128 : (W * NH <= 256) ? 256 : 512;
  // CTAs per SM requested from the launch (TMEM permitting; the host sizes the partial slots with
  // mlp_tc_ctas_per_sm, which must agree): the three-plane split runs one CTA per SM
  static constexpr int MINB = (P == 1 && TMEM_COLS <= 256) ? 2 : 1;
  // activation buffers: h_1..h_{NH-1} (G_{l-1} written in place of h_{l-1}); G_NH takes h_1's
  // buffer and h_1 is recomputed for dW_2 -- unless one more buffer fits the per-CTA shared
  // memory (XBUF: W = 64, and W = 128 at 3 hidden layers), which then holds G_NH
  static constexpr int NBUF0 = NH - 1 > 2 ? NH - 1 : 2;
  static constexpr uint32_t FIXED = NWRES_() * WBUF + NDER * ACT_BYTES + 8192 + 4 * 3 * W + 4 * NH * W + 4 * (W + 4) +
                                    16 * kTB + 4 * CH * kTB + 16 * kTB + 64 + (STG > 0 ? 4 * (THREADS / 32) * 4 * (8 * 20 + 16) : 0);
  static constexpr bool XBUF = NH >= 3 && (NBUF0 + 1) * ABUF + FIXED <= (MINB == 2 ? 113u * 1024u : 232448u);
  static constexpr int NBUF = NBUF0 + (XBUF ? 1 : 0);
  static constexpr uint32_t oAct = 0;
  static constexpr uint32_t oWh = oAct + NBUF * ABUF;
  static constexpr uint32_t oDer = oWh + NWRES * WBUF;     // bf16 act'(z_l), l = 2..NH-1 (SiLU)
  static constexpr uint32_t oOnes = oDer + NDER * ACT_BYTES;  // bf16 [16][128] ones (MN-major)
  static constexpr uint32_t oXm = oOnes + 4096;            // bf16 [16][128] [1, x, y, z split]
  static constexpr uint32_t oW1 = oXm + 4096;              // fp32 [W][3]
  static constexpr uint32_t oBias = oW1 + 4 * 3 * W;       // fp32 [NH][W]
  static constexpr uint32_t oWo = oBias + 4 * NH * W;      // fp32 [W] + bo
  static constexpr uint32_t oX = oWo + 4 * (W + 4);        // fp32 [kTB][4]
  static constexpr uint32_t oUp = oX + 4 * 4 * kTB;        // fp32 [CH][kTB] u partials
  static constexpr uint32_t oU = oUp + 4 * CH * kTB;       // fp32 [kTB]
  static constexpr uint32_t oUb = oU + 4 * kTB;            // fp32 [kTB]
  static constexpr uint32_t oAux = oUb + 4 * kTB;          // fp32 [kTB]
  static constexpr uint32_t oItem = oAux + 4 * kTB;        // int  [kTB]
  static constexpr uint32_t oBar = oItem + 4 * kTB;        // mbarriers (MMA, weights) + tmem base
  static constexpr int SLD = 20;                          // staging row stride (floats): 16 columns + pad
  static constexpr int SPB = 8 * SLD + 16;                 // staging point-block stride: points p and p+1
                                                           // of one item instruction hit disjoint banks
  static constexpr uint32_t oStg = oBar + 64;              // fp32 [warp][4 points][SPB] (stable form, W = 64)
  static constexpr uint32_t bytes = oStg + (STG > 0 ? 4 * (THREADS / 32) * 4 * SPB : 0);
  static_assert(bytes == NBUF * ABUF + FIXED, "FIXED mirrors the carve");
  static_assert(bytes <= 232448, "shared memory");
  static constexpr int MDW = W;                            // M of the dW / tail MMAs (o-rows); at W = 64
                                                           // the M = 64 layout: unit o in TMEM lane
                                                           // 32 (o / 16) + o % 16 (scripts/r2/m64_probe.cu)
  static_assert(4 * (4 * 2 * W + 4) <= (int)ABUF * NBUF, "flush scratch");
  // theta offsets within one network (G17)
  static constexpr int64_t tW1 = 0, tB1 = 3 * W;
  __host__ __device__ static constexpr int64_t tWl(int l) { return 4 * W + (int64_t)(l - 2) * (W * W + W); }
  __host__ __device__ static constexpr int64_t tBl(int l) { return tWl(l) + W * W; }
  static constexpr int64_t tWo = 4 * W + (int64_t)NHH * (W * W + W);
  static constexpr int64_t tBo = tWo + W;
};

// one thread's 32 columns of a row -> bf16 core-matrix buffer
__device__ __forceinline__ void store_chunk_bf16(uint32_t buf, int row, int chunk, const float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    st_shared_v4(buf + core_off(kTB, row, chunk * 4 + q), pack_bf16(h[8 * q], h[8 * q + 1]),
                 pack_bf16(h[8 * q + 2], h[8 * q + 3]), pack_bf16(h[8 * q + 4], h[8 * q + 5]),
                 pack_bf16(h[8 * q + 6], h[8 * q + 7]));
}
// P planes of one thread's 32 columns of a row: plane p at buf + p * plane
template <int P>
__device__ __forceinline__ void store_chunk_planes(uint32_t buf, uint32_t plane, int row, int chunk, const float (&h)[32]) {
  if (P == 1) {
    store_chunk_bf16(buf, row, chunk, h);
    return;
  }
  float r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = h[j];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      w[j] = pack_bf16(r[2 * j], r[2 * j + 1]);
      r[2 * j] -= bf_lo(w[j]);         // exact: the rounding error of a bf16 rounding is an fp32
      r[2 * j + 1] -= bf_hi(w[j]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      st_shared_v4(buf + p * plane + core_off(kTB, row, chunk * 4 + q), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
}
__device__ __forceinline__ void load_chunk_bf16(uint32_t buf, int row, int chunk, float (&h)[32]);
// sum of the P planes (exact for the split of an fp32 value up to its last 2^-24 bits)
template <int P>
__device__ __forceinline__ void load_chunk_planes(uint32_t buf, uint32_t plane, int row, int chunk, float (&h)[32]) {
  load_chunk_bf16(buf + (P - 1) * plane, row, chunk, h);
#pragma unroll
  for (int p = P - 2; p >= 0; --p) {
    float t[32];
    load_chunk_bf16(buf + p * plane, row, chunk, t);
#pragma unroll
    for (int j = 0; j < 32; ++j) h[j] += t[j];
  }
}
__device__ __forceinline__ void load_chunk_bf16(uint32_t buf, int row, int chunk, float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
    ld_shared_v4(buf + core_off(kTB, row, chunk * 4 + q), w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[8 * q + 2 * e] = bf_lo(w[e]);
      h[8 * q + 2 * e + 1] = bf_hi(w[e]);
    }
  }
}

}  // namespace

#ifdef NBM_TC_TRACE
__device__ long long g_tc_trace[8][32];
#define TR(k)                                                                         \
  do {                                                                                \
    if (TRAIN && blockIdx.x == 0 && tid == 0 && t - t0 < 8) g_tc_trace[t - t0][k] = clock64(); \
  } while (0)
#else
#define TR(k) \
  do {        \
  } while (0)
#endif

// STAB: stencil tiles in the stable difference form (G27; bf16, tanh, training pass only)
// stable maps staged through shared memory, one thread per (point, column) (W = 64, where the
// staging tile fits next to two CTAs per SM); W = 128 uses the in-register octet maps
template <int W, bool STAB>
constexpr int tc_stage_cols() { return (STAB && W == 64) ? 32 : 0; }

template <int W, int NH, int ACT, bool TRAIN, int P = 1, bool STAB = false>
__global__ void __launch_bounds__(TcLayout<W, NH, ACT, P, tc_stage_cols<W, STAB>()>::THREADS,
                                  TcLayout<W, NH, ACT, P, tc_stage_cols<W, STAB>()>::MINB) k_mlp_tc(const MlpParams prm) {
  using L = TcLayout<W, NH, ACT, P, tc_stage_cols<W, STAB>()>;
  constexpr bool SST = tc_stage_cols<W, STAB>() > 0;
  static_assert(!STAB || (P == 1 && ACT == NBM_ACT_TANH && TRAIN), "stable form: bf16 tanh training pass");
  constexpr int TPT = STAB ? kTPTS : kTPT;   // stencil points per tile
  constexpr uint32_t AP = L::ACT_BYTES, WP = L::WMAT_BYTES;   // plane strides (P = 3)
  // activation: MUFU tanh.approx for the bf16 path (G16), accurate tanhf for the fp32 split (G15)
  auto act_tanh = [](float x) { return P == 3 ? tanhf(x) : tanh_fast(x); };
  constexpr bool SILU = L::SILU, STREAM = L::STREAM;
  constexpr int NHH = L::NHH;
  constexpr int NT = L::NT;
  constexpr int THREADS = L::THREADS;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = tc::smem_u32(smem);
  float* sW1 = reinterpret_cast<float*>(smem + L::oW1);
  float* sBias = reinterpret_cast<float*>(smem + L::oBias);
  float* sWo = reinterpret_cast<float*>(smem + L::oWo);
  float* sX = reinterpret_cast<float*>(smem + L::oX);
  float* sUp = reinterpret_cast<float*>(smem + L::oUp);
  float* sU = reinterpret_cast<float*>(smem + L::oU);
  float* sUb = reinterpret_cast<float*>(smem + L::oUb);
  float* sAux = reinterpret_cast<float*>(smem + L::oAux);
  int* sItem = reinterpret_cast<int*>(smem + L::oItem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* wbar = reinterpret_cast<uint64_t*>(smem + L::oBar + 8);
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(smem + L::oBar + 16);
  uint64_t* dwbar = reinterpret_cast<uint64_t*>(smem + L::oBar + 24);   // dW MMA of the backward step
  __shared__ int segTiles[kNumSeg], segCnt[kNumSeg], segStart[kNumSeg];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, chunk = warp >> 2;
  const int row = quad * 32 + lane;                       // tile row = TMEM lane
  const uint32_t tlane = (uint32_t)(quad * 32) << 16;
  const uint32_t ccol = (uint32_t)(chunk * 32);            // this thread's column chunk
  // the dW / tail unit o held in this thread's TMEM lane (-1: none): lane = o for M = 128, lane
  // 32 (o / 16) + o % 16 for the M = 64 layout of W = 64
  const int o_lane = L::MDW == 64 ? (lane < 16 ? quad * 16 + lane : -1) : (row < W ? row : -1);
  if (tid < kNumSeg) {
    int c = prm.counts[prm.cnt_slot[tid]];
    segCnt[tid] = c;
    segStart[tid] = prm.start_slot[tid] >= 0 ? prm.counts[prm.start_slot[tid]] : 0;
    int per = prm.seg.kind[tid] == kSegStencil ? TPT : kTB;
    segTiles[tid] = (c + per - 1) / per;
  }
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(wbar, 1);
    tc::mbar_init(dwbar, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(sTmem, L::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *sTmem;

  int firstTile[kNumSeg + 1];
  int total = 0;
#pragma unroll
  for (int s = 0; s < kNumSeg; ++s) { firstTile[s] = total; total += segTiles[s]; }
  firstTile[kNumSeg] = total;
  const int G = gridDim.x, cta = blockIdx.x;
  const int t0 = (int)((int64_t)total * cta / G), t1 = (int)((int64_t)total * (cta + 1) / G);

  constexpr uint32_t LBO_ACT = kTB * 16, LBO_W = W * 16;
  const uint32_t aAct = sbase + L::oAct, aWh = sbase + L::oWh;
  constexpr uint32_t ID_FWD = tc::idesc_bf16(kTB, W, 0, 0);   // A K-major, B K-major
  constexpr uint32_t ID_DH = tc::idesc_bf16(kTB, W, 0, 1);    // A K-major, B MN-major
  constexpr uint32_t ID_DW = tc::idesc_bf16(L::MDW, W, 1, 1);    // A MN-major, B MN-major
  constexpr uint32_t ID_TAIL = tc::idesc_bf16(L::MDW, 16, 1, 1); // M = W, N = 16, both MN-major
  const uint32_t aOnes = sbase + L::oOnes, aXm = sbase + L::oXm;
  uint32_t phase = 0, dwphase = 0;
  // streamed weights (SiLU): the stage holds W_{wl} of net wnet once wbar completes
  uint32_t wphase = 0;
  int wnet = -1, wl = -1;
  bool wpending = false;
  // the MMA-issuing warp (warp 0, converged): every lane keeps the same bookkeeping
  auto wload = [&](int net, int l) {   // warp 0 only; the stage must be free (no MMA in flight)
    if (!STREAM || (net == wnet && l == wl)) return;
    if (lane == 0) {
      // the P planes of W_l: the packed image holds [net][l][plane][W x W] (launch_pack_weights)
      tc::mbar_arrive_expect_tx(wbar, L::WBUF);
      tc::bulk_copy_g2s(aWh, prm.wimg + ((int64_t)net * NHH + (l - 2)) * P * W * W, L::WBUF, wbar);
    }
    wnet = net;
    wl = l;
    wpending = true;
  };
  auto wwait = [&]() {   // warp 0 only, before an MMA reading the stage
    if (STREAM && wpending) {
      tc::mbar_wait(wbar, wphase);
      wphase ^= 1;
      wpending = false;
    }
  };
  auto wmat = [&](int l) -> uint32_t { return STREAM ? aWh : aWh + (l - 2) * L::WBUF; };
  const uint32_t aDer = sbase + L::oDer;
  {  // constant operands of the tail reductions
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem + L::oOnes);
    uint32_t* xm = reinterpret_cast<uint32_t*>(smem + L::oXm);
    for (int i = tid; i < 1024; i += THREADS) {
      ones[i] = 0x3F803F80u;   // bf16 1.0 pairs
      xm[i] = 0u;
    }
    tc::fence_proxy_async_smem();
  }

  // transposed gradients (lane = column chunk*32 + lane over this warp's 32 rows):
  // gWo = wo, gBN = b_NH; gbo = bo (chunk-0 warps).  Tensor-core reduced gradients
  // (chunk-0 threads, unit o = row): tg[0..NH-3] = b_2..b_{NH-1}, tg[NH-2] = b_1,
  // tg[NH-1..NH+1] = W1[o][0..2].
  float gWo = 0.0f, gBN = 0.0f, gbo = 0.0f;
  float tg[NT];
  double lossAcc = 0.0;
  int curNet = -1;
  bool touched[2] = {false, false};
  bool dwFresh = true;
  bool tailPending = false;   // the last tile's tail MMAs are in flight (read before buffer 0 is reused)

  auto flush = [&](int net) {
    float* out = prm.part + ((int64_t)net * G + cta) * prm.p_stride;
    NBM_CHECK(((int64_t)net * G + cta + 1) * prm.p_stride <= prm.part_len);
    if (!dwFresh) {
      tc::tc_fence_after();
#pragma unroll 1
      for (int l = 2; l <= NH; ++l) {
        float v[32];
        tc::tmem_ld32(tmem + tlane + (uint32_t)(W * (l - 1)) + ccol, v);   // dW_l[o = o_lane][i]
        if (o_lane >= 0) {
          float4* dst = reinterpret_cast<float4*>(out + L::tWl(l) + (int64_t)o_lane * W + ccol);
#pragma unroll
          for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    } else {
      for (int l = 2; l <= NH; ++l)
        for (int i = tid; i < W * W; i += THREADS) out[L::tWl(l) + i] = 0.0f;
    }
    // tensor-core reduced gradients: one thread per unit o (chunk-0 warps)
    if (chunk == 0 && o_lane >= 0) {
      const int o = o_lane;
#pragma unroll
      for (int l = 2; l <= NH - 1; ++l) out[L::tBl(l) + o] = tg[l - 2];
      out[L::tB1 + o] = tg[NH - 2];
      out[L::tW1 + 3 * o + 0] = tg[NH - 1];
      out[L::tW1 + 3 * o + 1] = tg[NH];
      out[L::tW1 + 3 * o + 2] = tg[NH + 1];
    }
    // transposed gradients: 4 quadrant-warps per column chunk, summed in quadrant order
    float* scr = reinterpret_cast<float*>(smem + L::oAct);   // [4][2][W] + [4] bo
    __syncthreads();
    scr[(quad * 2 + 0) * W + ccol + lane] = gBN;
    scr[(quad * 2 + 1) * W + ccol + lane] = gWo;
    if (chunk == 0 && lane == 0) scr[8 * W + quad] = gbo;
    __syncthreads();
    for (int i = tid; i < 2 * W; i += THREADS) {
      const int v = i / W, col = i % W;
      const float s = ((scr[(0 * 2 + v) * W + col] + scr[(1 * 2 + v) * W + col]) + scr[(2 * 2 + v) * W + col]) +
                      scr[(3 * 2 + v) * W + col];
      out[(v == 0 ? (NH == 1 ? L::tB1 : L::tBl(NH)) : L::tWo) + col] = s;
    }
    if (tid == 0) out[L::tBo] = ((scr[8 * W] + scr[8 * W + 1]) + scr[8 * W + 2]) + scr[8 * W + 3];
    __syncthreads();
    touched[net] = true;
  };

  auto load_net = [&](int net) {
    const float* th = prm.theta + (int64_t)net * prm.p_net;
    for (int i = tid; i < 3 * W; i += THREADS) sW1[i] = th[L::tW1 + i];
    for (int i = tid; i < W; i += THREADS) {
      sBias[i] = th[L::tB1 + i];
      for (int l = 2; l <= NH; ++l) sBias[(l - 1) * W + i] = th[L::tBl(l) + i];
      sWo[i] = th[L::tWo + i];
    }
    if (tid == 0) sWo[W] = th[L::tBo];
    for (int l = 0; l < (STREAM ? 0 : NHH); ++l) {   // hidden weights -> bf16 core-matrix layout
      const float* Wl = th + L::tWl(l + 2);
      for (int q = tid; q < W * (W / 8); q += THREADS) {
        const int o = q / (W / 8), c8 = q % (W / 8);
        const float* src = Wl + (int64_t)o * W + c8 * 8;   // net+ theta is not 16-B aligned
        float r[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = src[e];
#pragma unroll
        for (int p = 0; p < P; ++p) {   // plane p of the exact bf16 split (P = 1: the RNE bf16 copy)
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            w[e] = pack_bf16(r[2 * e], r[2 * e + 1]);
            r[2 * e] -= bf_lo(w[e]);
            r[2 * e + 1] -= bf_hi(w[e]);
          }
          st_shared_v4(aWh + l * L::WBUF + p * WP + core_off(W, o, c8), w[0], w[1], w[2], w[3]);
        }
      }
    }
    tc::fence_proxy_async_smem();
    if (warp == 0) {   // (a forward-only pass may still be prefetching the previous network's W_2)
      wwait();
      wload(net, 2);
    }
#pragma unroll
    for (int v = 0; v < NT; ++v) tg[v] = 0.0f;
    gWo = gBN = gbo = 0.0f;
  };

  // one GEMM of ksteps x K=16 on the tensor core, issued by warp 0 (one elected lane); the
  // descriptors advance by the K step in their 16-byte address field
  auto gemm = [&](uint32_t dcol, uint32_t a0, uint32_t a_step, uint32_t a_lbo, uint32_t a_sbo, uint32_t b0,
                  uint32_t b_step, uint32_t b_lbo, uint32_t b_sbo, uint32_t idesc, int ksteps, bool acc) {
    const uint64_t ad = tc::sdesc(a0, a_lbo, a_sbo), bd = tc::sdesc(b0, b_lbo, b_sbo);
#pragma unroll 4
    for (int s = 0; s < ksteps; ++s)
      tc::mma_bf16_w(tmem + dcol, ad + (uint64_t)((s * a_step) >> 4), bd + (uint64_t)((s * b_step) >> 4), idesc,
                     (acc || s > 0) ? 1u : 0u);
  };
  // the plane products of a split GEMM (P = 3): planes i + j <= 2, the smallest first; P = 1: one
  auto gemm_p = [&](uint32_t dcol, uint32_t a0, uint32_t a_step, uint32_t a_lbo, uint32_t a_sbo, uint32_t a_pl,
                    uint32_t b0, uint32_t b_step, uint32_t b_lbo, uint32_t b_sbo, uint32_t b_pl, uint32_t idesc,
                    int ksteps, bool acc) {
    if (P == 1) {
      gemm(dcol, a0, a_step, a_lbo, a_sbo, b0, b_step, b_lbo, b_sbo, idesc, ksteps, acc);
      return;
    }
    const int pi[6] = {2, 1, 0, 1, 0, 0}, pj[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll 1
    for (int q = 0; q < 6; ++q)
      gemm(dcol, a0 + pi[q] * a_pl, a_step, a_lbo, a_sbo, b0 + pj[q] * b_pl, b_step, b_lbo, b_sbo, idesc, ksteps,
           acc || q > 0);
  };
  auto wait_mma = [&]() {
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::tc_fence_after();
  };
  // ---- stable maps through shared memory (SST, W = 64), warp-local: a warp holds its lane
  // quadrant's 4 points (rows 8p..8p+7) x its 32-column chunk, so it stages them in its own
  // [32][SLD] fp32 block in two 16-column halves, each lane maps two (point, column) items in
  // place, and the lanes read their rows back: __syncwarp only, no CTA barriers ----
  float* sStg = reinterpret_cast<float*>(smem + L::oStg) + warp * 4 * L::SPB;
  constexpr int SLD = L::SLD, SPB = L::SPB;
  float* myStg = sStg + (lane >> 3) * SPB + (lane & 7) * SLD;   // this lane's row
  auto stage_half = [&](float (&v)[32], int hf, auto&& item) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<float4*>(myStg + 4 * q) =
          make_float4(v[16 * hf + 4 * q], v[16 * hf + 4 * q + 1], v[16 * hf + 4 * q + 2], v[16 * hf + 4 * q + 3]);
    __syncwarp();
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
      const int it = lane + 32 * k2, p = it >> 4, c = it & 15;
      item(p, c, (int)ccol + 16 * hf + c, 4 * quad + p);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 f = *reinterpret_cast<const float4*>(myStg + 4 * q);
      v[16 * hf + 4 * q] = f.x; v[16 * hf + 4 * q + 1] = f.y; v[16 * hf + 4 * q + 2] = f.z; v[16 * hf + 4 * q + 3] = f.w;
    }
    __syncwarp();
  };
  // forward: v = the row's raw pre-activation (no bias) -> a, P_d, Q_d; bl = the layer's biases
  auto stage_fwd = [&](float (&v)[32], const float* bl) {
#pragma unroll   // compile-time halves: v stays in registers
    for (int hf = 0; hf < 2; ++hf)
      stage_half(v, hf, [&](int p, int c, int col, int k) {
        float* h = sStg + p * SPB + c;
        const float t = tanh_fast(h[0] + bl[col]);
        const float s2 = fmaf(-t, t, 1.0f);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const float pp = h[(1 + d) * SLD], D = h[(4 + d) * SLD];
          const float gp = stab::stab_g(t, s2, pp), gm = stab::stab_g(t, s2, D - pp);
          h[(1 + d) * SLD] = fmaf(s2, pp, gp);
          h[(4 + d) * SLD] = fmaf(s2, D, gp) + gm;
        }
        h[0] = t;
        h[7 * SLD] = 0.0f;
      });
  };
  // backward: top (hbufA == 0): v = h_NH (fp32), upstream ub wo; else v = the upstream products
  // and the activations are the bf16 copies in hbufA.  v <- (g_z, g_p, g_D)
  auto stage_bwd = [&](float (&v)[32], uint32_t hbufA) {
    const uint16_t* hb16 = reinterpret_cast<const uint16_t*>(smem + (hbufA - sbase));
#pragma unroll   // compile-time halves: v stays in registers
    for (int hf = 0; hf < 2; ++hf)
      stage_half(v, hf, [&](int p, int c, int col, int k) {
        float* g = sStg + p * SPB + c;
        float H[7], R[7];
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          if (hbufA) {
            H[j] = __uint_as_float((uint32_t)hb16[(core_off(kTB, 8 * k + j, col >> 3) + (col & 7) * 2) >> 1] << 16);
            R[j] = g[j * SLD];
          } else {
            H[j] = g[j * SLD];
            R[j] = sUb[8 * k + j] * sWo[col];
          }
        }
        const float t = H[0], t2 = t + t;
        float gz = R[0] * fmaf(-t, t, 1.0f);
        float gp[3], gd[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const float P = H[1 + d], Q = H[4 + d], M = Q - P, gP = R[1 + d], gQ = R[4 + d];
          gz -= gP * P * (t2 + P) + gQ * fmaf(t2, Q, fmaf(P, P, M * M));
          const float tp = t + P, tm = t + M;
          gp[d] = fmaf(gP, fmaf(-tp, tp, 1.0f), gQ * (M - P) * (t2 + M + P));
          gd[d] = gQ * fmaf(-tm, tm, 1.0f);
        }
        g[0] = gz;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          g[(1 + d) * SLD] = gp[d];
          g[(4 + d) * SLD] = gd[d];
        }
        g[7 * SLD] = 0.0f;
      });
  };

  // layer 1 for this thread's 32 columns: h = tanh(W1 x + b1); on a stable-form tile the row
  // input is x (centre), h e_d (P_d rows) or 0 (Q_d rows, pad) and the bias enters the centre only
  auto layer1 = [&](float x0, float x1, float x2, float (&h)[32], bool stab) {
    if (STAB && stab) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = ccol + j;
        h[j] = fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, sW1[3 * n] * x0));
      }
      if (SST) stage_fwd(h, sBias);
      else {   // the octet maps in two 16-column halves (bounded register working set)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float a16[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) a16[j] = h[16 * hf + j];
          stab::stab_fwd<16>(a16, sBias + ccol + 16 * hf, lane);
#pragma unroll
          for (int j = 0; j < 16; ++j) h[16 * hf + j] = a16[j];
        }
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = ccol + j;
      const float z = fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, fmaf(sW1[3 * n], x0, sBias[n])));
      h[j] = SILU ? z * sigmoid_fast(z) : act_tanh(z);
    }
  };

  // global loads of one tile for thread tid < kTB: the item slot `tid` (index + aux) and the
  // coordinates of tile row `tid` (stencil arm generated on the fly).  Issued one tile ahead.
  struct Fetch { int item; float aux, x0, x1, x2; };
  auto fetch = [&](int tt) -> Fetch {
    Fetch f{-1, 0.0f, 0.0f, 0.0f, 0.0f};
    if (tt >= t1 || tid >= kTB) return f;
    int sg = 0;
    while (tt >= firstTile[sg + 1]) ++sg;
    const int knd = prm.seg.kind[sg];
    const int pr = knd == kSegStencil ? TPT : kTB;
    const int fst = (tt - firstTile[sg]) * pr;
    const int nv = min(pr, segCnt[sg] - fst);
    const int* its = prm.seg.items[sg] + segStart[sg];
    if (tid < pr && tid < nv) {
      f.item = item_at(prm.seg, sg, its, fst + tid);
      f.aux = prm.aux_by_item[sg] ? prm.seg.aux[sg][f.item] : prm.seg.aux[sg][segStart[sg] + fst + tid];
    }
    if (STAB && knd == kSegStencil) {   // row 8k + jr: x, h e_1..3 (P_d), 0 (Q_d, pad)
      const int k = tid >> 3, jr = tid & 7;
      if (k < nv && jr == 0) {
        const float* src = prm.seg.src[sg] + 3 * (int64_t)item_at(prm.seg, sg, its, fst + k);
        f.x0 = src[0]; f.x1 = src[1]; f.x2 = src[2];
      } else if (k < nv && jr < 4) {
        if (jr == 1) f.x0 = prm.h; else if (jr == 2) f.x1 = prm.h; else f.x2 = prm.h;
      }
    } else if (knd == kSegStencil) {
      const int j = tid / kTPT, p = tid - j * kTPT;
      if (j < 7 && p < nv) {
        const float* src = prm.seg.src[sg] + 3 * (int64_t)item_at(prm.seg, sg, its, fst + p);
        f.x0 = src[0]; f.x1 = src[1]; f.x2 = src[2];
        if (j > 0) {   // arms +x, -x, +y, -y, +z, -z (exact on the lattice)
          const float hs = (j & 1) ? prm.h : -prm.h;
          if (j <= 2) f.x0 = __fadd_rn(f.x0, hs); else if (j <= 4) f.x1 = __fadd_rn(f.x1, hs); else f.x2 = __fadd_rn(f.x2, hs);
        }
      }
    } else if (tid < nv) {
      const float* src = prm.seg.src[sg] + 3 * (int64_t)item_at(prm.seg, sg, its, fst + tid);
      f.x0 = src[0]; f.x1 = src[1]; f.x2 = src[2];
    }
    return f;
  };
  Fetch cur = fetch(t0);
  // completion of the tile-tail reductions: fold them into the register accumulators
  auto tail_collect = [&]() {
    wait_mma();
    if (chunk == 0) {
      float v[16];
#pragma unroll
      for (int l = 2; l <= NH - 1; ++l) {
        tc::tmem_ld16(tmem + tlane + (uint32_t)(16 * (l - 2)), v);
        tg[l - 2] += v[0];
      }
      tc::tmem_ld16(tmem + tlane + (uint32_t)(16 * (NH - 2)), v);
      tg[NH - 2] += v[0];
      if (P == 1) {
        tg[NH - 1] += v[1] + v[2];
        tg[NH] += v[3] + v[4];
        tg[NH + 1] += v[5] + v[6];
      } else {
        tg[NH - 1] += (v[3] + v[2]) + v[1];
        tg[NH] += (v[6] + v[5]) + v[4];
        tg[NH + 1] += (v[9] + v[8]) + v[7];
      }
    }
    tailPending = false;
  };

  int seg = 0;
  for (int t = t0; t < t1; ++t) {
    while (t >= firstTile[seg + 1]) ++seg;
    const int kind = prm.seg.kind[seg], net = prm.seg.net[seg];
    const int lt = t - firstTile[seg];
    const int per = kind == kSegStencil ? TPT : kTB;
    const int first = lt * per;
    const int nvalid = min(per, segCnt[seg] - first);
    const bool stab = STAB && kind == kSegStencil;                 // warp-uniform
    const bool centre = !stab || (row & 7) == 0;                   // rows that carry the biases
    if (net != curNet) {
      if (tailPending) {
        tail_collect();
        tc::tc_fence_before();
        __syncthreads();
      }
      if (TRAIN && curNet >= 0) flush(curNet);
      load_net(net);
      dwFresh = true;
      curNet = net;
      __syncthreads();
    }
    // ---- gather: items, aux and the row's coordinates were prefetched during the previous tile ----
    if (tid < kTB) {
      if (tid < per) {
        sItem[tid] = cur.item;
        sAux[tid] = cur.aux;
      }
      sX[4 * tid] = cur.x0; sX[4 * tid + 1] = cur.x1; sX[4 * tid + 2] = cur.x2;
    }
    __syncthreads();
    TR(0);
    const float x0 = sX[4 * row], x1 = sX[4 * row + 1], x2 = sX[4 * row + 2];
    {  // ---- layer 1 -> bf16 h1 (buffer 0; the previous tile's tail MMAs may still read it) ----
      float h[32];
      layer1(x0, x1, x2, h, stab);
      if (tailPending) tail_collect();
      store_chunk_planes<P>(aAct, AP, row, chunk, h);
    }
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    TR(1);
    // ---- hidden layers 2..NH on the tensor cores ----
    Fetch nxt;
#pragma unroll 1
    for (int l = 2; l <= NH; ++l) {
      if (warp == 0) {
        wwait();
        tc::tc_fence_after();
        gemm_p(0, aAct + (l - 2) * L::ABUF, 2 * LBO_ACT, LBO_ACT, 128, AP, wmat(l), 2 * LBO_W, LBO_W, 128, WP, ID_FWD,
               W / 16, false);
        tc::mma_commit_w(bar);
      }
      if (!TRAIN && l == 2) nxt = fetch(t + 1);   // the next tile's loads overlap this tile
      wait_mma();
      // prefetch the next layer's weights; a forward-only pass ends the tile on W_NH, so the next
      // tile's W_2 is loaded here (the training pass reloads it through its backward)
      if (warp == 0 && (l < NH || !TRAIN)) wload(curNet, l < NH ? l + 1 : 2);
      TR(2 + 2 * (l - 2));
      float v[32];
      const float* bl = sBias + (l - 1) * W + ccol;
      if (STAB && stab && !SST) {   // the octet maps in two 16-column halves (bounded register working set)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float a16[16];
          tc::tmem_ld16(tmem + tlane + ccol + 16 * hf, a16);
          stab::stab_fwd<16>(a16, bl + 16 * hf, lane);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[16 * hf + j] = a16[j];
        }
      } else {
        tc::tmem_ld32(tmem + tlane + ccol, v);
      }
      if (STAB && stab) {
        if (SST) stage_fwd(v, sBias + (l - 1) * W);
      } else if (!SILU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = act_tanh(v[j] + bl[j]);
      }
      if (l < NH) {
        if (SILU) {
          float d[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float z = v[j] + bl[j], sg = sigmoid_fast(z);
            v[j] = z * sg;
            d[j] = sg * fmaf(z, 1.0f - sg, 1.0f);   // SiLU'(z)
          }
          if (TRAIN && l >= 2 && l <= NH - 1) store_chunk_bf16(aDer + (l - 2) * L::ACT_BYTES, row, chunk, d);   // P = 1
        }
        store_chunk_planes<P>(aAct + (l - 1) * L::ABUF, AP, row, chunk, v);
        tc::fence_proxy_async_smem();
      } else {
        float z[32];
        if (SILU) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            z[j] = v[j] + bl[j];
            v[j] = z[j] * sigmoid_fast(z[j]);
          }
        }
        float up = 0.0f;
#pragma unroll
        for (int j = 0; j < 32; ++j) up = fmaf(sWo[ccol + j], v[j], up);
        sUp[chunk * kTB + row] = up;
        if (TRAIN) {   // keep fp32 h_NH (tanh) or z_NH (SiLU) for the backward
          if (SILU) tc::tmem_st32(tmem + tlane + ccol, z);
          else tc::tmem_st32(tmem + tlane + ccol, v);
        }
      }
      tc::tc_fence_before();
      __syncthreads();
      TR(3 + 2 * (l - 2));
    }
    if (tid < kTB) {
      float u = sUp[tid];
#pragma unroll
      for (int c = 1; c < L::CH; ++c) u += sUp[c * kTB + tid];
      if (!stab || (tid & 7) == 0) u += sWo[W];   // differences carry no output bias
      if (!TRAIN && tid < nvalid) prm.u_out[sItem[tid]] = u;
      sU[tid] = u;
    }
    __syncthreads();
    TR(8);
    if (!TRAIN) {
      cur = nxt;
      continue;
    }
    // ---- residual epilogue -> cotangents (S4) ----
    if (stab) {   // r = c_c u + c_hat sum_d DU_d - b/d (G27); cotangents c_c 2r/N (centre), c_hat 2r/N (Q_d)
      if (tid < kTB) {
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
      if (tid < kTPT) {
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
          for (int j = 1; j < 7; ++j) acc = fmaf(cj[j - 1], sU[j * kTPT + tid], acc);
          r = acc - sAux[tid];
          lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;
        }
        const float rc = prm.two_over_n * r;
        sUb[tid] = rc;
#pragma unroll
        for (int j = 1; j < 7; ++j) sUb[j * kTPT + tid] = rc * cj[j - 1];
      } else if (tid >= 7 * kTPT && tid < kTB) {
        sUb[tid] = 0.0f;
      }
    } else if (tid < kTB) {
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
    TR(9);
    const float ub = sUb[row];
    if (chunk == 0) {   // output bias
      float b = centre ? ub : 0.0f;
#pragma unroll
      for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
      gbo += b;
    }
    // ---- output layer backward: dwo += ub h_NH; G_NH = ub wo (1 - h_NH^2) -> bf16 ----
    const uint32_t gbufNH = L::XBUF ? aAct + (NH - 1) * L::ABUF : (NH == 2) ? aAct + L::ABUF : aAct;
    {
      float hv[32], v[32];
      tc::tmem_ld32(tmem + tlane + ccol, hv);
      if (SILU) {   // hv holds z_NH: v = h, hv = act'
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float z = hv[j], sg = sigmoid_fast(z);
          v[j] = z * sg;
          hv[j] = sg * fmaf(z, 1.0f - sg, 1.0f);
        }
      } else if (STAB && stab) {   // G_NH = the backward map of (ub wo) through the last activation
        if (SST) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = hv[j];
          stage_bwd(hv, 0u);
        } else {   // w_o's gradient first, then the octet maps in 16-column halves
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = hv[j] * ub;
          gWo += warp_transpose_sum(v, lane);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            float a16[16], g16[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              a16[j] = hv[16 * hf + j];
              g16[j] = ub * sWo[ccol + 16 * hf + j];
            }
            stab::stab_bwd<16>(g16, a16, lane);
#pragma unroll
            for (int j = 0; j < 16; ++j) hv[16 * hf + j] = g16[j];
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] = hv[j];
          hv[j] = 1.0f - hv[j] * hv[j];
        }
      }
      if (!(STAB && stab && !SST)) {   // (the octet-map branch above formed it already)
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= ub;
        gWo += warp_transpose_sum(v, lane);
      }
      if (!(STAB && stab)) {
#pragma unroll
        for (int j = 0; j < 32; ++j) hv[j] *= ub * sWo[ccol + j];
      }
      store_chunk_planes<P>(gbufNH, AP, row, chunk, hv);
      if (!centre) {   // b_NH: centre rows only
#pragma unroll
        for (int j = 0; j < 32; ++j) hv[j] = 0.0f;
      }
      gBN += warp_transpose_sum(hv, lane);
    }
    tc::tc_fence_before();
    tc::fence_proxy_async_smem();
    __syncthreads();
    TR(10);
    // ---- hidden layers backward ----
#pragma unroll 1
    for (int l = NH; l >= 2; --l) {
      const uint32_t gbuf = (l == NH) ? gbufNH : aAct + (l - 1) * L::ABUF;   // G_l
      const uint32_t hbuf = aAct + (l - 2) * L::ABUF;                        // h_{l-1}
      if (warp == 0) {
        wwait();
        tc::tc_fence_after();
        // acc = G_l W_l: A = G (K-major), B = W_l (N = i, K = o: MN-major); its epilogue starts
        // while the dW MMA below still runs
        gemm_p(0, gbuf, 2 * LBO_ACT, LBO_ACT, 128, AP, wmat(l), 256, 128, LBO_W, WP, ID_DH, W / 16, false);
        tc::mma_commit_w(bar);
        // dW_l += G_l^T h_{l-1}: A = G (M = o, MN-major), B = h (N = i, MN-major), K = rows
        gemm_p((uint32_t)(W * (l - 1)), gbuf, 256, 128, LBO_ACT, AP, hbuf, 256, 128, LBO_ACT, AP, ID_DW, kTB / 16,
               !dwFresh);
        tc::mma_commit_w(dwbar);
      }
      if (l == NH) nxt = fetch(t + 1);   // the next tile's loads, under the longest MMA phase
      wait_mma();
      if (warp == 0) wload(curNet, l > 2 ? l - 1 : 2);   // next GEMM's weights (W_2 for the next tile)
      TR(11 + 2 * (NH - l));
      // G_{l-1} = acc * (1 - h~^2), h~ = the bf16 operand copy of h_{l-1} (own row, chunk)
      float v[32], hq[32];
      if (!(STAB && stab && !SST)) tc::tmem_ld32(tmem + tlane + ccol, v);
      if (STAB && stab) {                  // the backward map of the difference form (G27)
        if (SST) {
          stage_bwd(v, hbuf);
        } else {   // the octet maps in two 16-column halves (a bounded register working set)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            float a16[16], h16[16];
            tc::tmem_ld16(tmem + tlane + ccol + 16 * hf, a16);
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              uint32_t w[4];
              ld_shared_v4(hbuf + core_off(kTB, row, chunk * 4 + 2 * hf + qq), w[0], w[1], w[2], w[3]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                h16[8 * qq + 2 * e] = bf_lo(w[e]);
                h16[8 * qq + 2 * e + 1] = bf_hi(w[e]);
              }
            }
            stab::stab_bwd<16>(a16, h16, lane);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[16 * hf + j] = a16[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) hq[j] = 1.0f;
      } else if (!SILU) {                  // tanh' = 1 - h~^2 (bf16 operand copy)
        load_chunk_planes<P>(hbuf, AP, row, chunk, hq);
#pragma unroll
        for (int j = 0; j < 32; ++j) hq[j] = 1.0f - hq[j] * hq[j];
      } else if (l - 1 >= 2) {             // SiLU': stored bf16 derivative
        load_chunk_bf16(aDer + (l - 3) * L::ACT_BYTES, row, chunk, hq);
      } else if (L::NDER >= 2 && !L::XBUF) {   // SiLU' of layer 1 (fp32), formed with h1 at l = 3
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
            ld_shared_v4(aDer + b * L::ACT_BYTES + core_off(kTB, row, chunk * 4 + q), w[0], w[1], w[2], w[3]);
#pragma unroll
            for (int e = 0; e < 4; ++e) hq[16 * b + 4 * q + e] = __uint_as_float(w[e]);
          }
      } else {                             // SiLU' of layer 1: recomputed exactly from x
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = ccol + j;
          const float z = fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, fmaf(sW1[3 * n], x0, sBias[n])));
          const float sg = sigmoid_fast(z);
          hq[j] = sg * fmaf(z, 1.0f - sg, 1.0f);
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= hq[j];
      tc::mbar_wait(dwbar, dwphase);           // dW_l has read h_{l-1} (and G_l)
      dwphase ^= 1;
      store_chunk_planes<P>(hbuf, AP, row, chunk, v);   // G_{l-1} in place: h_{l-1} is consumed
      if (l - 1 == 2 && NH >= 3 && !L::XBUF) {   // h1 again for dW_2 (buffer 0's G_NH is consumed)
        float h[32];
        if (SILU && L::NDER >= 2) {
          // with SiLU'(z1) in fp32 for the l = 2 epilogue, in this thread's own (row, chunk)
          // blocks of the two act' buffers (layer 2's was read above, layer 3's at l = 4)
          float d[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = ccol + j;
            const float z = fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, fmaf(sW1[3 * n], x0, sBias[n])));
            const float sg = sigmoid_fast(z);
            h[j] = z * sg;
            d[j] = sg * fmaf(z, 1.0f - sg, 1.0f);
          }
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_shared_v4(aDer + b * L::ACT_BYTES + core_off(kTB, row, chunk * 4 + q), __float_as_uint(d[16 * b + 4 * q]),
                           __float_as_uint(d[16 * b + 4 * q + 1]), __float_as_uint(d[16 * b + 4 * q + 2]),
                           __float_as_uint(d[16 * b + 4 * q + 3]));
        } else {
          layer1(x0, x1, x2, h, stab);
        }
        store_chunk_planes<P>(aAct, AP, row, chunk, h);
      }
      if (l == 2 && chunk == 0) {   // tail operand row: [1, x_hi, x_lo, y_hi, y_lo, z_hi, z_lo, 0]
        const float xh = __bfloat162float(__float2bfloat16_rn(x0)), yh = __bfloat162float(__float2bfloat16_rn(x1)),
                    zh = __bfloat162float(__float2bfloat16_rn(x2));
        if (P == 1) {   // the bias column is 1 on the rows that carry biases (centre rows, G27)
          const float cm = centre ? 1.0f : 0.0f;
          st_shared_v4(aXm + row * 16, pack_bf16(cm, xh), pack_bf16(x0 - xh, yh), pack_bf16(x1 - yh, zh),
                       pack_bf16(x2 - zh, 0.0f));
          if (STAB) {   // ones operand of db_2..db_{NH-1}: the same row mask
            const uint32_t m2 = pack_bf16(cm, cm);
            st_shared_v4(aOnes + row * 16, m2, m2, m2, m2);
          }
        } else {   // [1, x1, x2, x3, y1, y2, y3, z1 | z2, z3, 0...]: each coordinate as three bf16 planes
          float pl[9];
          const float xs[3] = {x0, x1, x2};
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float r = xs[c];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              pl[3 * c + q] = __bfloat162float(__float2bfloat16_rn(r));
              r -= pl[3 * c + q];
            }
          }
          st_shared_v4(aXm + row * 16, pack_bf16(1.0f, pl[0]), pack_bf16(pl[1], pl[2]), pack_bf16(pl[3], pl[4]),
                       pack_bf16(pl[5], pl[6]));
          st_shared_v4(aXm + 2048 + row * 16, pack_bf16(pl[7], pl[8]), 0u, 0u, 0u);
        }
      }
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      TR(12 + 2 * (NH - l));
    }
    // ---- tile tail: bias gradients of layers 1..NH-1 and dW_1 on the tensor core ----
    if (warp == 0) {
      tc::tc_fence_after();
      for (int l = 2; l <= NH - 1; ++l)   // db_l = G_l^T 1   (G_l in buffer l-1; every plane of G)
        for (int p = 0; p < P; ++p)
          gemm((uint32_t)(16 * (l - 2)), aAct + (l - 1) * L::ABUF + p * AP, 256, 128, LBO_ACT, aOnes, 256, 128, 2048,
               ID_TAIL, kTB / 16, p > 0);
      // [db_1 | dW_1 (x, y, z as bf16 planes)] = G_1^T X   (G_1 in buffer 0)
      for (int p = 0; p < P; ++p)
        gemm((uint32_t)(16 * (NH - 2)), aAct + p * AP, 256, 128, LBO_ACT, aXm, 256, 128, 2048, ID_TAIL, kTB / 16,
             p > 0);
      tc::mma_commit_w(bar);
    }
    tailPending = true;   // collected under the next tile's gather and layer 1
    cur = nxt;
    TR(20);
    TR(21);
    dwFresh = false;
  }
  if (TRAIN) {
    if (tailPending) {
      tail_collect();
      tc::tc_fence_before();
      __syncthreads();
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
      for (int w = 0; w < THREADS / 32; ++w) s += wl[w];
      prm.lpart[cta] = s;
    }
  }
  if (warp == 0) wwait();   // no weight load may outlive the CTA (a forward-only pass prefetches W_2)
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, L::TMEM_COLS);
}

template <int W, int NH, int ACT, bool TRAIN, int P = 1, bool STAB = false>
static cudaError_t launch_tc_t(const MlpParams& p, int grid, cudaStream_t s) {
  using L = TcLayout<W, NH, ACT, P, tc_stage_cols<W, STAB>()>;
  auto kern = k_mlp_tc<W, NH, ACT, TRAIN, P, STAB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, (const void*)kern, (int)L::bytes); e != cudaSuccess) return e;
  kern<<<grid * L::MINB, L::THREADS, L::bytes, s>>>(p);
  return cudaGetLastError();
}

#ifdef NBM_TC_TRACE
extern "C" int nbm_debug_tc_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_tc_trace, sizeof(g_tc_trace));
}
#endif

int mlp_tc_supported(int width, int n_hidden, int act, int planes) {
  if (planes == 3) return width == 64 && n_hidden >= 2 && n_hidden <= 4 && act == NBM_ACT_TANH;
  return (width == 64 || width == 128) && n_hidden >= 2 && n_hidden <= 4 &&
         (act == NBM_ACT_TANH || act == NBM_ACT_SILU);
}

// CTAs per SM of the tensor-core kernel (2 when a CTA needs <= 256 TMEM columns and its shared
// memory fits twice; the three-plane split needs one SM per CTA)
int mlp_tc_ctas_per_sm(int width, int n_hidden, int planes) {
  return planes == 1 && width * n_hidden <= 256 ? 2 : 1;
}

template <int ACT>
static cudaError_t launch_tc_act(int width, int n_hidden, bool train, const MlpParams& p, int grid, cudaStream_t s) {
#define NBM_TC_CASES(WW)                                                                                      \
  switch (n_hidden) {                                                                                         \
    case 2: return train ? launch_tc_t<WW, 2, ACT, true>(p, grid, s) : launch_tc_t<WW, 2, ACT, false>(p, grid, s); \
    case 3: return train ? launch_tc_t<WW, 3, ACT, true>(p, grid, s) : launch_tc_t<WW, 3, ACT, false>(p, grid, s); \
    case 4: return train ? launch_tc_t<WW, 4, ACT, true>(p, grid, s) : launch_tc_t<WW, 4, ACT, false>(p, grid, s); \
  }
  if (width == 128) { NBM_TC_CASES(128) }
  if (width == 64) { NBM_TC_CASES(64) }
#undef NBM_TC_CASES
  return cudaErrorInvalidValue;
}

// training pass with the stencil tiles in the stable difference form (G27): bf16, tanh
static cudaError_t launch_tc_stab(int width, int n_hidden, const MlpParams& p, int grid, cudaStream_t s) {
  constexpr int T = NBM_ACT_TANH;
#define NBM_TC_SCASES(WW)                                                  \
  switch (n_hidden) {                                                      \
    case 2: return launch_tc_t<WW, 2, T, true, 1, true>(p, grid, s);       \
    case 3: return launch_tc_t<WW, 3, T, true, 1, true>(p, grid, s);       \
    case 4: return launch_tc_t<WW, 4, T, true, 1, true>(p, grid, s);       \
  }
  if (width == 128) { NBM_TC_SCASES(128) }
  if (width == 64) { NBM_TC_SCASES(64) }
#undef NBM_TC_SCASES
  return cudaErrorInvalidValue;
}

cudaError_t launch_mlp_tc(int width, int n_hidden, int act, int planes, bool train, bool stable,
                          const MlpParams& p, int grid, cudaStream_t s) {
  if (stable) {
    if (!train) return launch_mlp_tc(width, n_hidden, act, planes, false, false, p, grid, s);   // no stencil rows
    if (planes != 1 || act != NBM_ACT_TANH) return cudaErrorInvalidValue;
    return launch_tc_stab(width, n_hidden, p, grid, s);
  }
  if (planes == 3) {   // fp32-accurate split GEMMs (W = 64, tanh)
    static_assert(TcLayout<64, 3, NBM_ACT_TANH, 3>::MINB == 1, "split kernel: one CTA per SM");
    if (width != 64 || act != NBM_ACT_TANH) return cudaErrorInvalidValue;
    switch (n_hidden) {
      case 2: return train ? launch_tc_t<64, 2, NBM_ACT_TANH, true, 3>(p, grid, s) : launch_tc_t<64, 2, NBM_ACT_TANH, false, 3>(p, grid, s);
      case 3: return train ? launch_tc_t<64, 3, NBM_ACT_TANH, true, 3>(p, grid, s) : launch_tc_t<64, 3, NBM_ACT_TANH, false, 3>(p, grid, s);
      case 4: return train ? launch_tc_t<64, 4, NBM_ACT_TANH, true, 3>(p, grid, s) : launch_tc_t<64, 4, NBM_ACT_TANH, false, 3>(p, grid, s);
    }
    return cudaErrorInvalidValue;
  }
  return act == NBM_ACT_SILU ? launch_tc_act<NBM_ACT_SILU>(width, n_hidden, train, p, grid, s)
                             : launch_tc_act<NBM_ACT_TANH>(width, n_hidden, train, p, grid, s);
}

// bf16 image of the hidden weights in the tensor-core core-matrix layout ([o][i], R = W), in
// `planes` exact bf16 planes (1: the RNE copy; 3: the split of PREC_FP32X, plane p = bf16 of
// what the planes before it leave): element (o, i) of plane p of W_l (net k) at
// ((k*(NH-1) + l-2)*planes + p)*W*W + (i/8)*W*8 + o*8 + i%8.
__global__ void k_pack_weights(const float* __restrict__ theta, int64_t p_net, int W, int nhh, int n_nets, int planes,
                               uint16_t* __restrict__ wimg) {
  const int64_t total = (int64_t)n_nets * nhh * W * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / ((int64_t)W * W);
    const int net = (int)(m / nhh), l = (int)(m % nhh) + 2;
    const int r = (int)(e % ((int64_t)W * W)), o = r / W, i = r % W;
    float v = theta[(int64_t)net * p_net + 4 * W + (int64_t)(l - 2) * (W * W + W) + r];
    for (int p = 0; p < planes; ++p) {
      const __nv_bfloat16 b = __float2bfloat16_rn(v);
      wimg[(m * planes + p) * W * W + (int64_t)(i / 8) * W * 8 + o * 8 + (i % 8)] = __bfloat16_as_ushort(b);
      v -= __bfloat162float(b);   // exact: the rounding error of a bf16 rounding is an fp32
    }
  }
}

cudaError_t launch_pack_weights(const ArchInfo& a, const float* theta, uint16_t* wimg, cudaStream_t s) {
  const int nhh = a.n_hidden - 1;
  if (nhh <= 0) return cudaSuccess;
  const int planes = a.prec == NBM_PREC_FP32X ? 3 : 1;
  k_pack_weights<<<148 * 4, 256, 0, s>>>(theta, a.p_net, a.width, nhh, a.n_nets, planes, wimg);
  return cudaGetLastError();
}

}  // namespace nbm
