// mlp_w256.cu -- K3w: fused bf16 tensor-core MLP kernel for hidden width 256 (config 4,
// c5-w256; SURVEY 7.3 hard part 4), run by CTA PAIRS (thread-block clusters of 2, tcgen05
// cta_group::2).  At W = 256 neither the weights (128 KB per matrix) nor three activation
// tiles nor one layer's dW (256 KB fp32 = all of one SM's TMEM) fit on one SM, and a
// per-CTA dW flush of 256 KB per layer per 128-row tile saturates the SM->L2 write path
// (measured: scripts/red_bench.cu).  The pair therefore works as one 256-row tile:
//   * forward / dH GEMMs are M = 256 pair MMAs (each CTA holds its own 128 rows as A); each
//     CTA streams only ITS N-half of every 64-deep weight K-slice (16 KB) through a 4-stage
//     ring, halving the weight traffic per row; the peer forwards its slice arrivals to the
//     leader's barrier (remote mbarrier arrive), the leader issues, completion is multicast;
//   * dW_l = G_l^T h_{l-1} is ONE pair MMA with M = 256 outputs (CTA r owns outputs
//     [128 r, 128 r + 128) in TMEM columns [256, 512)), N = 256 inputs and K = the pair's 256
//     rows: each CTA bulk-loads, from the parked (L2-resident) copies of both CTAs, the
//     o-half of G_l and the i-half of h_{l-1} it owns.  Per row, the fp32 dW flush is half
//     of the single-CTA design's, and it overlaps the next dH GEMM;
//   * h_1..h_{NH-1} and G_2..G_NH are parked as bf16 in per-CTA global scratch; act'(h) in
//     the backward epilogue is read back from there (ld.global.cg, coalesced).
// The flush order across pairs is not fixed: W = 256 is deterministic only within
// tolerance (G21).  512 threads: warp w owns TMEM lane quadrant w % 4 (tile rows / dW
// outputs) and columns [64 (w/4), 64 (w/4) + 64).  Rounding points as the W <= 128 kernel
// (G16), tanh only.
#include <cuda_bf16.h>
#include <math.h>

#include "nbm_internal.cuh"
#include "stab.cuh"
#include "tc_ptx.cuh"

namespace nbm {

namespace {

constexpr int W = 256;
constexpr int kB = 128;        // tile rows per CTA (256 per pair)
constexpr int kPT = 18;        // stencil points per tile
constexpr int kPTS = 16;       // stencil points per tile of the stable form (G27): 8 rows per point
constexpr int kThreads = 512;
constexpr int kStages = 4;     // weight ring: one whole GEMM's slices in flight
constexpr uint32_t ACT = kB * W * 2;        // 64 KB bf16 activation tile
constexpr uint32_t QTR = ACT / 2;           // 32 KB: one 128-column half of it
constexpr uint32_t HSLICE = 64 * 128 * 2;   // 16 KB: one CTA's N-half of a 64-deep K-slice
constexpr uint32_t LBO_ACT = kB * 16;       // 2048: K-core stride of activation tiles
static_assert(kThreads * 128 == ACT, "one discarded L2 line per thread per parked tile");

template <int NH>
struct Lay {
  static constexpr uint32_t oX = 0;                       // activation tile 0
  static constexpr uint32_t oY = oX + ACT;                // activation tile 1
  static constexpr uint32_t oW = oY + ACT;                // weight ring
  static constexpr uint32_t oW1 = oW + kStages * HSLICE;  // fp32 [W][3]
  static constexpr uint32_t oBias = oW1 + 4 * 3 * W;      // fp32 [NH][W]
  static constexpr uint32_t oWo = oBias + 4 * NH * W;     // fp32 [W] + bo
  static constexpr uint32_t oX3 = oWo + 4 * (W + 4);      // fp32 [kB][4]
  static constexpr uint32_t oUp = oX3 + 16 * kB;          // fp32 [4][kB]
  static constexpr uint32_t oU = oUp + 16 * kB;
  static constexpr uint32_t oUb = oU + 4 * kB;
  static constexpr uint32_t oAux = oUb + 4 * kB;
  static constexpr uint32_t oItem = oAux + 4 * kB;
  static constexpr uint32_t oSG = oItem + 4 * kB;         // fp32 [NH + 4][W] small gradients + b_o
  static constexpr uint32_t oBar = oSG + 4 * ((NH + 4) * W + 4);   // full[4], empty[4], mma, dw, ld, park + tmem base
  static constexpr uint32_t bytes = oBar + 128;
  static_assert(bytes <= 227 * 1024, "shared memory");
  static constexpr int kScr = NH + 1;                     // parked tiles per CTA: h_1..h_{NH-1}, G x2
  static constexpr int64_t tW1 = 0, tB1 = 3 * W;
  __host__ __device__ static constexpr int64_t tWl(int l) { return 4 * W + (int64_t)(l - 2) * (W * W + W); }
  __host__ __device__ static constexpr int64_t tBl(int l) { return tWl(l) + W * W; }
  static constexpr int64_t tWo = 4 * W + (int64_t)(NH - 1) * (W * W + W);
  static constexpr int64_t tBo = tWo + W;
};

__device__ __forceinline__ uint32_t pk(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ float th(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float tsum(float (&v)[32], int lane) {   // warp transpose-sum
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
__device__ __forceinline__ void sts4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  tc::check_smem(a, 16);
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
// drop a dead 128-byte line of the parked scratch from L2 without writing it back to HBM
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint4 ldcg4(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// 32 columns (chunk c) of row r: fp32 -> bf16 core layout in shared memory (+ optional global copy)
__device__ __forceinline__ void put_chunk(uint32_t buf, uint8_t* gbuf, int r, int c, const float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t off = (uint32_t)((c * 4 + q) * LBO_ACT + r * 16);
    const uint32_t a = pk(h[8 * q], h[8 * q + 1]), b = pk(h[8 * q + 2], h[8 * q + 3]);
    const uint32_t cc = pk(h[8 * q + 4], h[8 * q + 5]), d = pk(h[8 * q + 6], h[8 * q + 7]);
    sts4(buf + off, a, b, cc, d);
    if (gbuf) *reinterpret_cast<uint4*>(gbuf + off) = make_uint4(a, b, cc, d);
  }
}
// half hf (16 columns) of chunk c of row r (stable-form epilogues, G27: 16-column halves keep
// the shuffled maps within the 128-register budget of the 512-thread CTA)
__device__ __forceinline__ void put_half(uint32_t buf, int r, int c, int hf, const float (&h)[16]) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t off = (uint32_t)((c * 4 + 2 * hf + q) * LBO_ACT + r * 16);
    sts4(buf + off, pk(h[8 * q], h[8 * q + 1]), pk(h[8 * q + 2], h[8 * q + 3]), pk(h[8 * q + 4], h[8 * q + 5]),
         pk(h[8 * q + 6], h[8 * q + 7]));
  }
}
__device__ __forceinline__ void get_half_g(const uint8_t* gbuf, int r, int c, int hf, float (&h)[16]) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint4 w4 = ldcg4(gbuf + (c * 4 + 2 * hf + q) * LBO_ACT + r * 16);
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[8 * q + 2 * e] = __uint_as_float(w[e] << 16);
      h[8 * q + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  }
}
// Two / four transpose-sums interleaved stage by stage (independent shuffle chains: the single
// chain's 5 dependent stages are latency-bound).  tsum2: lane l receives column l of a and of b.
__device__ __forceinline__ void tsum2(float (&a)[32], float (&b)[32], int lane, float& ra, float& rb) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float sa = up ? a[i] : a[i + s], ka = up ? a[i + s] : a[i];
      const float sb = up ? b[i] : b[i + s], kb = up ? b[i + s] : b[i];
      a[i] = ka + __shfl_xor_sync(0xffffffffu, sa, s);
      b[i] = kb + __shfl_xor_sync(0xffffffffu, sb, s);
    }
  }
  ra = a[0];
  rb = b[0];
}
// column sums over the warp's rows of v x0, v x1, v x2 and v (layer-1 gradients): the first
// stage forms the products on the fly, so only 4 x 16 partial sums are live after it
__device__ __forceinline__ void tsum_x4(const float (&v)[32], float x0, float x1, float x2, int lane, float (&r)[4]) {
  float p[4][16];
  {
    const bool up = (lane & 16) != 0;
    const float xs[4] = {x0, x1, x2, 1.0f};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float send = up ? v[i] : v[i + 16], keep = up ? v[i + 16] : v[i];
#pragma unroll
      for (int d = 0; d < 4; ++d) p[d][i] = keep * xs[d] + __shfl_xor_sync(0xffffffffu, send * xs[d], 16);
    }
  }
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i)
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        const float send = up ? p[d][i] : p[d][i + s], keep = up ? p[d][i + s] : p[d][i];
        p[d][i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
  }
#pragma unroll
  for (int d = 0; d < 4; ++d) r[d] = p[d][0];
}
// 16-column warp transpose-sum: lanes l and l + 16 receive the sum over the warp's 32 rows of
// column l % 16
__device__ __forceinline__ float tsum16(float (&v)[16], int lane) {
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? v[i] : v[i + s];
      const float keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// chunk c of row r of a parked (global) bf16 tile -> fp32
__device__ __forceinline__ void get_chunk_g(const uint8_t* gbuf, int r, int c, float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 w4 = ldcg4(gbuf + (c * 4 + q) * LBO_ACT + r * 16);
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[8 * q + 2 * e] = __uint_as_float(w[e] << 16);
      h[8 * q + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  }
}

}  // namespace

#ifdef NBM_TC_TRACE
__device__ long long g_w256_trace[8][48];
__device__ long long g_w256_ld[2][64][4];   // [cta 0/1][gemm #][queue s0, queue s3, full s0, full s3]
#define TRW(k)                                                                                           \
  do {                                                                                                   \
    if (TRAIN && blockIdx.x == 0 && tid == 0 && u - u0 < 8) g_w256_trace[u - u0][k] = clock64();          \
  } while (0)
#else
#define TRW(k) \
  do {         \
  } while (0)
#endif

struct W256Params {
  MlpParams m;
  const uint16_t* wfwd;   // [2][NH-1][4 slices][2 halves][128 o][64 i] K-major core layout
  const uint16_t* wbwd;   // [2][NH-1][4 slices][2 halves][64 o][128 i] MN-major core layout
  uint8_t* hscr;          // [grid][NH+1][64 KB] parked activations / G
  float* rep;             // [R][2][p_stride] gradient replicas (red.global.add)
  int nrep;
};

// STAB: stencil tiles in the stable difference form (G27; training pass only)
template <int NH, bool TRAIN, bool STAB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) k_mlp_w256(const W256Params P) {
  static_assert(!STAB || TRAIN, "stable form: training pass");
  constexpr int TPT = STAB ? kPTS : kPT;
  using L = Lay<NH>;
  const MlpParams& prm = P.m;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = tc::smem_u32(smem);
  float* sW1 = reinterpret_cast<float*>(smem + L::oW1);
  float* sBias = reinterpret_cast<float*>(smem + L::oBias);
  float* sWo = reinterpret_cast<float*>(smem + L::oWo);
  float* sX = reinterpret_cast<float*>(smem + L::oX3);
  float* sUp = reinterpret_cast<float*>(smem + L::oUp);
  float* sU = reinterpret_cast<float*>(smem + L::oU);
  float* sUb = reinterpret_cast<float*>(smem + L::oUb);
  float* sAux = reinterpret_cast<float*>(smem + L::oAux);
  int* sItem = reinterpret_cast<int*>(smem + L::oItem);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem + L::oBar);   // [4]
  uint64_t* bempty = bfull + 4;                                      // [4]
  uint64_t* bmma = bfull + 8;
  uint64_t* bdw = bfull + 9;
  uint64_t* bld = bfull + 10;
  uint64_t* bpark = bfull + 11;   // the peer's parked G_l (and h) are complete in global memory
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(smem + L::oBar + 112);
  __shared__ int segPairs[kNumSeg], segCnt[kNumSeg], segStart[kNumSeg];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, cg = warp >> 2;
  const int row = quad * 32 + lane;
  const uint32_t tlane = (uint32_t)(quad * 32) << 16;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  if (tid < kNumSeg) {
    const int c = prm.counts[prm.cnt_slot[tid]];
    const int per = prm.seg.kind[tid] == kSegStencil ? TPT : kB;
    segCnt[tid] = c;
    segStart[tid] = prm.start_slot[tid] >= 0 ? prm.counts[prm.start_slot[tid]] : 0;
    segPairs[tid] = ((c + per - 1) / per + 1) / 2;
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(bfull + s, leader ? 2 : 1);   // leader: own bytes + the peer's forward
      tc::mbar_init(bempty + s, 1);
    }
    tc::mbar_init(bmma, 1);
    tc::mbar_init(bdw, 1);
    tc::mbar_init(bld, leader ? 2 : 1);
    tc::mbar_init(bpark, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc2(sTmem, 512);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *sTmem;   // [0,256): GEMM accumulator, [256,512): dW
  for (int i = tid; i < (NH + 4) * W + 4; i += kThreads) reinterpret_cast<float*>(smem + L::oSG)[i] = 0.0f;
  __shared__ int firstPair[kNumSeg + 1];   // shared: a per-thread array indexed at run time is local memory
  if (tid == 0) {
    int tot = 0;
    for (int s = 0; s < kNumSeg; ++s) { firstPair[s] = tot; tot += segPairs[s]; }
    firstPair[kNumSeg] = tot;
  }
  __syncthreads();
  const int total = firstPair[kNumSeg];
  const int NC = gridDim.x >> 1, q = blockIdx.x >> 1;
  const int u0 = (int)((int64_t)total * q / NC), u1 = (int)((int64_t)total * (q + 1) / NC);
  const uint32_t aBuf[2] = {sb + L::oX, sb + L::oY};
  const uint32_t ring = sb + L::oW;
  uint8_t* myScr = P.hscr + (int64_t)blockIdx.x * L::kScr * ACT;
  const uint8_t* pairScr0 = P.hscr + (int64_t)(2 * q) * L::kScr * ACT;
  auto hslot = [&](int j) -> int64_t { return (int64_t)(j - 1) * ACT; };                 // h_j, j in 1..NH-1
  auto gslot = [&](int l) -> int64_t { return (int64_t)(NH - 1 + (l & 1)) * ACT; };     // G_l
  uint32_t ph_full[kStages] = {0, 0, 0, 0}, ph_empty[kStages] = {0, 0, 0, 0};
  uint32_t ph_mma = 0, ph_dw = 0, ph_ld = 0, ph_park = 0;
  bool ringUsed = false;
  int gcount = 0, qcount = 0;   // GEMMs issued / queued (trace)

  auto seg_of = [&](int u) {
    int s = 0;
    while (u >= firstPair[s + 1]) ++s;
    return s;
  };
  // ---- weight ring (tid 0 of each CTA) ----
  auto queue_gemm = [&](bool bwd, int net, int l) {
    const uint16_t* base = (bwd ? P.wbwd : P.wfwd) + ((int64_t)net * (NH - 1) + (l - 2)) * 4 * 2 * (HSLICE / 2);
    for (int s = 0; s < kStages; ++s) {
      if (ringUsed) {   // the previous GEMM's MMAs on this stage are done
        tc::mbar_wait(bempty + s, ph_empty[s]);
        ph_empty[s] ^= 1;
      }
      tc::mbar_arrive_expect_tx(bfull + s, HSLICE);
      tc::bulk_copy_g2s(ring + s * HSLICE, base + (int64_t)(s * 2 + rank) * (HSLICE / 2), HSLICE, bfull + s);
#ifdef NBM_TC_TRACE
      if (blockIdx.x < 2 && qcount < 64 && (s == 0 || s == 3)) g_w256_ld[blockIdx.x][qcount][s == 0 ? 0 : 1] = clock64();
#endif
    }
    ++qcount;
  };
  // acc = A * B over 4 K-slices of 64; the peer forwards its slice arrivals, the leader issues
  auto issue_gemm = [&](uint32_t a0, bool bwd, uint32_t idesc) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_wait(bfull + s, ph_full[s]);
      ph_full[s] ^= 1;
#ifdef NBM_TC_TRACE
      if (blockIdx.x < 2 && gcount < 64 && (s == 0 || s == 3)) g_w256_ld[blockIdx.x][gcount][s == 0 ? 2 : 3] = clock64();
#endif
      if (!leader) {
        tc::arrive_leader(bfull + s);
        continue;
      }
      tc::tc_fence_after();
      const uint32_t wb = ring + s * HSLICE;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int kk = s * 4 + k;   // global K-step (16)
        const uint64_t ad = tc::sdesc(a0 + kk * 2 * LBO_ACT, LBO_ACT, 128);
        // forward: B = [128 o][64 i] K-major (LBO 2048, SBO 128); dH: B = [64 o][128 i] MN-major
        const uint64_t bd = bwd ? tc::sdesc(wb + k * 256, 128, 1024) : tc::sdesc(wb + k * 4096, 2048, 128);
        tc::mma2_bf16(tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
      }
      tc::mma2_commit(bempty + s);
    }
    if (leader) tc::mma2_commit(bmma);
    ringUsed = true;
    ++gcount;
  };
  auto wait_bar = [&](uint64_t* b, uint32_t& ph) {
    tc::mbar_wait(b, ph);
    ph ^= 1;
    tc::tc_fence_after();
  };

  constexpr uint32_t ID_FWD = tc::idesc_bf16(2 * kB, W, 0, 0);
  constexpr uint32_t ID_DH = tc::idesc_bf16(2 * kB, W, 0, 1);
  constexpr uint32_t ID_DW = tc::idesc_bf16(2 * kB, W, 1, 1);
  // small gradients (b_1..b_NH, W1[:,0..2], wo, b_o), accumulated in shared memory per column
  // (no per-thread arrays: dynamically indexed register arrays became local memory)
  constexpr int NV = NH + 4;
  float* sSG = reinterpret_cast<float*>(smem + L::oSG);
  auto sg_add = [&](int v, int c, float x) { atomicAdd(&sSG[v * W + c * 32 + lane], x); };
  double lossAcc = 0.0;
  float* rep = P.rep + (int64_t)(q % P.nrep) * 2 * prm.p_stride;
  NBM_CHECK((int64_t)(q % P.nrep + 1) * 2 * prm.p_stride <= prm.rep_len);
  NBM_CHECK((int64_t)(blockIdx.x + 1) * L::kScr * ACT <= prm.hscr_len && (int64_t)(2 * q + 2) * L::kScr * ACT <= prm.hscr_len);
  bool pend = false;   // TMEM [256,512) holds an unflushed dW
  int pendNet = 0, pendL = 2;

  // this CTA's 128 outputs x 256 inputs of dW_pendL.  The replicas hold hidden-weight blocks
  // input-quad-major ([i/4][o][i%4], see k_reduce_rep), so one warp-wide red.v4 covers 32
  // consecutive outputs = 512 contiguous bytes.
  // k0..k1-1: the thread's column chunks to flush (the forward spreads dW_2's flush over GEMMs)
  auto flush_dw_part = [&](int k0, int k1) {
    float* out = rep + (int64_t)pendNet * prm.p_stride + L::tWl(pendL) + (int64_t)(kB * rank + row) * 4;
    NBM_CHECK(pendNet < 2 && (int64_t)(W / 4 - 1) * W * 4 + (kB * rank + row) * 4 + 4 <= (int64_t)W * W);   // inside W_pendL
    for (int k = k0; k < k1; ++k) {
      const int c = 2 * cg + k;
      float v[32];
      tc::tmem_ld32(tmem + tlane + 256u + (uint32_t)(c * 32), v);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        red4(out + (int64_t)(c * 8 + i) * (W * 4), v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
    if (k1 == 2) pend = false;
  };
  auto flush_dw = [&]() { flush_dw_part(0, 2); };
  auto flush_small = [&](int net) {   // all threads, between barriers; leaves sSG zeroed
    float* out = rep + (int64_t)net * prm.p_stride;
    for (int i = tid; i < W; i += kThreads) {
      for (int v = 0; v < NH; ++v) {
        atomicAdd(out + (v == 0 ? L::tB1 : L::tBl(v + 1)) + i, sSG[v * W + i]);
        sSG[v * W + i] = 0.0f;
      }
      for (int c = 0; c < 3; ++c) {
        atomicAdd(out + L::tW1 + 3 * i + c, sSG[(NH + c) * W + i]);
        sSG[(NH + c) * W + i] = 0.0f;
      }
      atomicAdd(out + L::tWo + i, sSG[(NH + 3) * W + i]);
      sSG[(NH + 3) * W + i] = 0.0f;
    }
    if (tid == 0) {
      atomicAdd(out + L::tBo, sSG[NV * W]);
      sSG[NV * W] = 0.0f;
    }
  };
  auto load_net = [&](int net) {
    const float* thp = prm.theta + (int64_t)net * prm.p_net;
    for (int i = tid; i < 3 * W; i += kThreads) sW1[i] = thp[L::tW1 + i];
    for (int i = tid; i < W; i += kThreads) {
      sBias[i] = thp[L::tB1 + i];
      for (int l = 2; l <= NH; ++l) sBias[(l - 1) * W + i] = thp[L::tBl(l) + i];
      sWo[i] = thp[L::tWo + i];
    }
    if (tid == 0) sWo[W] = thp[L::tBo];
  };
  auto layer1 = [&](int c, float x0, float x1, float x2, float (&h)[32]) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = c * 32 + j;
      h[j] = th(fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, fmaf(sW1[3 * n], x0, sBias[n]))));
    }
  };

  // stable form (G27), 16 columns: row inputs x / h e_d / 0, the bias on the centre rows only
  auto layer1_stab = [&](int c, int hf, float x0, float x1, float x2, float (&h)[16]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = c * 32 + hf * 16 + j;
      h[j] = fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, sW1[3 * n] * x0));
    }
    stab::stab_fwd<16>(h, sBias + c * 32 + hf * 16, lane);
  };

  // global loads of pair-tile uu for thread tid < kB: item slot tid (index + aux) and the
  // coordinates of this CTA's tile row tid (stencil arm generated on the fly); issued one tile ahead
  struct Fetch { int item; float aux, x0, x1, x2; };
  auto fetch = [&](int uu) -> Fetch {
    Fetch f{-1, 0.0f, 0.0f, 0.0f, 0.0f};
    if (uu >= u1 || tid >= kB) return f;
    const int sg = seg_of(uu);
    const int knd = prm.seg.kind[sg];
    const int pr = knd == kSegStencil ? TPT : kB;
    const int fst = ((uu - firstPair[sg]) * 2 + (int)rank) * pr;
    const int nv = max(0, min(pr, segCnt[sg] - fst));
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
      const int j = tid / kPT, p = tid - j * kPT;
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
  Fetch cur = fetch(u0), nxt;
  if (u0 < u1 && tid == 0) queue_gemm(false, prm.seg.net[seg_of(u0)], 2);
  int curNet = -1;
  bool h1Staged = false;   // the tile's h_1 was formed under the previous tile's dW_2 (TMEM stash)
  for (int u = u0; u < u1; ++u) {
    const int seg = seg_of(u);
    const int kind = prm.seg.kind[seg], net = prm.seg.net[seg];
    const int per = kind == kSegStencil ? TPT : kB;
    const int first = ((u - firstPair[seg]) * 2 + (int)rank) * per;
    const int nvalid = max(0, min(per, segCnt[seg] - first));   // 0: the pair's odd tail (all rows void)
    const bool stab = STAB && kind == kSegStencil;              // block-uniform
    const bool centre = !stab || (row & 7) == 0;                // rows that carry the biases
    const int nextNet = u + 1 < u1 ? prm.seg.net[seg_of(u + 1)] : -1;
    if (net != curNet) {
      __syncthreads();
      if (TRAIN && curNet >= 0) flush_small(curNet);
      load_net(net);
      curNet = net;
      __syncthreads();
    }
    // ---- gather: items, aux and coordinates were prefetched during the previous tile ----
    if (!h1Staged) {
      if (tid < kB) {
        if (tid < per) {
          sItem[tid] = cur.item;
          sAux[tid] = cur.aux;
        }
        sX[4 * tid] = cur.x0; sX[4 * tid + 1] = cur.x1; sX[4 * tid + 2] = cur.x2;
      }
      __syncthreads();
    }
    TRW(0);
    const float x0 = sX[4 * row], x1 = sX[4 * row + 1], x2 = sX[4 * row + 2];
    // ---- layer 1 -> h1 (tile 0, parked copy) ----
    if (h1Staged) {   // formed under the previous dW_2: TMEM stash -> tile 0
      tc::tc_fence_after();
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = 2 * cg + k;
        uint32_t pkd[16];
        tc::tmem_ld16u(tmem + tlane + (uint32_t)(64 * cg) + 16u * k, pkd);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
          sts4(aBuf[0] + (uint32_t)((c * 4 + qq) * LBO_ACT + row * 16), pkd[4 * qq], pkd[4 * qq + 1], pkd[4 * qq + 2],
               pkd[4 * qq + 3]);
      }
      h1Staged = false;
    } else for (int k = 0; k < 2; ++k) {
      if (STAB && stab) {
        for (int hf = 0; hf < 2; ++hf) {
          float h[16];
          layer1_stab(2 * cg + k, hf, x0, x1, x2, h);
          put_half(aBuf[0], row, 2 * cg + k, hf, h);
        }
      } else {
        float h[32];
        layer1(2 * cg + k, x0, x1, x2, h);
        put_chunk(aBuf[0], nullptr, row, 2 * cg + k, h);
      }
    }
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync_relaxed();   // both CTAs' A tiles are written before the leader's pair MMA
    tc::tc_fence_after();
    if (TRAIN && tid == 0) {      // park h1 (bulk store; completion waited before the backward)
      tc::bulk_copy_s2g(myScr + hslot(1), aBuf[0], ACT);
      tc::bulk_commit();
    }
    TRW(1);
    // ---- forward hidden layers ----
    for (int l = 2; l <= NH; ++l) {
      if (tid == 0) issue_gemm(aBuf[(l - 2) & 1], false, ID_FWD);
      if (l == 3) TRW(24);
      if (l == 2) nxt = fetch(u + 1);  // the next tile's loads overlap this tile
      // the previous tile's dW_2 under this tile's forward GEMMs: split over the last two (the first
      // one's weight slices are still arriving, and the flush's writes hold up their reads)
#ifndef NBM_W256_FLUSH_AT_L2
      if (TRAIN && pend) {
        if (NH >= 4 && l == NH - 1) flush_dw_part(0, 1);
        else if (NH >= 4 && l == NH) flush_dw_part(1, 2);
        else if (NH < 4 && l == NH) flush_dw();
      }
#else
      if (TRAIN && pend) flush_dw();
#endif
      if (tid == 0) {                  // the next GEMM's slices
        if (l < NH) queue_gemm(false, net, l + 1);
        else if (TRAIN) queue_gemm(true, net, NH);
        else if (nextNet >= 0) queue_gemm(false, nextNet, 2);
      }
      if (l == 3) TRW(25);
      if (TRAIN && tid == 0) tc::bulk_wait_read0();   // parked copies have left the tiles
      wait_bar(bmma, ph_mma);
      TRW(2 + 2 * (l - 2));
      float up = 0.0f;
      if (STAB && stab) for (int k = 0; k < 2; ++k) {   // stable form: 16-column halves
        const int c = 2 * cg + k;
        for (int hf = 0; hf < 2; ++hf) {
          const uint32_t col = (uint32_t)(c * 32 + hf * 16);
          float v[16];
          tc::tmem_ld16(tmem + tlane + col, v);
          stab::stab_fwd<16>(v, sBias + (l - 1) * W + col, lane);
          if (l < NH) {
            put_half(aBuf[(l - 1) & 1], row, c, hf, v);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) up = fmaf(sWo[col + j], v[j], up);
            tc::tmem_st16(tmem + tlane + col, v);
          }
        }
      }
      if (!(STAB && stab)) for (int k = 0; k < 2; ++k) {
        const int c = 2 * cg + k;
        float v[32];
        tc::tmem_ld32(tmem + tlane + (uint32_t)(c * 32), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = th(v[j] + sBias[(l - 1) * W + c * 32 + j]);
        if (l < NH) {
          put_chunk(aBuf[(l - 1) & 1], nullptr, row, c, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) up = fmaf(sWo[c * 32 + j], v[j], up);
          if (TRAIN) tc::tmem_st32(tmem + tlane + (uint32_t)(c * 32), v);
        }
      }
      if (l == NH) sUp[cg * kB + row] = up;
      tc::tc_fence_before();
      if (l < NH) tc::fence_proxy_async_smem();
      __syncthreads();
      if (l < NH) tc::cluster_sync_relaxed();
      tc::tc_fence_after();
      if (TRAIN && l < NH && tid == 0) {   // park h_l
        tc::bulk_copy_s2g(myScr + hslot(l), aBuf[(l - 1) & 1], ACT);
        tc::bulk_commit();
      }
      TRW(3 + 2 * (l - 2));
    }
    if (tid < kB) {
      const float uu = ((sUp[tid] + sUp[kB + tid]) + sUp[2 * kB + tid]) + sUp[3 * kB + tid] +
                       ((!stab || (tid & 7) == 0) ? sWo[W] : 0.0f);   // differences carry no output bias
      if (!TRAIN && tid < nvalid) prm.u_out[sItem[tid]] = uu;
      sU[tid] = uu;
    }
    __syncthreads();
    cur = nxt;
    if (!TRAIN) continue;
    // ---- residual epilogue ----
    if (stab) {   // r = c_c u + c_hat sum_d DU_d - b/d (G27); cotangents c_c 2r/N (centre), c_hat 2r/N (Q_d)
      if (tid < kB) {
        const int k = tid >> 3, jr = tid & 7;
        float ubv = 0.0f;
        if (k < nvalid) {
          const float chat = prm.seg.chat[seg], cc = prm.seg.ccen[seg];
          const float du = (sU[8 * k + 4] + sU[8 * k + 5]) + sU[8 * k + 6];
          const float r = fmaf(cc, sU[8 * k], chat * du) - sAux[k];
          if (jr == 0) lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;
          const float rc = prm.two_over_n * r;
          ubv = jr == 0 ? rc * cc : (jr >= 4 && jr < 7) ? rc * chat : 0.0f;
        }
        sUb[tid] = ubv;
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
          lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;
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
    const float ub = sUb[row];
    if (cg == 0) {
      float b = centre ? ub : 0.0f;
#pragma unroll
      for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
      if (lane == 0) atomicAdd(&sSG[NV * W], b);
    }
    const uint32_t gb = aBuf[(NH - 1) & 1];   // G_l (own rows, all outputs), then the dW operand G-halves
    const uint32_t hb = aBuf[NH & 1];         // the dW operand h-halves
    // ---- G_NH = ub wo (1 - h_NH^2) -> gb + parked copy ----
    if (STAB && stab) for (int k = 0; k < 2; ++k) {   // stable form: the backward map of ub wo, halves
      const int c = 2 * cg + k;
      for (int hf = 0; hf < 2; ++hf) {
        const uint32_t col = (uint32_t)(c * 32 + hf * 16);
        float hv[16], v[16];
        tc::tmem_ld16(tmem + tlane + col, hv);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ub * hv[j];
        float sm = tsum16(v, lane);
        if ((lane >> 4) == hf) sg_add(NH + 3, c, sm);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ub * sWo[col + j];
        stab::stab_bwd<16>(v, hv, lane);
        put_half(gb, row, c, hf, v);
        if (!centre) {   // b_NH: centre rows only
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.0f;
        }
        sm = tsum16(v, lane);
        if ((lane >> 4) == hf) sg_add(NH - 1, c, sm);
      }
    }
    if (!(STAB && stab)) for (int k = 0; k < 2; ++k) {
      const int c = 2 * cg + k;
      float hv[32], v[32];
      tc::tmem_ld32(tmem + tlane + (uint32_t)(c * 32), hv);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = ub * hv[j];
#pragma unroll
      for (int j = 0; j < 32; ++j) hv[j] = ub * sWo[c * 32 + j] * (1.0f - hv[j] * hv[j]);
      put_chunk(gb, nullptr, row, c, hv);
      float s_wo, s_b;
      tsum2(v, hv, lane, s_wo, s_b);
      sg_add(NH + 3, c, s_wo);
      sg_add(NH - 1, c, s_b);
    }
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync_relaxed();
    tc::tc_fence_after();
    if (tid == 0) {   // park G_NH
      // park only the output half the peer's dW needs (this CTA's rows, outputs of CTA rank ^ 1);
      // this CTA's own half stays in place in gb for its dW K-steps
      tc::bulk_copy_s2g(myScr + gslot(NH) + (rank ^ 1u) * QTR, gb + (rank ^ 1u) * QTR, QTR);
      tc::bulk_commit();
    }
    TRW(10);
    // ---- backward hidden layers ----
    for (int l = NH; l >= 2; --l) {
      if (tid == 0) issue_gemm(gb, true, ID_DH);   // acc = G_l W_l
      TRW(26 + 3 * (NH - l));
      if (pend) flush_dw();            // dW_{l+1} under the dH GEMM
      if (tid == 0) {
        if (l > 2) queue_gemm(true, net, l - 1);
        else if (nextNet >= 0) queue_gemm(false, nextNet, 2);
        tc::bulk_wait0();                 // parked G_l (and, at l = NH, every parked h) is complete
        if (l == NH) asm volatile("fence.proxy.async.global;" ::: "memory");
        tc::arrive_remote(bpark, rank ^ 1u);
      }
      TRW(27 + 3 * (NH - l));
      wait_bar(bmma, ph_mma);
      if (l == NH) __syncthreads();       // the parked h are readable (ld.global) from here on
      if (tid == 0) {
        tc::mbar_wait(bpark, ph_park);    // the peer's parked G_l is complete
        ph_park ^= 1;
        // the dW operands: h_{l-1}[rows of CTA t][this CTA's input half], t = 0, 1, and
        // G_l[rows of the peer][the outputs this CTA owns] (its own rows' block is in place)
        tc::mbar_arrive_expect_tx(bld, 3 * QTR);
        for (int t = 0; t < 2; ++t) {
          const uint8_t* scr = pairScr0 + (int64_t)t * L::kScr * ACT + rank * QTR;
          tc::bulk_copy_g2s(hb + t * QTR, scr + hslot(l - 1), QTR, bld);
          if (t != (int)rank) tc::bulk_copy_g2s(gb + t * QTR, scr + gslot(l), QTR, bld);
        }
      }
      TRW(28 + 3 * (NH - l));
      TRW(11 + 4 * (NH - l));
      // G_{l-1} (bf16, the next dH GEMM's A tile) waits for the dW MMA in TMEM: packed in place in
      // this warp's accumulator columns [64 cg, 64 cg + 32) (chunk k at + 16 k, after the chunk and
      // the one before it have been read), not in a register tile held across the wait
      const uint32_t stash = tmem + tlane + (uint32_t)(64 * cg);
      const uint8_t* hprev = myScr + hslot(l - 1);
      if (STAB && stab) for (int k = 0; k < 2; ++k) {   // stable form: 16-column halves
        const int c = 2 * cg + k;
        uint32_t pkd[16];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float v[16], hq[16];
          tc::tmem_ld16(tmem + tlane + (uint32_t)(c * 32 + hf * 16), v);
          get_half_g(hprev, row, c, hf, hq);
          stab::stab_bwd<16>(v, hq, lane);
          const bool mine = (lane >> 4) == hf;   // lane l accumulates column 32 k + l
          if (l - 1 >= 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j) pkd[8 * hf + j] = pk(v[2 * j], v[2 * j + 1]);
            if (!centre) {   // b_{l-1}: centre rows only (v is consumed)
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = 0.0f;
            }
            const float sm = tsum16(v, lane);
            if (mine) sg_add(l - 2, c, sm);
          } else {           // layer 1: dW1 += G1 x^T (x = the row input), db1 += G1 (centre rows)
            const float xs[3] = {x0, x1, x2};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              float tv[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) tv[j] = v[j] * xs[d];
              const float sm = tsum16(tv, lane);
              if (mine) sg_add(NH + d, c, sm);
            }
            if (!centre) {
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = 0.0f;
            }
            const float sm = tsum16(v, lane);
            if (mine) sg_add(0, c, sm);
          }
        }
        if (l - 1 >= 2) tc::tmem_st16u(stash + 16u * k, pkd);
      }
      if (!(STAB && stab)) for (int k = 0; k < 2; ++k) {
        const int c = 2 * cg + k;
        float v[32], hq[32];
        tc::tmem_ld32(tmem + tlane + (uint32_t)(c * 32), v);
        get_chunk_g(hprev, row, c, hq);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= 1.0f - hq[j] * hq[j];
        if (l - 1 >= 2) {
          uint32_t pkd[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pkd[j] = pk(v[2 * j], v[2 * j + 1]);
          tc::tmem_st16u(stash + 16u * k, pkd);
          sg_add(l - 2, c, tsum(v, lane));
        } else {   // layer 1: dW1 += G1 x^T, db1 += G1
          float r4[4];
          tsum_x4(v, x0, x1, x2, lane, r4);
          sg_add(NH, c, r4[0]);
          sg_add(NH + 1, c, r4[1]);
          sg_add(NH + 2, c, r4[2]);
          sg_add(0, c, r4[3]);
        }
      }
      tc::tc_fence_before();
      __syncthreads();   // this CTA's TMEM reads (flush, epilogue) are done
      TRW(12 + 4 * (NH - l));
      if (tid == 0) {
        tc::mbar_wait(bld, ph_ld);   // own halves landed (+ the peer's forward, leader)
        ph_ld ^= 1;
        if (!leader) {
          tc::arrive_leader(bld);
        } else {
          tc::tc_fence_after();
          // dW_l[o][i] = sum over the pair's 256 rows: K-steps 0..7 rows of CTA 0, 8..15 of CTA 1
          for (int t = 0; t < 2; ++t)
            for (int kk = 0; kk < kB / 16; ++kk)
              tc::mma2_bf16(tmem + 256, tc::sdesc(gb + t * QTR + kk * 256, 128, LBO_ACT),
                            tc::sdesc(hb + t * QTR + kk * 256, 128, LBO_ACT), ID_DW, (t | kk) ? 1u : 0u);
          tc::mma2_commit(bdw);
        }
      }
      // the next tile's gather and layer 1 under dW_2 (same network, direct form): h_1 bf16 into this
      // warp's accumulator columns (free at l = 2), copied to tile 0 once dW_2 has released it
      if (!STAB && TRAIN && l == 2 && nextNet == net) {
        if (tid < kB) {   // (slots past the next tile's item count hold item -1 / aux 0: unread)
          sItem[tid] = cur.item;
          sAux[tid] = cur.aux;
          sX[4 * tid] = cur.x0; sX[4 * tid + 1] = cur.x1; sX[4 * tid + 2] = cur.x2;
        }
        __syncthreads();
        const float y0 = sX[4 * row], y1 = sX[4 * row + 1], y2 = sX[4 * row + 2];
        for (int k = 0; k < 2; ++k) {
          float h[32];
          layer1(2 * cg + k, y0, y1, y2, h);
          uint32_t pkd[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pkd[j] = pk(h[2 * j], h[2 * j + 1]);
          tc::tmem_st16u(tmem + tlane + (uint32_t)(64 * cg) + 16u * k, pkd);
        }
        tc::tc_fence_before();
        h1Staged = true;
      }
      wait_bar(bdw, ph_dw);
      // both CTAs' bulk loads of h_{l-1} and G_l (and this CTA's act' reads) are complete: the
      // parked copies are dead, so they leave L2 without a write-back to HBM
      discard_l2(myScr + hslot(l - 1) + tid * 128);
      if (tid < kThreads / 2) discard_l2(myScr + gslot(l) + (rank ^ 1u) * QTR + tid * 128);
      pend = true;
      pendNet = net;
      pendL = l;
      TRW(13 + 4 * (NH - l));
      if (l > 2) {   // G_{l-1} (own rows, all outputs) -> gb for the next dH GEMM
        tc::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int c = 2 * cg + k;
          uint32_t pkd[16];
          tc::tmem_ld16u(stash + 16u * k, pkd);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            sts4(gb + (uint32_t)((c * 4 + qq) * LBO_ACT + row * 16), pkd[4 * qq], pkd[4 * qq + 1], pkd[4 * qq + 2],
                 pkd[4 * qq + 3]);
        }
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        __syncthreads();
        tc::cluster_sync_relaxed();   // both A tiles written
        tc::tc_fence_after();
        if (tid == 0) {               // park G_{l-1}
          tc::bulk_copy_s2g(myScr + gslot(l - 1) + (rank ^ 1u) * QTR, gb + (rank ^ 1u) * QTR, QTR);
          tc::bulk_commit();
        }
      }
      TRW(14 + 4 * (NH - l));
    }
  }
  if (TRAIN) {
    if (pend) flush_dw();
    __syncthreads();
    if (curNet >= 0) flush_small(curNet);
    for (int o = 16; o; o >>= 1) lossAcc += __shfl_xor_sync(0xffffffffu, lossAcc, o);
    __shared__ double wl[kThreads / 32];
    if (lane == 0) wl[warp] = lossAcc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += wl[w];
      prm.lpart[blockIdx.x] = s;
    }
  }
  if (tid == 0) tc::bulk_wait0();
  tc::tc_fence_before();
  tc::cluster_sync();   // no pair MMA may still target the peer's TMEM
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc2(tmem, 512);
}

// forward image: [net][l][slice s][half r] = W_l[o in [128 r, 128 r + 128)][i in [64 s, 64 s + 64)],
//   K-major core layout: (i'/8)*2048 B + o'*16 B + (i'%8)*2 B
// backward image: [net][l][slice s][half r] = W_l[o in [64 s, 64 s + 64)][i in [128 r, 128 r + 128)],
//   MN-major core layout: (i'/8)*1024 B + o'*16 B + (i'%8)*2 B
__global__ void k_pack_w256(const float* __restrict__ theta, int64_t p_net, int nhh, int n_nets,
                            uint16_t* __restrict__ wf, uint16_t* __restrict__ wb) {
  const int64_t total = (int64_t)n_nets * nhh * W * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / (W * W);
    const int net = (int)(m / nhh), l = (int)(m % nhh) + 2;
    const int r = (int)(e % (W * W)), o = r / W, i = r % W;
    const uint16_t v = __bfloat16_as_ushort(__float2bfloat16_rn(
        theta[(int64_t)net * p_net + 4 * W + (int64_t)(l - 2) * (W * W + W) + r]));
    const int64_t base = m * W * W;   // 4 slices x 2 halves of 8192 elements
    {
      const int s = i / 64, ip = i % 64, h = o / 128, op = o % 128;
      wf[base + (int64_t)(s * 2 + h) * 8192 + (ip / 8) * 1024 + op * 8 + (ip % 8)] = v;
    }
    {
      const int s = o / 64, op = o % 64, h = i / 128, ip = i % 128;
      wb[base + (int64_t)(s * 2 + h) * 8192 + (ip / 8) * 512 + op * 8 + (ip % 8)] = v;
    }
  }
}

#ifdef NBM_TC_TRACE
extern "C" int nbm_debug_w256_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_w256_trace, sizeof(g_w256_trace));
}
extern "C" int nbm_debug_w256_ld(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_w256_ld, sizeof(g_w256_ld));
}
#endif

template <int NH, bool TRAIN, bool STAB = false>
static cudaError_t launch_w256_t(const W256Params& p, int grid, cudaStream_t s) {
  auto kern = k_mlp_w256<NH, TRAIN, STAB>;
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once(attr, (const void*)kern, (int)Lay<NH>::bytes); e != cudaSuccess) return e;
  kern<<<grid, kThreads, Lay<NH>::bytes, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_mlp_w256(int n_hidden, bool train, bool stable, const MlpParams& m, const uint16_t* wf,
                            const uint16_t* wb, uint8_t* hscr, float* rep, int nrep, int grid, cudaStream_t s) {
  W256Params p{m, wf, wb, hscr, rep, nrep};
  grid &= ~1;   // CTA pairs
  if (grid < 2 || nrep < 1) return cudaErrorInvalidValue;
  if (stable && train) {
    switch (n_hidden) {
      case 2: return launch_w256_t<2, true, true>(p, grid, s);
      case 3: return launch_w256_t<3, true, true>(p, grid, s);
      case 4: return launch_w256_t<4, true, true>(p, grid, s);
    }
    return cudaErrorInvalidValue;
  }
  switch (n_hidden) {
    case 2: return train ? launch_w256_t<2, true>(p, grid, s) : launch_w256_t<2, false>(p, grid, s);
    case 3: return train ? launch_w256_t<3, true>(p, grid, s) : launch_w256_t<3, false>(p, grid, s);
    case 4: return train ? launch_w256_t<4, true>(p, grid, s) : launch_w256_t<4, false>(p, grid, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pack_w256(const ArchInfo& a, const float* theta, uint16_t* wf, uint16_t* wb, cudaStream_t s) {
  const int nhh = a.n_hidden - 1;
  if (nhh <= 0) return cudaSuccess;
  k_pack_w256<<<148 * 4, 256, 0, s>>>(theta, a.p_net, nhh, a.n_nets, wf, wb);
  return cudaGetLastError();
}

// K4r for the replica paths (bf16 W = 256, fp32 W >= 128): grad = sum of the replicas in fixed
// replica order, loss from lpart.  quad_major (bf16 W = 256): the hidden-weight blocks W_l[o][i]
// sit input-quad-major in the replicas, [i/4][o][i%4]; otherwise in the natural layout.
__global__ void k_reduce_rep(const float* __restrict__ rep, int nrep, int64_t p_net, int64_t p_stride, int n_nets,
                             int n_hidden, int quad_major, int accumulate, const double* __restrict__ lpart, int G, float* __restrict__ grad,
                             float* __restrict__ loss, int* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_nets * p_net) {
    const int net = (int)(i / p_net);
    const int64_t j = i - net * p_net;
    int64_t jr = j;   // position in the replica
    if (quad_major && j >= 4 * W && j < 4 * W + (int64_t)(n_hidden - 1) * (W * W + W)) {
      const int64_t lo = (j - 4 * W) % (W * W + W);
      if (lo < W * W) {
        const int o = (int)(lo / W), in = (int)(lo % W);
        jr = j - lo + ((int64_t)(in / 4) * W + o) * 4 + (in % 4);
      }
    }
    double s = accumulate ? (double)grad[i] : 0.0;   // multi-resolution levels add up
    for (int r = 0; r < nrep; ++r) s += rep[((int64_t)r * 2 + net) * p_stride + jr];
    const float v = (float)s;
    grad[i] = v;
    if (!isfinite(v)) atomicOr(err, kErrNonfinite);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = accumulate ? (double)*loss : 0.0;
    for (int g = 0; g <= G; ++g) s += lpart[g];
    *loss = (float)s;
    if (!isfinite(*loss)) atomicOr(err, kErrNonfinite);
  }
}

cudaError_t launch_reduce_rep(const float* rep, int nrep, int64_t p_net, int64_t p_stride, int n_nets, int n_hidden,
                              int quad_major, int accumulate, const double* lpart, int G, float* grad, float* loss,
                              int* err, cudaStream_t s) {
  const int64_t P = n_nets * p_net;
  k_reduce_rep<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(rep, nrep, p_net, p_stride, n_nets, n_hidden, quad_major, accumulate, lpart, G,
                                                           grad, loss, err);
  return cudaGetLastError();
}

}  // namespace nbm
