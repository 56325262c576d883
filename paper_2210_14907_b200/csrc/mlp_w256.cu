// mlp_w256.cu -- K3w: fused bf16 tensor-core MLP kernel for hidden width 256 (config 4,
// c5-w256; SURVEY 7.3 hard part 4).  At W = 256 neither the weights (128 KB per matrix)
// nor three activation buffers (64 KB each) nor one layer's dW (256 KB fp32 = all of TMEM)
// fit on chip, so this kernel:
//   * streams the hidden weights through a 2-stage shared-memory ring in 32 KB K-slices
//     (cp.async.bulk + mbarrier complete_tx) from two packed bf16 images (forward slices
//     along the input index, backward slices along the output index);
//   * keeps two 64 KB activation buffers on chip and parks h_1..h_{NH-1} (bf16) in a
//     per-CTA global scratch (L2-resident) that is brought back by bulk copies for the
//     backward pass;
//   * computes each tile's dW_l = G_l^T h_{l-1} in two 128-output halves into a TMEM
//     scratch (columns [256,512); the working accumulator uses [0,256)) and flushes it with
//     vector reductions (red.global.add.v4.f32) into a few replica buffers.  The flush order
//     across CTAs is not fixed: W = 256 is deterministic only within tolerance (G21).
// 512 threads: warp w owns TMEM lane quadrant w % 4 (tile rows) and columns
// [64 (w/4), 64 (w/4) + 64).  Rounding points as the W <= 128 kernel (G16),
// tanh only.
#include <cuda_bf16.h>
#include <math.h>

#include "nbm_internal.cuh"
#include "tc_ptx.cuh"

namespace nbm {

namespace {

constexpr int W = 256;
constexpr int kB = 128;        // tile rows
constexpr int kPT = 18;        // stencil points per tile
constexpr int kThreads = 512;
constexpr uint32_t ACT = kB * W * 2;      // 64 KB bf16 activation buffer
constexpr uint32_t SLICE = 64 * W * 2;    // 32 KB weight K-slice
constexpr uint32_t LBO_ACT = kB * 16;     // 2048: K-core stride of activation buffers

template <int NH>
struct Lay {
  static constexpr uint32_t oX = 0;                     // activation buffer 0
  static constexpr uint32_t oY = oX + ACT;              // activation buffer 1
  static constexpr uint32_t oW = oY + ACT;              // 2 weight stages
  static constexpr uint32_t oW1 = oW + 2 * SLICE;       // fp32 [W][3]
  static constexpr uint32_t oBias = oW1 + 4 * 3 * W;    // fp32 [NH][W]
  static constexpr uint32_t oWo = oBias + 4 * NH * W;   // fp32 [W] + bo
  static constexpr uint32_t oX3 = oWo + 4 * (W + 4);    // fp32 [kB][4]
  static constexpr uint32_t oUp = oX3 + 16 * kB;        // fp32 [4][kB]
  static constexpr uint32_t oU = oUp + 16 * kB;
  static constexpr uint32_t oUb = oU + 4 * kB;
  static constexpr uint32_t oAux = oUb + 4 * kB;
  static constexpr uint32_t oItem = oAux + 4 * kB;
  static constexpr uint32_t oBar = oItem + 4 * kB;      // mma, full[2], empty[2], hload + tmem base
  static constexpr uint32_t bytes = oBar + 64;
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
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ void lds4(uint32_t a, uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a) : "memory");
}
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
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
__device__ __forceinline__ void get_chunk(uint32_t buf, int r, int c, float (&h)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
    lds4(buf + (uint32_t)((c * 4 + q) * LBO_ACT + r * 16), w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      h[8 * q + 2 * e] = __uint_as_float(w[e] << 16);
      h[8 * q + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  }
}

}  // namespace

struct W256Params {
  MlpParams m;
  const uint16_t* wfwd;   // [2][NH-1][4 slices][256 o][64 i] K-major core layout
  const uint16_t* wbwd;   // [2][NH-1][4 slices][64 o][256 i] MN-major core layout
  uint8_t* hscr;          // [grid][NH-1][64 KB] parked activations
  float* rep;             // [R][2][p_stride] gradient replicas (red.global.add)
  int nrep;
};

template <int NH, bool TRAIN>
__global__ void __launch_bounds__(kThreads, 1) k_mlp_w256(const W256Params P) {
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
  uint64_t* bmma = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* bfull = bmma + 1;    // [2]
  uint64_t* bempty = bmma + 3;   // [2]
  uint64_t* bh = bmma + 5;       // activation reload
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(smem + L::oBar + 48);
  __shared__ int segTiles[kNumSeg], segCnt[kNumSeg], segStart[kNumSeg];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, cg = warp >> 2;
  const int row = quad * 32 + lane;
  const uint32_t tlane = (uint32_t)(quad * 32) << 16;
  if (tid < kNumSeg) {
    const int c = prm.counts[prm.cnt_slot[tid]];
    segCnt[tid] = c;
    segStart[tid] = prm.start_slot[tid] >= 0 ? prm.counts[prm.start_slot[tid]] : 0;
    segTiles[tid] = (c + (prm.seg.kind[tid] == kSegStencil ? kPT : kB) - 1) / (prm.seg.kind[tid] == kSegStencil ? kPT : kB);
  }
  if (tid == 0) {
    for (int i = 0; i < 6; ++i) tc::mbar_init(bmma + i, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc(sTmem, 512);
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
  const uint32_t aBuf[2] = {sb + L::oX, sb + L::oY};
  uint8_t* hscr = P.hscr + (int64_t)cta * (NH - 1) * ACT;
  uint32_t ph_mma = 0, ph_full[2] = {0, 0}, ph_empty[2] = {0, 0}, ph_h = 0;
  bool empty_armed[2] = {false, false};   // an MMA commit is pending on the stage
  bool pending_full[2] = {false, false};  // a bulk copy into the stage has not been waited on

  // ---- weight slice pipeline (tid 0 only) ----
  int curNet = -1;
  auto slice_ptr = [&](bool bwd, int l, int s) -> const uint16_t* {
    const uint16_t* base = bwd ? P.wbwd : P.wfwd;
    return base + (((int64_t)curNet * (NH - 1) + (l - 2)) * 4 + s) * (SLICE / 2);
  };
  auto load_slice = [&](int st, bool bwd, int l, int s) {
    if (pending_full[st]) {           // drain an unused prefetch (e.g. on a network switch)
      tc::mbar_wait(bfull + st, ph_full[st]);
      ph_full[st] ^= 1;
      pending_full[st] = false;
    }
    if (empty_armed[st]) {            // wait until the MMAs that read this stage are done
      tc::mbar_wait(bempty + st, ph_empty[st]);
      ph_empty[st] ^= 1;
      empty_armed[st] = false;
    }
    tc::mbar_arrive_expect_tx(bfull + st, SLICE);
    tc::bulk_copy_g2s(sb + L::oW + st * SLICE, slice_ptr(bwd, l, s), SLICE, bfull + st);
    pending_full[st] = true;
  };
  // GEMM with streamed B: acc[dcol] = A * B over 4 K-slices of 64.  Slices 0 and 1 must
  // already be loading into stages 0 and 1; the next GEMM's first two slices are queued.
  auto gemm_streamed = [&](uint32_t a0, bool bwd, int l, uint32_t idesc, int nl, bool nbwd, bool has_next) {
    for (int s = 0; s < 4; ++s) {
      const int st = s & 1;
      tc::mbar_wait(bfull + st, ph_full[st]);
      ph_full[st] ^= 1;
      pending_full[st] = false;
      tc::tc_fence_after();
      const uint32_t wb = sb + L::oW + st * SLICE;
      for (int k = 0; k < 4; ++k) {
        const int kk = s * 4 + k;   // global K-step (16)
        uint64_t ad, bd;
        if (!bwd) {   // forward: A = h (K-major), B = slice [256 o][64 i] K-major (LBO 4096, SBO 128)
          ad = tc::sdesc(a0 + kk * 2 * LBO_ACT, LBO_ACT, 128);
          bd = tc::sdesc(wb + k * 2 * 4096, 4096, 128);
        } else {      // dH: A = G (K-major over o), B = slice [64 o][256 i] MN-major (LBO 128, SBO 1024)
          ad = tc::sdesc(a0 + kk * 2 * LBO_ACT, LBO_ACT, 128);
          bd = tc::sdesc(wb + k * 256, 128, 1024);
        }
        tc::mma_bf16(tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
      }
      tc::mma_commit(bempty + st);
      empty_armed[st] = true;
      if (s + 2 < 4) load_slice(st, bwd, l, s + 2);
      else if (has_next) load_slice(st, nbwd, nl, s - 2);
    }
    tc::mma_commit(bmma);
  };
  auto wait_mma = [&]() {
    tc::mbar_wait(bmma, ph_mma);
    ph_mma ^= 1;
    tc::tc_fence_after();
  };

  constexpr uint32_t ID_FWD = tc::idesc_bf16(kB, W, 0, 0);
  constexpr uint32_t ID_DH = tc::idesc_bf16(kB, W, 0, 1);
  constexpr uint32_t ID_DW = tc::idesc_bf16(128, W, 1, 1);
  // small gradients per lane (column 64 cg + 32 k + lane): b_1..b_NH, W1[:,0..2], wo
  constexpr int NV = NH + 4;
  float g[NV][2];
  float gbo = 0.0f;
  double lossAcc = 0.0;
  float* rep = P.rep + (int64_t)(cta % P.nrep) * 2 * prm.p_stride;

  auto flush_small = [&](int net) {
    float* out = rep + (int64_t)net * prm.p_stride;
    for (int k = 0; k < 2; ++k) {
      const int col = 64 * cg + 32 * k + lane;
      for (int v = 0; v < NH; ++v) atomicAdd(out + (v == 0 ? L::tB1 : L::tBl(v + 1)) + col, g[v][k]);
      for (int c = 0; c < 3; ++c) atomicAdd(out + L::tW1 + 3 * col + c, g[NH + c][k]);
      atomicAdd(out + L::tWo + col, g[NH + 3][k]);
    }
    if (cg == 0 && lane == 0) atomicAdd(out + L::tBo, gbo);
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
    for (int v = 0; v < NV; ++v) g[v][0] = g[v][1] = 0.0f;
    gbo = 0.0f;
  };
  auto layer1 = [&](int c, float x0, float x1, float x2, float (&h)[32]) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = c * 32 + j;
      h[j] = th(fmaf(sW1[3 * n + 2], x2, fmaf(sW1[3 * n + 1], x1, fmaf(sW1[3 * n], x0, sBias[n]))));
    }
  };

  int seg = 0;
  for (int t = t0; t < t1; ++t) {
    while (t >= firstTile[seg + 1]) ++seg;
    const int kind = prm.seg.kind[seg], net = prm.seg.net[seg];
    const int per = kind == kSegStencil ? kPT : kB;
    const int first = (t - firstTile[seg]) * per;
    const int nvalid = min(per, segCnt[seg] - first);
    if (net != curNet) {
      __syncthreads();
      if (TRAIN && curNet >= 0) flush_small(curNet);
      load_net(net);
      curNet = net;
      if (tid == 0) {   // queue the first GEMM's slices (stages are idle between tiles)
        load_slice(0, false, 2, 0);
        load_slice(1, false, 2, 1);
      }
      __syncthreads();
    }
    // ---- gather ----
    const int* items = prm.seg.items[seg] + segStart[seg];
    if (tid < per) {
      const int it = tid < nvalid ? items[first + tid] : -1;
      sItem[tid] = it;
      float a = 0.0f;
      if (it >= 0) a = prm.aux_by_item[seg] ? prm.seg.aux[seg][it] : prm.seg.aux[seg][segStart[seg] + first + tid];
      sAux[tid] = a;
    }
    __syncthreads();
    if (tid < kB) {
      float x0 = 0.0f, x1 = 0.0f, x2 = 0.0f;
      if (kind == kSegStencil) {
        const int j = tid / kPT, p = tid - j * kPT;
        if (j < 7 && p < nvalid) {
          const float* src = prm.seg.src[seg] + 3 * (int64_t)sItem[p];
          x0 = src[0]; x1 = src[1]; x2 = src[2];
          if (j > 0) {
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
    const float x0 = sX[4 * row], x1 = sX[4 * row + 1], x2 = sX[4 * row + 2];
    // ---- layer 1 -> h1 (buffer 0, parked copy) ----
    for (int k = 0; k < 2; ++k) {
      float h[32];
      layer1(2 * cg + k, x0, x1, x2, h);
      put_chunk(aBuf[0], TRAIN ? hscr : nullptr, row, 2 * cg + k, h);
    }
    if (TRAIN) asm volatile("fence.proxy.async.global;" ::: "memory");   // parked h1 -> later bulk reads
    tc::fence_proxy_async_smem();
    __syncthreads();
    // ---- forward hidden layers ----
    for (int l = 2; l <= NH; ++l) {
      const uint32_t ain = aBuf[(l - 2) & 1];
      if (tid == 0) {
        // next GEMM: forward l+1, or (training) the backward dH of layer NH
        const bool has_next = (l < NH) || TRAIN;
        gemm_streamed(ain, false, l, ID_FWD, l < NH ? l + 1 : NH, l == NH, has_next);
      }
      wait_mma();
      float up = 0.0f;
      for (int k = 0; k < 2; ++k) {
        const int c = 2 * cg + k;
        float v[32];
        tc::tmem_ld32(tmem + tlane + (uint32_t)(c * 32), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = th(v[j] + sBias[(l - 1) * W + c * 32 + j]);
        if (l < NH) {
          put_chunk(aBuf[(l - 1) & 1], TRAIN ? hscr + (int64_t)(l - 1) * ACT : nullptr, row, c, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) up = fmaf(sWo[c * 32 + j], v[j], up);
          if (TRAIN) tc::tmem_st32(tmem + tlane + (uint32_t)(c * 32), v);
        }
      }
      if (l == NH) sUp[cg * kB + row] = up;
      if (TRAIN && l < NH) asm volatile("fence.proxy.async.global;" ::: "memory");
      tc::tc_fence_before();
      if (l < NH) tc::fence_proxy_async_smem();
      __syncthreads();
    }
    if (tid < kB) {
      const float u = ((sUp[tid] + sUp[kB + tid]) + sUp[2 * kB + tid]) + sUp[3 * kB + tid] + sWo[W];
      if (!TRAIN && tid < nvalid) prm.u_out[sItem[tid]] = u;
      sU[tid] = u;
    }
    __syncthreads();
    if (!TRAIN) {
      if (tid == 0) {   // restore the next tile's first slices
        load_slice(0, false, 2, 0);
        load_slice(1, false, 2, 1);
      }
      continue;
    }
    // ---- residual epilogue ----
    if (kind == kSegStencil) {
      if (tid < kPT) {
        float r = 0.0f;
        if (tid < nvalid) {
          const float chat = prm.seg.chat[seg];
          float acc = sU[tid];
#pragma unroll
          for (int j = 1; j < 7; ++j) acc = fmaf(chat, sU[j * kPT + tid], acc);
          r = acc - sAux[tid];
          lossAcc += 0.5 * (double)prm.two_over_n * (double)r * (double)r;
        }
        const float rc = prm.two_over_n * r;
        sUb[tid] = rc;
        const float rj = rc * prm.seg.chat[seg];
#pragma unroll
        for (int j = 1; j < 7; ++j) sUb[j * kPT + tid] = rj;
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
      float b = ub;
#pragma unroll
      for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
      gbo += b;
    }
    // ---- G_NH = ub wo (1 - h_NH^2) -> buffer (NH-1)&1 ----
    for (int k = 0; k < 2; ++k) {
      const int c = 2 * cg + k;
      float hv[32], v[32];
      tc::tmem_ld32(tmem + tlane + (uint32_t)(c * 32), hv);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = ub * hv[j];
      g[NH + 3][k] += tsum(v, lane);
#pragma unroll
      for (int j = 0; j < 32; ++j) hv[j] = ub * sWo[c * 32 + j] * (1.0f - hv[j] * hv[j]);
      put_chunk(aBuf[(NH - 1) & 1], nullptr, row, c, hv);
      g[NH - 1][k] += tsum(hv, lane);
    }
    tc::tc_fence_before();
    tc::fence_proxy_async_smem();
    __syncthreads();
    // ---- backward hidden layers ----
    for (int l = NH; l >= 2; --l) {
      const uint32_t gb = aBuf[(l - 1) & 1];   // G_l
      const uint32_t hb = aBuf[(l - 2) & 1];   // h_{l-1}
      // dW_l in two 128-output halves through the TMEM scratch, flushed by vector reductions
      for (int half = 0; half < 2; ++half) {
        if (tid == 0) {
          tc::tc_fence_after();
          for (int kk = 0; kk < kB / 16; ++kk)
            tc::mma_bf16(tmem + 256, tc::sdesc(gb + half * 16 * LBO_ACT + kk * 256, 128, LBO_ACT),
                         tc::sdesc(hb + kk * 256, 128, LBO_ACT), ID_DW, kk > 0 ? 1u : 0u);
          tc::mma_commit(bmma);
        }
        wait_mma();
        float* out = rep + (int64_t)curNet * prm.p_stride + L::tWl(l) + (int64_t)(half * 128 + row) * W;
        for (int k = 0; k < 2; ++k) {
          const int c = 2 * cg + k;
          float v[32];
          tc::tmem_ld32(tmem + tlane + 256u + (uint32_t)(c * 32), v);
#pragma unroll
          for (int q = 0; q < 8; ++q) red4(out + c * 32 + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
        tc::tc_fence_before();
        __syncthreads();
      }
      // acc = G_l W_l (streamed backward slices); then the next slices: dH_{l-1} or the next tile
      if (tid == 0) {
        tc::tc_fence_after();
        if (l > 2) gemm_streamed(gb, true, l, ID_DH, l - 1, true, true);
        else gemm_streamed(gb, true, l, ID_DH, 2, false, true);   // next tile's forward W_2
      }
      wait_mma();
      if (l > 2 && tid == 0) {   // bring h_{l-2} back into the buffer that held G_l
        tc::mbar_arrive_expect_tx(bh, ACT);
        tc::bulk_copy_g2s(gb, hscr + (int64_t)(l - 3) * ACT, ACT, bh);
      }
      for (int k = 0; k < 2; ++k) {
        const int c = 2 * cg + k;
        float v[32], hq[32];
        tc::tmem_ld32(tmem + tlane + (uint32_t)(c * 32), v);
        get_chunk(hb, row, c, hq);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= 1.0f - hq[j] * hq[j];
        if (l - 1 >= 2) {
          put_chunk(hb, nullptr, row, c, v);   // G_{l-1} in place of h_{l-1}
          g[l - 2][k] += tsum(v, lane);
        } else {   // layer 1: dW1 += G1 x^T, db1 += G1
          float tv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) tv[j] = v[j] * x0;
          g[NH][k] += tsum(tv, lane);
#pragma unroll
          for (int j = 0; j < 32; ++j) tv[j] = v[j] * x1;
          g[NH + 1][k] += tsum(tv, lane);
#pragma unroll
          for (int j = 0; j < 32; ++j) tv[j] = v[j] * x2;
          g[NH + 2][k] += tsum(tv, lane);
          g[0][k] += tsum(v, lane);
        }
      }
      if (l > 2 && tid == 0) {   // the reload must land before dW_{l-1} reads it
        tc::mbar_wait(bh, ph_h);
        ph_h ^= 1;
      }
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
    }
  }
  if (TRAIN) {
    __syncthreads();
    if (curNet >= 0) flush_small(curNet);
    for (int o = 16; o; o >>= 1) lossAcc += __shfl_xor_sync(0xffffffffu, lossAcc, o);
    __shared__ double wl[kThreads / 32];
    if (lane == 0) wl[warp] = lossAcc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) s += wl[w];
      prm.lpart[cta] = s;
    }
  }
  // drain the slice pipeline before exit (queued bulk copies must complete)
  if (tid == 0) {
    for (int st = 0; st < 2; ++st) {
      if (pending_full[st]) tc::mbar_wait(bfull + st, ph_full[st]);
      if (empty_armed[st]) tc::mbar_wait(bempty + st, ph_empty[st]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// forward image: slice s of W_l = [256 o][64 i] K-major core layout: (i'/8)*4096 + o*16 + (i'%8)*2
// backward image: slice s of W_l = [64 o][256 i] MN-major core layout: (i/8)*1024 + o'*16 + (i%8)*2
__global__ void k_pack_w256(const float* __restrict__ theta, int64_t p_net, int nhh, int n_nets,
                            uint16_t* __restrict__ wf, uint16_t* __restrict__ wb) {
  const int64_t total = (int64_t)n_nets * nhh * W * W;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / (W * W);
    const int net = (int)(m / nhh), l = (int)(m % nhh) + 2;
    const int r = (int)(e % (W * W)), o = r / W, i = r % W;
    const uint16_t v = __bfloat16_as_ushort(__float2bfloat16_rn(
        theta[(int64_t)net * p_net + 4 * W + (int64_t)(l - 2) * (W * W + W) + r]));
    const int64_t base = m * W * W;   // 4 slices of 64*256 elements
    {
      const int s = i / 64, ip = i % 64;
      wf[base + (int64_t)s * 64 * W + (ip / 8) * 2048 + o * 8 + (ip % 8)] = v;
    }
    {
      const int s = o / 64, op = o % 64;
      wb[base + (int64_t)s * 64 * W + (i / 8) * 512 + op * 8 + (i % 8)] = v;
    }
  }
}

template <int NH, bool TRAIN>
static cudaError_t launch_w256_t(const W256Params& p, int grid, cudaStream_t s) {
  auto kern = k_mlp_w256<NH, TRAIN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay<NH>::bytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  kern<<<grid, kThreads, Lay<NH>::bytes, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_mlp_w256(int n_hidden, bool train, const MlpParams& m, const uint16_t* wf,
                            const uint16_t* wb, uint8_t* hscr, float* rep, int nrep, int grid, cudaStream_t s) {
  W256Params p{m, wf, wb, hscr, rep, nrep};
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

// K4r for W = 256: grad = sum of the replicas (fixed replica order), loss from lpart.
__global__ void k_reduce_rep(const float* __restrict__ rep, int nrep, int64_t p_net, int64_t p_stride, int n_nets,
                             const double* __restrict__ lpart, int G, float* __restrict__ grad,
                             float* __restrict__ loss, int* __restrict__ err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_nets * p_net) {
    const int net = (int)(i / p_net);
    const int64_t j = i - net * p_net;
    double s = 0.0;
    for (int r = 0; r < nrep; ++r) s += rep[((int64_t)r * 2 + net) * p_stride + j];
    const float v = (float)s;
    grad[i] = v;
    if (!isfinite(v)) atomicOr(err, kErrNonfinite);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int g = 0; g <= G; ++g) s += lpart[g];
    *loss = (float)s;
    if (!isfinite(*loss)) atomicOr(err, kErrNonfinite);
  }
}

cudaError_t launch_reduce_rep(const float* rep, int nrep, int64_t p_net, int64_t p_stride, int n_nets,
                              const double* lpart, int G, float* grad, float* loss, int* err, cudaStream_t s) {
  const int64_t P = n_nets * p_net;
  k_reduce_rep<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(rep, nrep, p_net, p_stride, n_nets, lpart, G, grad, loss, err);
  return cudaGetLastError();
}

}  // namespace nbm
