// nbm.cu -- the C ABI of libnbm.so (include/nbm.h): descriptor validation, workspace,
// the per-call launch sequence of the hot path, K4r gradient reduction and the
// timing hook.  See DESIGN.md section 5 for the kernel list.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "nbm_internal.cuh"

using namespace nbm;

namespace {

// counts[] slot map (device int[16]):
//   0..5   class totals (kCls*), 6..11 class starts in list[], 12/13 crossed rows per
//   network, 15 always zero.
constexpr int kSlotZero = 15;

thread_local std::string g_create_error;

int fail(nbm_handle* h, int code, const std::string& msg) {
  if (h) h->last_error = msg;
  return code;
}

int cuda_fail(nbm_handle* h, cudaError_t e, const char* where) {
  return fail(h, NBM_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool h_on_lattice(float h, int64_t* H) {
  double v = (double)h * kLattice;
  if (!(h > 0.0f) || !(h < 1.0f) || v != floor(v)) return false;
  *H = (int64_t)v;
  return true;
}

int check_arch(const nbm_arch* a, ArchInfo* out, std::string* why) {
  if (!a || !a->sizes || a->n_layers < 3 || a->n_layers > kMaxLayers) {
    *why = "arch: need 3..8 layer sizes [3, W, ..., W, 1]";
    return NBM_E_INVALID_ARCH;
  }
  if (a->sizes[0] != 3 || a->sizes[a->n_layers - 1] != 1) {
    *why = "arch: sizes[0] must be 3 and the last 1 (S:174)";
    return NBM_E_INVALID_ARCH;
  }
  int W = a->sizes[1];
  for (int l = 1; l < a->n_layers - 1; ++l)
    if (a->sizes[l] != W) { *why = "arch: hidden widths must be uniform"; return NBM_E_INVALID_ARCH; }
  if (a->n_nets != 1 && a->n_nets != 2) { *why = "arch: n_nets must be 1 or 2"; return NBM_E_INVALID_ARCH; }
  if (a->act != NBM_ACT_TANH && a->act != NBM_ACT_SILU && a->act != NBM_ACT_SINE) { *why = "arch: bad activation"; return NBM_E_INVALID_ARCH; }
  if (a->prec != NBM_PREC_FP32 && a->prec != NBM_PREC_BF16 && a->prec != NBM_PREC_FP32X) {
    *why = "arch: bad precision"; return NBM_E_INVALID_ARCH;
  }
  int nh = a->n_layers - 2;
  bool ok = false;
  if (a->prec == NBM_PREC_FP32)
    ok = mlp_fp32_supported(W, nh, a->act) || (a->act == NBM_ACT_TANH && mlp_fp32w_supported(W, nh));
  if (a->prec == NBM_PREC_BF16) ok = mlp_tc_supported(W, nh, a->act, 1) || (W == 256 && nh >= 2 && nh <= 4 && a->act == NBM_ACT_TANH);
  if (a->prec == NBM_PREC_FP32X) ok = mlp_tc_supported(W, nh, a->act, 3);
  if (!ok) {
    *why = "arch: unsupported (prec, act, width, depth) combination in this build";
    return NBM_E_INVALID_ARCH;
  }
  if (a->stencil != NBM_STENCIL_DIRECT && a->stencil != NBM_STENCIL_STABLE) {
    *why = "arch: bad stencil evaluation";
    return NBM_E_INVALID_ARCH;
  }
  if (a->stencil == NBM_STENCIL_STABLE &&
      !(a->act == NBM_ACT_TANH && (a->prec == NBM_PREC_BF16 || a->prec == NBM_PREC_FP32))) {
    *why = "arch: the stable stencil form needs tanh with BF16 or FP32 (G27)";
    return NBM_E_INVALID_ARCH;
  }
  if (out) {
    memset(out, 0, sizeof(*out));
    out->n_layers = a->n_layers;
    out->width = W;
    out->n_hidden = nh;
    out->act = a->act;
    out->prec = a->prec;
    out->n_nets = a->n_nets;
    out->stencil = a->stencil;
    int64_t p = 0;
    for (int l = 0; l < a->n_layers; ++l) out->sizes[l] = a->sizes[l];
    for (int l = 1; l < a->n_layers; ++l) p += (int64_t)a->sizes[l] * a->sizes[l - 1] + a->sizes[l];
    out->p_net = p;
  }
  return NBM_OK;
}

int check_problem(const nbm_problem* p, DevProblem* out, std::string* why) {
  if (!p) { *why = "problem: null"; return NBM_E_ARG; }
  for (int d = 0; d < 3; ++d)
    if (p->box_lo[d] != -1.0f || p->box_hi[d] != 1.0f) { *why = "problem: box must be [-1,1]^3 (G23)"; return NBM_E_INVALID_PROBLEM; }
  if (!(p->beta_minus > 0.0f) || !(p->beta_plus > 0.0f)) { *why = "problem: beta must be > 0 (S:236)"; return NBM_E_INVALID_PROBLEM; }
  if (!(p->k_minus >= 0.0f) || !(p->k_plus >= 0.0f)) { *why = "problem: k must be >= 0"; return NBM_E_INVALID_PROBLEM; }
  if (!(p->lambda_b >= 0.0f)) { *why = "problem: lambda_b must be >= 0"; return NBM_E_INVALID_PROBLEM; }
  const nbm_levelset& ls = p->ls;
  if (ls.kind < NBM_LS_NONE || ls.kind > NBM_LS_GRID) { *why = "problem: bad level-set kind"; return NBM_E_INVALID_PROBLEM; }
  if (ls.kind == NBM_LS_GRID) {
    if (ls.grid_n < 1 || ls.grid_n > 1024 || !ls.grid_phi) { *why = "problem: grid level set needs 1..1024 cells and nodal values"; return NBM_E_INVALID_PROBLEM; }
    const int64_t nn = (int64_t)(ls.grid_n + 1) * (ls.grid_n + 1) * (ls.grid_n + 1);
    for (int64_t i = 0; i < nn; ++i)
      if (!isfinite(ls.grid_phi[i])) { *why = "problem: non-finite level-set node"; return NBM_E_INVALID_PROBLEM; }
  }
  if (ls.kind == NBM_LS_SPHERES) {
    if (ls.n < 1 || ls.n > kMaxSpheres || !ls.centers || !ls.radii) { *why = "problem: spheres need 1..64 centres and radii"; return NBM_E_INVALID_PROBLEM; }
    for (int k = 0; k < ls.n; ++k)
      if (!(ls.radii[k] > 0.0f)) { *why = "problem: sphere radius must be > 0"; return NBM_E_INVALID_PROBLEM; }
  }
  if (ls.kind == NBM_LS_STAR && (ls.star_m < 0 || ls.star_m > 16 || ls.star_n < 0 || ls.star_n > 16 || !(ls.star_r0 > 0.0f))) {
    *why = "problem: bad star parameters"; return NBM_E_INVALID_PROBLEM;
  }
  if (!((p->source >= NBM_SRC_SINE3PI && p->source <= NBM_SRC_GAUSS) || p->source == NBM_SRC_PAPER41)) {
    *why = "problem: bad source"; return NBM_E_INVALID_PROBLEM;
  }
  if (p->mu_kind < NBM_MU_CONST || p->mu_kind > NBM_MU_LINEAR) { *why = "problem: bad mu kind"; return NBM_E_INVALID_PROBLEM; }
  if (p->mu_kind == NBM_MU_LINEAR)   // positive on the box: a linear field attains its minimum at a corner
    for (int s = 0; s < 2; ++s)
      for (int c = 0; c < 8; ++c) {
        const float* m = p->mu_lin[s];
        const double v = m[0] + ((c & 1) ? m[1] : -m[1]) + ((c & 2) ? m[2] : -m[2]) + ((c & 4) ? m[3] : -m[3]);
        if (!(v > 0.0)) { *why = "problem: linear mu must be > 0 on the box (S:236)"; return NBM_E_INVALID_PROBLEM; }
      }
  if (p->source == NBM_SRC_GAUSS && p->mu_kind != NBM_MU_CONST) { *why = "problem: Gaussian charges need constant mu"; return NBM_E_INVALID_PROBLEM; }
  if (p->source == NBM_SRC_GAUSS) {
    if (p->n_charges < 0 || p->n_charges > kMaxCharges || (p->n_charges > 0 && (!p->q || !p->charge_centers)) || !(p->charge_sigma > 0.0f)) {
      *why = "problem: bad charges"; return NBM_E_INVALID_PROBLEM;
    }
  }
  if (out) {
    memset(out, 0, sizeof(*out));
    out->ls_kind = ls.kind;
    if (ls.kind == NBM_LS_SPHERES) {
      out->n_spheres = ls.n;
      for (int k = 0; k < ls.n; ++k) {
        for (int d = 0; d < 3; ++d) out->centers[k][d] = out->centers_f[k][d] = ls.centers[3 * k + d];
        out->radii[k] = out->radii_f[k] = ls.radii[k];
      }
    }
    out->star_r0 = ls.star_r0; out->star_amp = ls.star_amp;
    out->star_m = ls.star_m; out->star_n = ls.star_n;
    for (int d = 0; d < 3; ++d) out->plane_n[d] = ls.plane_n[d];
    out->plane_c = ls.plane_c;
    out->grid_n = ls.kind == NBM_LS_GRID ? ls.grid_n : 0;
    out->grid_phi = nullptr;   // device copy made by nbm_create
    out->beta[0] = p->beta_minus; out->beta[1] = p->beta_plus;
    out->k[0] = p->k_minus; out->k[1] = p->k_plus;
    out->source = p->source;
    if (p->source == NBM_SRC_GAUSS) {
      out->n_charges = p->n_charges;
      for (int k = 0; k < p->n_charges; ++k) {
        out->q[k] = p->q[k];
        for (int d = 0; d < 3; ++d) out->charge_centers[k][d] = p->charge_centers[3 * k + d];
      }
      out->charge_sigma = p->charge_sigma;
    }
    out->lambda_b = p->lambda_b;
    out->mu_kind = p->mu_kind;
    for (int s = 0; s < 2; ++s)
      for (int c = 0; c < 4; ++c) out->mu_lin[s][c] = p->mu_lin[s][c];
  }
  return NBM_OK;
}

// K4r: grad[net][j] = sum over CTAs of the touched partials, in fixed order: 16 CTA groups
// (g = 16 m + k) summed per thread, then the 16 group sums in order; loss = the CTA loss
// partials plus the crossed rows' loss.  fp64 accumulation of the fp32 partials.  The
// partial loads of a thread are issued together (independent, up to kRedBatch in flight)
// before the fixed-order accumulation: the kernel is latency-bound otherwise.
constexpr int kRedCols = 32, kRedGroups = 16, kRedBatch = 8;
__global__ void __launch_bounds__(kRedCols * kRedGroups) k_reduce(
    const float* __restrict__ part, const int* __restrict__ touched, int G, int64_t p_net, int64_t p_stride,
    int n_nets, int accumulate, const double* __restrict__ lpart, float* __restrict__ grad,
    float* __restrict__ loss, int* __restrict__ err) {
  __shared__ double acc[kRedGroups][kRedCols];
  const int col = threadIdx.x % kRedCols, grp = threadIdx.x / kRedCols;
  const int64_t i = (int64_t)blockIdx.x * kRedCols + col;
  const int64_t P = n_nets * p_net;
  double s = 0.0;
  if (i < P) {
    const int net = (int)(i / p_net);
    const int64_t j = i - net * p_net;
    const float* base = part + (int64_t)net * G * p_stride + j;
    const int* tch = touched + net * G;
    for (int g0 = grp; g0 < G; g0 += kRedGroups * kRedBatch) {
      float v[kRedBatch];
#pragma unroll
      for (int b = 0; b < kRedBatch; ++b) {
        const int g = g0 + b * kRedGroups;
        v[b] = (g < G && tch[g]) ? base[(int64_t)g * p_stride] : 0.0f;
      }
#pragma unroll
      for (int b = 0; b < kRedBatch; ++b) s += (double)v[b];
    }
  }
  acc[grp][col] = s;
  __syncthreads();
  if (grp == 0 && i < P) {
    double t = accumulate ? (double)grad[i] : 0.0;   // multi-resolution levels add up
    for (int k = 0; k < kRedGroups; ++k) t += acc[k][col];
    const float v = (float)t;
    grad[i] = v;
    if (!isfinite(v)) atomicOr(err, kErrNonfinite);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t = accumulate ? (double)*loss : 0.0;
    for (int g = 0; g <= G; ++g) t += lpart[g];
    const float v = (float)t;
    *loss = v;
    if (!isfinite(v)) atomicOr(err, kErrNonfinite);
  }
}

double diag(const DevProblem& P, int s, double h) {   // d_s = k_s + 6 beta_s / h^2
  double h2 = h * h, c0 = P.k[s];
  for (int j = 0; j < 6; ++j) c0 += P.beta[s] / h2;
  return c0;
}

void fill_common(const nbm_handle* h, MlpParams& p, const float* theta, float hf) {
  memset(&p, 0, sizeof(p));
  p.counts = h->ws.counts;
  p.theta = theta;
  p.p_net = h->arch.p_net;
  p.h = hf;
  p.part = h->ws.part;
  p.wimg = h->ws.wimg;
  p.p_stride = (h->arch.p_net + 3) & ~3ll;
  p.touched = h->ws.touched;
  p.lpart = h->ws.lpart;
  p.part_len = 2 * (int64_t)h->ws.grid_mlp * p.p_stride;
  p.hscr_len = h->ws.hscr_len;
  p.rep_len = h->ws.rep_len;
#ifdef NBM_BOUNDS_SELFTEST
  p.part_len = 0;   // scripts/r2/bounds_check.sh: every partial-slot flush violates, the checks must fire
#endif
  for (int s = 0; s < kNumSeg; ++s) { p.cnt_slot[s] = kSlotZero; p.start_slot[s] = -1; p.seg.kind[s] = kSegXRows; }
}

bool is_w256(const ArchInfo& A) { return A.prec == NBM_PREC_BF16 && A.width == 256; }
bool is_fp32w(const ArchInfo& A) { return A.prec == NBM_PREC_FP32 && A.width >= 128; }
// paths whose gradients go through L2 replicas (per-tile dW flushes) instead of per-CTA partials
bool uses_rep(const ArchInfo& A) { return is_w256(A) || is_fp32w(A); }

// per-call weight images of the hidden layers (bf16 tensor-core layouts / fp32 wide-path slices)
cudaError_t launch_pack(const nbm_handle* h, const float* theta, cudaStream_t s) {
  const ArchInfo& A = h->arch;
  const Workspace& w = h->ws;
  if (is_fp32w(A)) return launch_pack_fp32w(A, theta, w.wimg32, s);
  if (A.prec == NBM_PREC_FP32X) return launch_pack_weights(A, theta, w.wimg, s);   // three planes (streamed at NH = 4)
  if (A.prec != NBM_PREC_BF16) return cudaSuccess;
  return is_w256(A) ? launch_pack_w256(A, theta, w.wimg, w.wimg_b, s) : launch_pack_weights(A, theta, w.wimg, s);
}

cudaError_t launch_mlp_h(const nbm_handle* h, bool train, const MlpParams& p, cudaStream_t s) {
  const ArchInfo& A = h->arch;
  const Workspace& w = h->ws;
  if (is_w256(A)) {
    return launch_mlp_w256(A.n_hidden, train, A.stencil == NBM_STENCIL_STABLE, p, w.wimg, w.wimg_b, w.hscr, w.rep,
                           w.nrep, w.grid_base, s);
  }
  if (is_fp32w(A))
    return launch_mlp_fp32w(A.width, A.n_hidden, train, A.stencil == NBM_STENCIL_STABLE, p, w.wimg32, w.rep, w.nrep,
                            w.grid_base, s);
  if (A.prec == NBM_PREC_BF16) {
    // the training pass of the direct form at W = 64 / 128 (tanh): K3h (two half-tiles in flight);
    // NBM_TCH_OFF selects K3t for comparison
    static const bool tch_off = getenv("NBM_TCH_OFF") != nullptr;
    if (train && A.stencil != NBM_STENCIL_STABLE && !tch_off && mlp_tch_supported(A.width, A.n_hidden, A.act))
      return launch_mlp_tch(A.width, A.n_hidden, p, w.grid_base, s);
    return launch_mlp_tc(A.width, A.n_hidden, A.act, 1, train, A.stencil == NBM_STENCIL_STABLE, p, w.grid_base, s);
  }
  if (A.prec == NBM_PREC_FP32X) return launch_mlp_tc(A.width, A.n_hidden, A.act, 3, train, false, p, w.grid_base, s);
  return launch_mlp_fp32(A.width, A.n_hidden, A.act, train, A.stencil == NBM_STENCIL_STABLE, p, w.grid_base, s);
}


}  // namespace

namespace nbm {
cudaError_t launch_reduce(const nbm_handle* h, bool accumulate, float* grad, float* loss, cudaStream_t s) {
  int64_t P = h->arch.p_net * h->arch.n_nets;
  k_reduce<<<(unsigned)((P + kRedCols - 1) / kRedCols), kRedCols * kRedGroups, 0, s>>>(h->ws.part, h->ws.touched, h->ws.grid_mlp,
                                                       h->arch.p_net, (h->arch.p_net + 3) & ~3ll,
                                                       h->arch.n_nets, accumulate ? 1 : 0, h->ws.lpart,
                                                       grad, loss, h->ws.err);
  return cudaGetLastError();
}
}  // namespace nbm

extern "C" {

const char* nbm_version(void) { return "nbm-b200 0.1 (sm_100a)"; }

int64_t nbm_arch_param_count(const nbm_arch* arch) {
  if (!arch || !arch->sizes || arch->n_layers < 2 || arch->n_nets < 1 || arch->n_nets > 2) return -1;
  int64_t p = 0;
  for (int l = 1; l < arch->n_layers; ++l) {
    if (arch->sizes[l] <= 0 || arch->sizes[l - 1] <= 0) return -1;
    p += (int64_t)arch->sizes[l] * arch->sizes[l - 1] + arch->sizes[l];
  }
  return p * arch->n_nets;
}

int nbm_check(const nbm_problem* problem, const nbm_arch* arch) {
  std::string why;
  int rc = check_problem(problem, nullptr, &why);
  if (rc) return rc;
  return check_arch(arch, nullptr, &why);
}

int nbm_create(const nbm_problem* problem, const nbm_arch* arch, int device, int64_t max_points,
               nbm_handle** out) {
  if (!out || max_points < 1 || max_points > (1ll << 27)) return NBM_E_ARG;
  *out = nullptr;
  std::string why;
  DevProblem dp;
  ArchInfo ai;
  int rc = check_problem(problem, &dp, &why);
  if (rc) { g_create_error = why; return rc; }
  rc = check_arch(arch, &ai, &why);
  if (rc) { g_create_error = why; return rc; }
  if (dp.mu_kind != NBM_MU_CONST && ai.prec == NBM_PREC_FP32X) {
    g_create_error = "variable mu: not supported by the split-plane fp32x kernel";
    return NBM_E_INVALID_ARCH;
  }
  if (dp.mu_kind != NBM_MU_CONST && ai.stencil == NBM_STENCIL_STABLE) {
    g_create_error = "the stable stencil form assumes constant mu per phase (G27)";
    return NBM_E_INVALID_ARCH;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { g_create_error = cudaGetErrorString(e); return NBM_E_CUDA; }
  nbm_handle* h = new nbm_handle();
  h->device = device;
  h->arch = ai;
  h->host_problem = dp;
  h->timing = false;
  h->timed_calls = 0;
  h->last_launches = 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  Workspace& w = h->ws;
  w.cap = max_points;
  w.xcap = max_points;
  int64_t items = 2 * max_points;
  w.nblk_cls = (int)((items + 1023) / 1024);
  w.grid_base = sms;
  w.grid_mlp = sms * ((ai.prec == NBM_PREC_BF16)    ? mlp_tc_ctas_per_sm(ai.width, ai.n_hidden, 1)
                      : (ai.prec == NBM_PREC_FP32X) ? mlp_tc_ctas_per_sm(ai.width, ai.n_hidden, 3)
                      : (ai.width <= 64 ? mlp_fp32_ctas_per_sm() : 1));
  std::vector<void**> ptrs;
  size_t sizes[32];
  int k = 0;
#define ALLOC(field, bytes) do { ptrs.push_back((void**)&(field)); sizes[k++] = (bytes); } while (0)
  ALLOC(h->d_problem, sizeof(DevProblem));
  ALLOC(w.cls, items);
  ALLOC(w.aux_tmp, items * sizeof(float));
  ALLOC(w.blk_counts, (size_t)w.nblk_cls * kNumCls * sizeof(int));
  ALLOC(w.blk_offsets, (size_t)w.nblk_cls * kNumCls * sizeof(int));
  ALLOC(w.counts, 16 * sizeof(int));
  ALLOC(w.list, items * sizeof(int));
  ALLOC(w.list_aux, items * sizeof(float));
  ALLOC(w.pcoef, dp.mu_kind != NBM_MU_CONST ? (size_t)max_points * 6 * sizeof(float) : 16);
  ALLOC(w.xrow_x, 7 * w.xcap * 3 * sizeof(float));
  ALLOC(w.xrow_u, 7 * w.xcap * sizeof(float));
  ALLOC(w.xrow_cot, 7 * w.xcap * sizeof(float));
  ALLOC(w.xrow_tag, 7 * w.xcap);
  ALLOC(w.xrec, 8 * w.xcap * sizeof(float));
  ALLOC(w.xlist, 2 * 7 * w.xcap * sizeof(int));
  ALLOC(w.part, 2 * (size_t)w.grid_mlp * ((ai.p_net + 3) & ~3ll) * sizeof(float));
  ALLOC(w.touched, 2 * (size_t)w.grid_mlp * sizeof(int));
  ALLOC(w.lpart, ((size_t)w.grid_mlp + 1) * sizeof(double));
  ALLOC(w.err, sizeof(int));
  ALLOC(w.epart, (size_t)2 * kErrBlocks * sizeof(double));
  ALLOC(w.bc, 2 * sizeof(float));
  const size_t nhh = ai.n_hidden > 1 ? ai.n_hidden - 1 : 1;
  ALLOC(w.wimg, (size_t)2 * nhh * ai.width * ai.width * (ai.prec == NBM_PREC_FP32X ? 3 : 1) * sizeof(uint16_t));
  const bool w256 = is_w256(ai), fw = is_fp32w(ai), urep = uses_rep(ai);
  // gradient replicas in L2 (fewer CTAs per address): K3w measured fastest with one (c4: 64.2 vs
  // 64.8 ms per launch with 16; its smaller L2 footprint outweighs the address sharing,
  // scripts/r2/exp_rep.sh), K3fw keeps 16
  w.nrep = urep ? (w256 ? 1 : 16) : 0;
  if (urep && getenv("NBM_W256_REPLICAS")) w.nrep = atoi(getenv("NBM_W256_REPLICAS"));
  ALLOC(w.wimg_b, w256 ? (size_t)2 * nhh * ai.width * ai.width * sizeof(uint16_t) : 16);
  w.hscr_len = w256 ? (int64_t)w.grid_mlp * (nhh + 2) * 128 * ai.width * 2 : 16;   // parks: NH + 1 tiles per CTA (mlp_w256.cu kScr)
  w.rep_len = urep ? (int64_t)w.nrep * 2 * ((ai.p_net + 3) & ~3ll) : 4;
  ALLOC(w.hscr, (size_t)w.hscr_len);
  ALLOC(w.rep, (size_t)w.rep_len * sizeof(float));
  ALLOC(w.wimg32, fw ? (size_t)2 * nhh * 2 * ai.width * ai.width * sizeof(float) : 16);
#undef ALLOC
  for (size_t i = 0; i < ptrs.size(); ++i) {
    e = cudaMalloc(ptrs[i], sizes[i]);
    if (e != cudaSuccess) {
      g_create_error = std::string("cudaMalloc: ") + cudaGetErrorString(e);
      nbm_destroy(h);
      return NBM_E_CUDA;
    }
  }
  if (dp.ls_kind == NBM_LS_GRID) {   // the sampled level set's nodes live on the device
    const size_t gb = (size_t)(dp.grid_n + 1) * (dp.grid_n + 1) * (dp.grid_n + 1) * sizeof(float);
    e = cudaMalloc(&h->d_grid, gb);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_grid, problem->ls.grid_phi, gb, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      g_create_error = std::string("grid level set: ") + cudaGetErrorString(e);
      nbm_destroy(h);
      return NBM_E_CUDA;
    }
    dp.grid_phi = h->d_grid;
    h->host_problem.grid_phi = h->d_grid;
  }
  e = cudaMemcpy(h->d_problem, &dp, sizeof(dp), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(w.counts, 0, 16 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(w.err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(w.touched, 0, 2 * (size_t)w.grid_mlp * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(w.lpart, 0, ((size_t)w.grid_mlp + 1) * sizeof(double));
  if (e != cudaSuccess) {
    g_create_error = cudaGetErrorString(e);
    nbm_destroy(h);
    return NBM_E_CUDA;
  }
  *out = h;
  return NBM_OK;
}

void nbm_destroy(nbm_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  void* ps[] = {h->d_problem, h->ws.cls, h->ws.aux_tmp, h->ws.blk_counts, h->ws.blk_offsets,
                h->ws.counts, h->ws.list, h->ws.list_aux, h->ws.xrow_x, h->ws.xrow_u, h->ws.xrow_cot,
                h->ws.xrow_tag, h->ws.xrec, h->ws.xlist, h->ws.part, h->ws.touched, h->ws.lpart,
                h->ws.err, h->ws.bc, h->d_grid, h->ws.pcoef, h->ws.wimg, h->ws.wimg_b, h->ws.hscr, h->ws.rep, h->ws.wimg32};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (cudaEvent_t ev : h->ev) cudaEventDestroy(ev);
  delete h;
}

int64_t nbm_param_count(const nbm_handle* h) { return h ? h->arch.p_net * h->arch.n_nets : -1; }

const char* nbm_last_error(const nbm_handle* h) {
  return h ? h->last_error.c_str() : g_create_error.c_str();
}

int nbm_status(nbm_handle* h, void* stream) {
  if (!h) return NBM_E_ARG;
  cudaSetDevice(h->device);
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "nbm_status");
  int word = 0;
  e = cudaMemcpy(&word, h->ws.err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(h->ws.err, 0, sizeof(int));
  if (e != cudaSuccess) return cuda_fail(h, e, "nbm_status");
  if (word & kErrOutOfDomain) return fail(h, NBM_E_OUT_OF_DOMAIN, "an arm p +- h e_d left the box (S:259)");
  if (word & kErrDegenerate) return fail(h, NBM_E_DEGENERATE, "degenerate level-set gradient at a crossing (S:117)");
  if (word & kErrNonfinite) return fail(h, NBM_E_NONFINITE, "non-finite loss or gradient (S:367)");
  return NBM_OK;
}

int nbm_init_params(nbm_handle* h, uint64_t seed, float* theta_dev, void* stream) {
  if (!h || !theta_dev) return NBM_E_ARG;
  cudaSetDevice(h->device);
  cudaError_t e = launch_init_params(h->arch, seed, theta_dev, (cudaStream_t)stream);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_init_params");
}

int nbm_sample(nbm_handle* h, uint64_t seed, uint64_t step, int kind, int64_t first_index,
               int64_t n, float h_cell, float* pts_dev, void* stream) {
  if (!h || (n > 0 && !pts_dev) || n < 0 || first_index < 0) return fail(h, NBM_E_ARG, "nbm_sample: bad arguments");
  if (kind != NBM_POINTS_INTERIOR && kind != NBM_POINTS_BOUNDARY) return fail(h, NBM_E_ARG, "nbm_sample: bad kind");
  int64_t H;
  if (!h_on_lattice(h_cell, &H)) return fail(h, NBM_E_INVALID_PROBLEM, "nbm_sample: h must be a multiple of 2^-24 in (0,1) (G9)");
  cudaSetDevice(h->device);
  cudaError_t e = launch_sample(kind, seed, step, nullptr, first_index, n, H, pts_dev, (cudaStream_t)stream);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_sample");
}

int nbm_sample_at(nbm_handle* h, uint64_t seed, const int64_t* step_dev, int kind, int64_t first_index, int64_t n,
                  float h_cell, float* pts_dev, void* stream) {
  if (!h || !step_dev || (n > 0 && !pts_dev) || n < 0 || first_index < 0) return fail(h, NBM_E_ARG, "nbm_sample_at: bad arguments");
  if (kind != NBM_POINTS_INTERIOR && kind != NBM_POINTS_BOUNDARY) return fail(h, NBM_E_ARG, "nbm_sample_at: bad kind");
  int64_t H;
  if (!h_on_lattice(h_cell, &H)) return fail(h, NBM_E_INVALID_PROBLEM, "nbm_sample_at: h must be a multiple of 2^-24 in (0,1) (G9)");
  cudaSetDevice(h->device);
  cudaError_t e = launch_sample(kind, seed, 0, step_dev, first_index, n, H, pts_dev, (cudaStream_t)stream);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_sample_at");
}

}  // extern "C"

namespace {
// One resolution level of the loss: interior residuals at cell width h_cell (= H 2^-24)
// weighted by `weight` (the level weight w_l of S:348; 1 for the single-level loss), the
// boundary term if `terms` selects it.  accumulate: add to loss/grad instead of writing.
int loss_grad_level(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n, const float* bpts_dev,
                    int64_t nb, float h_cell, int64_t H, int64_t n_global, int64_t nb_global, unsigned terms,
                    double weight, bool accumulate, bool pack, float* loss_dev, float* grad_dev, cudaStream_t s) {
  const DevProblem& P = h->host_problem;
  const ArchInfo& A = h->arch;
  const Workspace& w = h->ws;
  double hd = (double)h_cell;
  double dm = diag(P, 0, hd), dpl = diag(P, 1, hd);
  double ng = (double)(n_global > 0 ? n_global : 1), nbg = (double)(nb_global > 0 ? nb_global : 1);
  int launches = 0;
  cudaEvent_t* ev = nullptr;   // timing hook: 4 events of this call, no host synchronisation
  if (h->timing) {
    size_t base = (size_t)h->timed_calls * 4;
    while (h->ev.size() < base + 4) {
      cudaEvent_t x;
      if (cudaEventCreate(&x) != cudaSuccess) break;
      h->ev.push_back(x);
    }
    if (h->ev.size() >= base + 4) ev = &h->ev[base];
  }
  if (ev) cudaEventRecord(ev[0], s);
  cudaError_t e = launch_classify(h, pts_dev, n, bpts_dev, nb, H, dm, dpl, terms, false, s);
  launches += 3;
  if (e == cudaSuccess && pack && (A.prec == NBM_PREC_BF16 || A.prec == NBM_PREC_FP32X || is_fp32w(A))) {
    e = launch_pack(h, theta_dev, s);
    launches += 1;
  }
  if (e == cudaSuccess && uses_rep(A)) {
    e = cudaMemsetAsync(w.rep, 0, (size_t)w.nrep * 2 * ((A.p_net + 3) & ~3ll) * sizeof(float), s);
  }
  // no interface (NBM_LS_NONE): no crossed rows, so the crossed-row kernels are not launched;
  // their count slots and loss partial are zeroed here rather than trusted to hold the zeros
  // written at create (graph-capturable memsets)
  const bool crossing = P.ls_kind != NBM_LS_NONE;
  if (!crossing && e == cudaSuccess) e = cudaMemsetAsync(w.counts + 12, 0, 2 * sizeof(int), s);
  if (!crossing && e == cudaSuccess) e = cudaMemsetAsync(w.lpart + w.grid_mlp, 0, sizeof(double), s);
  if (crossing && e == cudaSuccess) e = launch_assemble_crossed(h, pts_dev, n, H, s);
  if (crossing) launches += 2;
  // pass A: forward-only over the crossed rows (u per row)
  MlpParams pa;
  fill_common(h, pa, theta_dev, h_cell);
  const int net1 = A.n_nets == 2 ? 1 : 0;
  for (int k = 0; k < 2; ++k) {
    pa.seg.kind[k] = kSegXRows;
    pa.seg.net[k] = k == 0 ? 0 : net1;
    pa.cnt_slot[k] = 12 + k;
    pa.seg.items[k] = w.xlist + (int64_t)k * 7 * w.xcap;
    pa.seg.src[k] = w.xrow_x;
    pa.seg.src_n[k] = 7 * w.xcap;
    pa.seg.aux[k] = w.xrow_cot;
    pa.aux_by_item[k] = 1;
  }
  pa.u_out = w.xrow_u;
  if (crossing && e == cudaSuccess) e = launch_mlp_h(h, false, pa, s);
  if (crossing && e == cudaSuccess) e = launch_crossed_residual(h, n_global > 0 ? n_global : 1, weight, s);
  if (crossing) launches += 2;
  // main fused pass over all segments (net- first, then net+)
  MlpParams pm;
  fill_common(h, pm, theta_dev, h_cell);
  pm.two_over_n = (float)(2.0 * weight / ng);
  pm.pcoef = P.mu_kind != NBM_MU_CONST ? w.pcoef : nullptr;
  for (int k = 0; k < 2; ++k) {
    const int s0 = 3 * k, net = k == 0 ? 0 : net1;
    const int side = k;
    pm.seg.kind[s0] = kSegStencil;
    pm.seg.net[s0] = net;
    pm.cnt_slot[s0] = kClsUnxMinus + side;
    pm.start_slot[s0] = kNumCls + kClsUnxMinus + side;
    pm.seg.items[s0] = w.list;
    pm.seg.src[s0] = pts_dev;
    pm.seg.src_n[s0] = n;
    pm.seg.aux[s0] = w.list_aux;
    double bs = P.beta[side], d = side ? dpl : dm;
    pm.seg.chat[s0] = (float)((-bs / (hd * hd)) / d);
    pm.seg.ccen[s0] = (float)(P.k[side] / d);
    pm.seg.kind[s0 + 1] = kSegXRows;
    pm.seg.net[s0 + 1] = net;
    pm.cnt_slot[s0 + 1] = 12 + k;
    pm.seg.items[s0 + 1] = w.xlist + (int64_t)k * 7 * w.xcap;
    pm.seg.src[s0 + 1] = w.xrow_x;
    pm.seg.src_n[s0 + 1] = 7 * w.xcap;
    pm.seg.aux[s0 + 1] = w.xrow_cot;
    pm.aux_by_item[s0 + 1] = 1;
    pm.seg.kind[s0 + 2] = kSegBRows;
    pm.seg.net[s0 + 2] = net;
    pm.cnt_slot[s0 + 2] = kClsBndMinus + side;
    pm.start_slot[s0 + 2] = kNumCls + kClsBndMinus + side;
    pm.seg.items[s0 + 2] = w.list;
    pm.seg.src[s0 + 2] = bpts_dev;
    pm.seg.src_n[s0 + 2] = nb;
    pm.seg.aux[s0 + 2] = w.list_aux;
    pm.seg.a[s0 + 2] = (float)(2.0 * P.lambda_b / nbg);
  }
  if (ev) cudaEventRecord(ev[1], s);
  if (e == cudaSuccess) e = launch_mlp_h(h, true, pm, s);
  launches += 1;
  if (ev) cudaEventRecord(ev[2], s);
  if (e == cudaSuccess)
    e = uses_rep(A) ? launch_reduce_rep(w.rep, w.nrep, A.p_net, (A.p_net + 3) & ~3ll, A.n_nets, A.n_hidden,
                                        is_w256(A) ? 1 : 0, accumulate ? 1 : 0, w.lpart, w.grid_mlp, grad_dev, loss_dev,
                                        w.err, s)
                   : launch_reduce(h, accumulate, grad_dev, loss_dev, s);
  launches += 1;
  if (ev) {
    cudaEventRecord(ev[3], s);
    h->timed_calls += 1;
  }
  h->last_launches = launches;
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_loss_grad");
}
}  // namespace

extern "C" {

int nbm_loss_grad(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n,
                  const float* bpts_dev, int64_t nb, float h_cell, int64_t n_global,
                  int64_t nb_global, unsigned terms, float* loss_dev, float* grad_dev, void* stream) {
  return nbm_loss_grad_ml(h, theta_dev, pts_dev, n, bpts_dev, nb, h_cell, 1, nullptr, n_global, nb_global, terms,
                          loss_dev, grad_dev, stream);
}

int nbm_loss_grad_ml(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n,
                     const float* bpts_dev, int64_t nb, float h0, int n_levels, const float* level_weights,
                     int64_t n_global, int64_t nb_global, unsigned terms, float* loss_dev, float* grad_dev,
                     void* stream) {
  if (!h || !theta_dev || !loss_dev || !grad_dev || n < 0 || nb < 0 || (n > 0 && !pts_dev) ||
      (nb > 0 && !bpts_dev) || n_levels < 1 || n_levels > 8)
    return fail(h, NBM_E_ARG, "nbm_loss_grad: bad arguments");
  if (n > h->ws.cap || nb > h->ws.cap) return fail(h, NBM_E_CAPACITY, "nbm_loss_grad: n or nb exceeds max_points");
  if (n_global < n || nb_global < nb) return fail(h, NBM_E_ARG, "nbm_loss_grad: global counts smaller than local");
  int64_t H0;
  if (!h_on_lattice(h0, &H0)) return fail(h, NBM_E_INVALID_PROBLEM, "nbm_loss_grad: h must be a multiple of 2^-24 in (0,1) (G9)");
  if (H0 % (1ll << (n_levels - 1)) != 0)
    return fail(h, NBM_E_INVALID_PROBLEM, "nbm_loss_grad_ml: h0 / 2^(L-1) must stay on the 2^-24 lattice (G9)");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  int launches = 0;
  for (int l = 0; l < n_levels; ++l) {
    const int64_t Hl = H0 >> l;
    const double wl = level_weights ? (double)level_weights[l] : 1.0;
    // the boundary residual does not depend on the cell width: counted once, at level 0
    const unsigned tl = l == 0 ? terms : (terms & ~(unsigned)NBM_TERM_BOUNDARY);
    const int rc = loss_grad_level(h, theta_dev, pts_dev, n, bpts_dev, l == 0 ? nb : 0, (float)((double)Hl / kLattice),
                                   Hl, n_global, nb_global, tl, wl, l > 0, l == 0, loss_dev, grad_dev, s);
    if (rc != NBM_OK) return rc;
    launches += h->last_launches;
  }
  h->last_launches = launches;
  return NBM_OK;
}

int nbm_classify(nbm_handle* h, const float* pts_dev, int64_t n, float h_cell, uint8_t* mask_dev,
                 uint8_t* cls_dev, void* stream) {
  if (!h || n < 0 || (n > 0 && (!pts_dev || !mask_dev || !cls_dev))) return fail(h, NBM_E_ARG, "nbm_classify: bad arguments");
  if (n > h->ws.cap) return fail(h, NBM_E_CAPACITY, "nbm_classify: n exceeds max_points");
  int64_t H;
  if (!h_on_lattice(h_cell, &H)) return fail(h, NBM_E_INVALID_PROBLEM, "nbm_classify: h must be a multiple of 2^-24 in (0,1) (G9)");
  if (n == 0) return NBM_OK;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  double hd = (double)h_cell;
  cudaError_t e = launch_classify(h, pts_dev, n, nullptr, 0, H, diag(h->host_problem, 0, hd),
                                  diag(h->host_problem, 1, hd), NBM_TERM_ALL, false, s, mask_dev);
  if (e == cudaSuccess) e = cudaMemcpyAsync(cls_dev, h->ws.cls, (size_t)n, cudaMemcpyDeviceToDevice, s);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_classify");
}

int nbm_eval(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n, float* u_dev,
             void* stream) {
  if (!h || !theta_dev || n < 0 || (n > 0 && (!pts_dev || !u_dev))) return fail(h, NBM_E_ARG, "nbm_eval: bad arguments");
  if (n > h->ws.cap) return fail(h, NBM_E_CAPACITY, "nbm_eval: n exceeds max_points");
  if (n == 0) return NBM_OK;
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const ArchInfo& A = h->arch;
  const Workspace& w = h->ws;
  cudaError_t e = launch_classify(h, pts_dev, n, nullptr, 0, 1, 1.0, 1.0, NBM_TERM_ALL, true, s);
  if (e == cudaSuccess) e = launch_pack(h, theta_dev, s);
  MlpParams p;
  fill_common(h, p, theta_dev, 0.0f);
  for (int k = 0; k < 2; ++k) {
    p.seg.kind[k] = kSegBRows;
    p.seg.net[k] = (A.n_nets == 2) ? k : 0;
    p.cnt_slot[k] = kClsBndMinus + k;
    p.start_slot[k] = kNumCls + kClsBndMinus + k;
    p.seg.items[k] = w.list;
    p.seg.src[k] = pts_dev;
    p.seg.src_n[k] = n;
    p.seg.aux[k] = w.list_aux;
  }
  p.u_out = u_dev;
  if (e == cudaSuccess) e = launch_mlp_h(h, false, p, s);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_eval");
}

int nbm_error_norms(nbm_handle* h, const float* theta_dev, int M, double* out_dev, void* stream) {
  if (!h || !theta_dev || !out_dev || M < 1 || M > 4096) return fail(h, NBM_E_ARG, "nbm_error_norms: bad arguments");
  const int src = h->host_problem.source;
  if (src != NBM_SRC_SINE3PI && src != NBM_SRC_PAIR && src != NBM_SRC_PAPER41)
    return fail(h, NBM_E_INVALID_PROBLEM, "nbm_error_norms: the problem has no closed-form solution");
  cudaSetDevice(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const Workspace& w = h->ws;
  const int64_t m1 = (int64_t)M + 1, total = m1 * m1 * m1;
  cudaError_t e = cudaSuccess;
  for (int64_t first = 0; first < total && e == cudaSuccess; first += w.cap) {
    const int64_t n = std::min<int64_t>(w.cap, total - first);
    e = launch_nodal_points(M, first, n, w.xrow_x, s);   // the crossed-row buffers are free here
    if (e != cudaSuccess) break;
    const int rc = nbm_eval(h, theta_dev, w.xrow_x, n, w.xrow_u, stream);
    if (rc != NBM_OK) return rc;
    e = launch_error_accum(h, w.xrow_x, w.xrow_u, n, first == 0, s);
  }
  if (e == cudaSuccess) e = launch_error_final(h, total, out_dev, s);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_error_norms");
}

int nbm_adam_step(nbm_handle* h, float* theta_dev, float* m_dev, float* v_dev, const float* grad_dev,
                  int64_t t, float lr, float b1, float b2, float eps, void* stream) {
  if (!h || !theta_dev || !m_dev || !v_dev || !grad_dev || t < 1) return fail(h, NBM_E_ARG, "nbm_adam_step: bad arguments");
  cudaSetDevice(h->device);
  float bc1 = (float)(1.0 - pow((double)b1, (double)t));
  float bc2 = (float)(1.0 - pow((double)b2, (double)t));
  cudaError_t e = launch_adam(h->arch.p_net * h->arch.n_nets, theta_dev, m_dev, v_dev, grad_dev, lr,
                              b1, b2, eps, bc1, bc2, (cudaStream_t)stream);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_adam_step");
}

int nbm_adam_step_at(nbm_handle* h, float* theta_dev, float* m_dev, float* v_dev, const float* grad_dev,
                     int64_t* t_dev, float lr, float b1, float b2, float eps, void* stream) {
  if (!h || !theta_dev || !m_dev || !v_dev || !grad_dev || !t_dev) return fail(h, NBM_E_ARG, "nbm_adam_step_at: bad arguments");
  cudaSetDevice(h->device);
  cudaError_t e = launch_adam_dev(h->arch.p_net * h->arch.n_nets, theta_dev, m_dev, v_dev, grad_dev, lr, b1, b2, eps,
                                  t_dev, h->ws.bc, (cudaStream_t)stream);
  return e == cudaSuccess ? NBM_OK : cuda_fail(h, e, "nbm_adam_step_at");
}

int nbm_timing_enable(nbm_handle* h, int enable) {
  if (!h) return NBM_E_ARG;
  h->timing = enable != 0;
  return NBM_OK;
}

int nbm_timing_read(nbm_handle* h, double* mlp_ms, double* total_ms, int64_t* calls) {
  if (!h) return NBM_E_ARG;
  double a = 0.0, b = 0.0;
  for (int64_t c = 0; c < h->timed_calls; ++c) {
    cudaEvent_t* ev = &h->ev[4 * c];
    cudaError_t e = cudaEventSynchronize(ev[3]);
    if (e != cudaSuccess) return cuda_fail(h, e, "nbm_timing_read");
    float x = 0.f, y = 0.f;
    cudaEventElapsedTime(&x, ev[1], ev[2]);
    cudaEventElapsedTime(&y, ev[0], ev[3]);
    a += x;
    b += y;
  }
  if (mlp_ms) *mlp_ms = a;
  if (total_ms) *total_ms = b;
  if (calls) *calls = h->timed_calls;
  h->timed_calls = 0;
  return NBM_OK;
}

int nbm_last_launch_count(const nbm_handle* h) { return h ? h->last_launches : 0; }

}  // extern "C"
