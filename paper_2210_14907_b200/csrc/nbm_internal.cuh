// nbm_internal.cuh -- internal declarations shared by the libnbm.so translation units.
// Nothing here is part of the C ABI (include/nbm.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "bounds.cuh"

#include "../../include/nbm.h"

namespace nbm {

constexpr int kMaxSpheres = 64;
constexpr int kMaxCharges = 64;
constexpr int kMaxLayers = 8;
constexpr int kLattice = 1 << 24;   // coordinates and h are multiples of 2^-24 (G9)

// sticky device error bits (nbm_status)
constexpr int kErrOutOfDomain = 1;
constexpr int kErrDegenerate = 2;
constexpr int kErrNonfinite = 4;

// Problem constants in fp64, resident in device memory (one copy per handle).
struct DevProblem {
  int ls_kind, n_spheres;
  double centers[kMaxSpheres][3];
  double radii[kMaxSpheres];
  double star_r0, star_amp;
  int star_m, star_n;
  double plane_n[3], plane_c;
  double beta[2], k[2];
  int source, n_charges;
  double q[kMaxCharges];
  double charge_centers[kMaxCharges][3];
  double charge_sigma;
  double lambda_b;
  float centers_f[kMaxSpheres][3];   // fp32 copies (exact: the inputs are fp32) for the filter
  float radii_f[kMaxSpheres];
  int mu_kind;                       // NBM_MU_*
  double mu_lin[2][4];
  int grid_n;                        // NBM_LS_GRID: Nc
  const float* grid_phi;             // NBM_LS_GRID: device copy of the nodal values (handle-owned)
};

// Point classes produced by the classification stage (S2).
enum : int {
  kClsUnxMinus = 0,   // interior, all 7 vertices in Omega-
  kClsUnxPlus = 1,    // interior, all 7 vertices in Omega+
  kClsCrossed = 2,    // interior, mixed stencil mask
  kClsBndMinus = 3,   // boundary point in Omega-
  kClsBndPlus = 4,    // boundary point in Omega+
  kClsSkip = 5,       // excluded (arm out of the box, or term not selected)
  kNumCls = 6
};

// Segments of the fused MLP kernel's tile space.  Ordered so that a CTA's
// contiguous tile range changes network at most once: net- segments first.
enum : int { kSegStencil = 0, kSegXRows = 1, kSegBRows = 2 };
constexpr int kNumSeg = 6;   // (stencil, xrows, brows) x (net-, net+)

struct SegTable {
  int kind[kNumSeg];
  int net[kNumSeg];
  const int* count[kNumSeg];   // device pointer to the item count
  const int* items[kNumSeg];   // item list (indices into src)
  const float* src[kNumSeg];   // AoS [][3] coordinates the items index
  int64_t src_n[kNumSeg];      // rows of src (bounds-checked builds: every item < src_n)
  const float* aux[kNumSeg];   // per-list-position scalar (rhs_hat / g / cotangent)
  float a[kNumSeg];            // boundary: 2 lambda_b / N_b,global
  float chat[kNumSeg];         // stencil: arm coefficient / diagonal (uncrossed row)
  float ccen[kNumSeg];         // stencil, stable form (G27): k / diagonal = 1 + 6 chat, in fp64
};

// item `pos` of a segment's list, range-checked in bounds-checked builds
__device__ __forceinline__ int item_at(const SegTable& t, int sg, const int* its, int pos) {
  const int it = its[pos];
  NBM_CHECK(it >= 0 && it < t.src_n[sg]);
  return it;
}

struct Workspace {
  int64_t cap;          // max points per call (interior and boundary each)
  int64_t xcap;         // crossed-point capacity (== cap)
  int nblk_cls;         // blocks of the classification grid at capacity
  // classification
  uint8_t* cls;         // [cap + cap]
  float* aux_tmp;       // [cap + cap]   rhs_hat (interior) or g (boundary) per point
  int* blk_counts;      // [nblk_cls][kNumCls]
  int* blk_offsets;     // [nblk_cls][kNumCls]
  int* counts;          // [16]: class counts, then segment counts
  int* list;            // [cap + cap]   class-partitioned indices
  float* list_aux;      // [cap + cap]
  float* pcoef;         // [cap][6] variable-mu arm coefficients c_j / d of the uncrossed rows
  // crossed rows (7 per crossed point)
  float* xrow_x;        // [7 xcap][3]
  float* xrow_u;        // [7 xcap]
  float* xrow_cot;      // [7 xcap]
  uint8_t* xrow_tag;    // [7 xcap]
  float* xrec;          // [xcap][8]  chat[7] (chat[0] = 1), rhs_hat
  int* xlist;           // [2][7 xcap] row ids partitioned by network
  // fused-MLP partials
  int grid_mlp;         // CTAs of the fused kernel (partial slots)
  int grid_base;        // launch argument: SMs (the kernel multiplies by its CTAs per SM)
  float* part;          // [2][grid_mlp][Pnet]
  int* touched;         // [2][grid_mlp]
  double* lpart;        // [grid_mlp + 1]  (+1: crossed rows' loss)
  int* err;             // sticky error word
  double* epart;        // [kErrBlocks][2] error-norm slots (sum e^2, max |e|)
  float* bc;            // [2] Adam bias corrections of the device step counter
  uint16_t* wimg;       // [2][NH-1][W*W] bf16 weight image (tensor-core path)
  uint16_t* wimg_b;     // W = 256: backward-sliced image
  float* wimg32;        // fp32 W >= 128: [2][NH-1][2][W*W] transposed / natural hidden weights
  uint8_t* hscr;        // W = 256: parked activations and G [grid][NH+1][64 KB]
  float* rep;           // bf16 W = 256 / fp32 W >= 128: gradient replicas [nrep][2][p_stride]
  int64_t hscr_len;     // bytes of hscr
  int64_t rep_len;      // floats of rep
  int nrep;
  // eval
  float* eval_aux;      // unused placeholder for symmetry
};

struct ArchInfo {
  int n_layers, width, n_hidden, act, prec, n_nets;
  int stencil;          // NBM_STENCIL_*
  int sizes[kMaxLayers];
  int64_t p_net;        // parameters per network
};

}  // namespace nbm

struct nbm_handle {
  int device;
  nbm::ArchInfo arch;
  nbm::DevProblem host_problem;
  nbm::DevProblem* d_problem;
  float* d_grid;                 // NBM_LS_GRID nodal values (device), else null
  nbm::Workspace ws;
  std::string last_error;
  // timing hook
  bool timing;
  std::vector<cudaEvent_t> ev;   // 4 events per timed call: total start, mlp start, mlp end, total end
  int64_t timed_calls;           // calls recorded since the last read
  int last_launches;
};

namespace nbm {

// cudaFuncSetAttribute applies to the current device only: `done` (a static of the caller,
// one per kernel instantiation) remembers the devices the >48 KB dynamic shared-memory limit
// has been raised on, so a second handle on another GPU (or another thread) sets it too.
inline cudaError_t smem_attr_once(std::atomic<uint64_t>& done, const void* kern, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// ---- launchers implemented in the .cu files ----
// sample_init.cu
cudaError_t launch_sample(int kind, uint64_t seed, uint64_t step, const int64_t* step_dev, int64_t first,
                          int64_t n, int64_t H, float* pts, cudaStream_t s);
cudaError_t launch_init_params(const ArchInfo& a, uint64_t seed, float* theta, cudaStream_t s);
cudaError_t launch_adam(int64_t P, float* theta, float* m, float* v, const float* g, float lr,
                        float b1, float b2, float eps, float bc1, float bc2, cudaStream_t s);
cudaError_t launch_adam_dev(int64_t P, float* theta, float* m, float* v, const float* g, float lr, float b1,
                            float b2, float eps, int64_t* t_dev, float* bc, cudaStream_t s);
// geometry.cu (compiled without FMA contraction)
cudaError_t launch_classify(const nbm_handle* h, const float* pts, int64_t n, const float* bpts,
                            int64_t nb, int64_t H, double inv_d_minus, double inv_d_plus,
                            unsigned terms, bool eval_only, cudaStream_t s,
                            uint8_t* mask_out = nullptr);
cudaError_t launch_assemble_crossed(const nbm_handle* h, const float* pts, int64_t n, int64_t H,
                                    cudaStream_t s);
cudaError_t launch_crossed_residual(const nbm_handle* h, int64_t n_global, double weight, cudaStream_t s);
constexpr int kErrBlocks = 296, kErrThreads = 256;   // error-norm reduction slots / block size
cudaError_t launch_nodal_points(int M, int64_t first, int64_t n, float* pts, cudaStream_t s);
cudaError_t launch_error_accum(const nbm_handle* h, const float* pts, const float* u, int64_t n, bool init,
                               cudaStream_t s);
cudaError_t launch_error_final(const nbm_handle* h, int64_t total, double* out, cudaStream_t s);
// mlp_fp32.cu
struct MlpParams {
  SegTable seg;
  const int* counts;         // device counts array (see nbm.cu for the slot map)
  int cnt_slot[kNumSeg];     // counts[cnt_slot] = items in the segment
  int start_slot[kNumSeg];   // counts[start_slot] = first list position (-1: 0)
  int aux_by_item[kNumSeg];  // aux indexed by item (1) or by list position (0)
  const float* theta;
  int64_t p_net;
  float h;
  float two_over_n;          // 2 / N_global
  int width_real;            // fp32 kernel: the network's hidden width (<= the kernel's W)
  const float* pcoef;        // variable mu: per interior point [n][6] arm coefficients c_j/d (else null)
  int64_t p_stride;          // partial-slot stride (p_net rounded up to 4 floats)
  float* part;               // [2][grid][p_stride]
  int* touched;              // [2][grid]
  double* lpart;             // [grid]
  float* u_out;              // forward-only mode: u_out[item] = u
  const uint16_t* wimg;      // bf16 hidden weights in the tensor-core smem layout [2][NH-1][W*W]
  // allocation lengths, for the bounds-checked build (NBM_CHECK): part (floats), the K3w parks
  // (bytes) and the gradient replicas (floats)
  int64_t part_len, hscr_len, rep_len;
};
cudaError_t launch_mlp_fp32(int width, int n_hidden, int act, bool train, bool stable, const MlpParams& p, int grid,
                            cudaStream_t s);
int mlp_fp32_supported(int width, int n_hidden, int act);
int mlp_fp32_ctas_per_sm();
// mlp_tc.cu (tcgen05 bf16)
cudaError_t launch_mlp_tc(int width, int n_hidden, int act, int planes, bool train, bool stable,
                          const MlpParams& p, int grid, cudaStream_t s);
int mlp_tc_supported(int width, int n_hidden, int act, int planes);
int mlp_tc_ctas_per_sm(int width, int n_hidden, int planes);
cudaError_t launch_pack_weights(const ArchInfo& a, const float* theta, uint16_t* wimg, cudaStream_t s);
// mlp_tch.cu (K3h: the bf16 training pass with two 64-row half-tiles in flight; tanh, direct form)
int mlp_tch_supported(int width, int n_hidden, int act);
cudaError_t launch_mlp_tch(int width, int n_hidden, const MlpParams& p, int grid, cudaStream_t s);
// mlp_fp32w.cu (fp32, W = 128 / 256: streamed weights, per-tile dW flushes into replicas)
int mlp_fp32w_supported(int width, int n_hidden);
cudaError_t launch_mlp_fp32w(int width, int n_hidden, bool train, bool stable, const MlpParams& p, const float* wimg,
                             float* rep, int nrep, int grid, cudaStream_t s);
cudaError_t launch_pack_fp32w(const ArchInfo& a, const float* theta, float* img, cudaStream_t s);
// mlp_w256.cu (tcgen05 bf16, W = 256: streamed weights, parked activations, dW replicas)
cudaError_t launch_mlp_w256(int n_hidden, bool train, bool stable, const MlpParams& m, const uint16_t* wf, const uint16_t* wb,
                            uint8_t* hscr, float* rep, int nrep, int grid, cudaStream_t s);
cudaError_t launch_pack_w256(const ArchInfo& a, const float* theta, uint16_t* wf, uint16_t* wb, cudaStream_t s);
cudaError_t launch_reduce_rep(const float* rep, int nrep, int64_t p_net, int64_t p_stride, int n_nets, int n_hidden,
                              int quad_major, int accumulate,
                              const double* lpart, int G, float* grad, float* loss, int* err, cudaStream_t s);
// reduce
cudaError_t launch_reduce(const nbm_handle* h, bool accumulate, float* grad, float* loss, cudaStream_t s);

}  // namespace nbm
