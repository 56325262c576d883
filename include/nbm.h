/*
 * nbm.h -- C ABI of libnbm.so, the B200-native hot path of the Neural
 * Bootstrapping Method (arXiv 2210.14907): batched discretized-residual loss
 * L = (1/N) sum r_i^2 + (lambda_b/N_b) sum r_b^2 and dL/dtheta over random
 * collocation points, with MLP surrogates evaluated on 7-point implicit cells
 * and the sharp-interface (jump-corrected) flux stencil.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Gk = reading k in
 * DESIGN.md section 3.
 *
 * Conventions for every entry point:
 *  - Return value: int status, NBM_OK (0) or one of the NBM_E_* codes below.
 *    nbm_last_error(h) gives a human-readable message for the last failure.
 *  - Pointers named *_dev are CUDA device pointers on the handle's device,
 *    owned by the caller (PyTorch tensors in the Python binding); the library
 *    never frees them and never keeps them beyond the call.
 *  - `stream` is a cudaStream_t passed as void*; every call that takes one is
 *    asynchronous on it and never synchronises the host (except nbm_status).
 *  - The library owns only the workspace allocated by nbm_create (class lists,
 *    crossed-row records, per-CTA gradient partials), sized by max_points.
 *  - A handle is bound to one device and is not thread-safe.
 */
#ifndef NBM_H
#define NBM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (S:99, S:117, S:259, S:367 mapped to the ABI) ---- */
#define NBM_OK                 0
#define NBM_E_INVALID_ARCH     1  /* sizes[0] != 3, last != 1, no hidden layer, unsupported width/depth */
#define NBM_E_INVALID_PROBLEM  2  /* beta <= 0, bad level set, box != [-1,1]^3 (G23), h not on the 2^-24 lattice (G9) */
#define NBM_E_CAPACITY         3  /* n or nb exceeds max_points given to nbm_create */
#define NBM_E_CUDA             4  /* a CUDA runtime error (message in nbm_last_error) */
#define NBM_E_ARG              5  /* null pointer / negative size / bad enum */
#define NBM_E_OUT_OF_DOMAIN    6  /* device-sticky: an arm p +- h e_d left the box */
#define NBM_E_DEGENERATE       7  /* device-sticky: |grad phi| < 1e-12 at a crossing */
#define NBM_E_NONFINITE        8  /* device-sticky: non-finite loss or gradient */

/* ---- level sets (configs in BASELINE.json) ---- */
#define NBM_LS_NONE     0  /* phi = -1: everything is Omega- (config 1) */
#define NBM_LS_SPHERES  1  /* phi = min_k (|x - c_k| - r_k), union of n spheres (configs 2, 4) */
#define NBM_LS_STAR     2  /* phi = r - r0 - amp sin(m th) cos(n ph), th from +z, ph = atan2(y,x) (config 3, G13) */
#define NBM_LS_PLANE    3  /* phi = n.x - c */
#define NBM_LS_GRID     4  /* Sampled level set ("a separate coarse mesh"): trilinear
                            * interpolation of nodal values on an (Nc+1)^3 grid over [-1,1]^3;
                            * crossings at the root of the linear interpolant between the arm's end
                            * values; normals by central differences of the interpolant with
                            * step hc/2 */

/* ---- data families: f, alpha = [u], sigma = [beta d_n u], g derived inside the library ---- */
#define NBM_SRC_SINE3PI  0  /* u = sin(pi x) sin(pi y) sin(pi z) on both sides (config 1) */
#define NBM_SRC_PAIR     1  /* u- = e^x cos(y) z, u+ = sin(x+y+z) (configs 2, 4, 5; G12) */
#define NBM_SRC_GAUSS    2  /* f = sum_k q_k N(x; c_k, s^2 I), alpha = sigma = g = 0 (config 3; G13) */
#define NBM_SRC_PAPER41  4  /* the paper's 4.1 benchmark: u- = e^z, u+ = cos(x) sin(y),
                             * f = k u - div(mu grad u) with the problem's mu+-, alpha = [u],
                             * sigma = [mu d_n u], g = u of the side */

/* diffusion coefficient mu+-(x) */
#define NBM_MU_CONST     0  /* beta_minus / beta_plus */
#define NBM_MU_PAPER41   1  /* mu- = y^2 ln(x+2) + 4, mu+ = e^{-z} */
#define NBM_MU_LINEAR    2  /* mu_s(x) = m0 + mx x + my y + mz z (mu_lin[s]); > 0 on the box */

#define NBM_ACT_TANH  0
#define NBM_ACT_SILU  1
#define NBM_ACT_SINE  2     /* P:68 "sine-activated neurons"; init +-sqrt(6/fan_in) */
#define NBM_PREC_FP32 0     /* IEEE fp32 arithmetic throughout (G15) */
#define NBM_PREC_BF16 1     /* bf16 tensor-core hidden GEMMs, fp32 accumulate (G16) */
#define NBM_PREC_FP32X 2    /* fp32-accurate hidden GEMMs on the tensor cores: each fp32 operand split
                             * exactly into three bf16 planes, the six plane products with
                             * i + j <= 2 summed in fp32 (relative error <= ~2^-22 per product),
                             * accurate tanh, everything else fp32 (G26); W = 64, 2-3 hidden layers */

/* evaluation of the uncrossed 7-point stencil (G27) */
#define NBM_STENCIL_DIRECT 0  /* the 7 network values, r = u + c_hat sum_j u_j - b/d */
#define NBM_STENCIL_STABLE 1  /* the same r through difference propagation: every hidden layer carries
                               * the centre activation, the first differences a(x + h e_d) - a(x) and
                               * the second differences a(x + h e_d) + a(x - h e_d) - 2 a(x) (tanh
                               * addition theorem, no cancellation), r = (k/d) u + c_hat sum_d D_d u
                               * - b/d; resolves r at small h (bf16 to ~1e-2, fp32 to the fp32
                               * bars).  Tanh networks, BF16 or FP32, constant mu; crossed and
                               * boundary rows are evaluated directly */

#define NBM_POINTS_INTERIOR 0
#define NBM_POINTS_BOUNDARY 1

/* loss terms (bitmask for nbm_loss_grad; per-term parity, SURVEY 8c rule 1) */
#define NBM_TERM_UNX_MINUS  1u  /* interior points whose 7 stencil vertices are all in Omega- */
#define NBM_TERM_UNX_PLUS   2u  /* ... all in Omega+ */
#define NBM_TERM_CROSSED    4u  /* interior points whose stencil mask is mixed */
#define NBM_TERM_BOUNDARY   8u  /* Dirichlet residuals on the cube faces */
#define NBM_TERM_ALL       15u

typedef struct nbm_levelset {
  int kind;                      /* NBM_LS_* */
  int n;                         /* number of spheres (NBM_LS_SPHERES, 1..64) */
  const float* centers;          /* host, [n][3], copied at create */
  const float* radii;            /* host, [n], copied at create, > 0 */
  float star_r0, star_amp;       /* NBM_LS_STAR */
  int star_m, star_n;            /* angular frequencies, 0..16 */
  float plane_n[3], plane_c;     /* NBM_LS_PLANE */
  int grid_n;                    /* NBM_LS_GRID: Nc cells per axis, 1..1024 */
  const float* grid_phi;         /* NBM_LS_GRID: host, [(Nc+1)^3] nodal values, x fastest
                                  * (S:145 order), copied to the device at create */
} nbm_levelset;

/* Problem descriptor (k u - div(beta grad u) = f, [u] = alpha,
 * [beta d_n u] = sigma, Dirichlet data on the cube).  Copied at create. */
typedef struct nbm_problem {
  float box_lo[3], box_hi[3];    /* must be [-1,1]^3 (G23) */
  nbm_levelset ls;
  float beta_minus, beta_plus;   /* > 0, constant per phase (P:40 mu-+) */
  float k_minus, k_plus;         /* >= 0, constant per phase (G20) */
  int source;                    /* NBM_SRC_* */
  int n_charges;                 /* NBM_SRC_GAUSS, 0..64 */
  const float* q;                /* host, [n_charges] */
  const float* charge_centers;   /* host, [n_charges][3] */
  float charge_sigma;            /* > 0 */
  float lambda_b;                /* boundary weight, >= 0 */
  int mu_kind;                   /* NBM_MU_*: variable coefficients are evaluated at the arm's face
                                  * midpoint (uncrossed arms) and at x_Gamma (crossed arms,
                                  * S:257); supported by the fp32 kernel (W <= 64) */
  float mu_lin[2][4];            /* NBM_MU_LINEAR: m0, mx, my, mz for Omega-, Omega+ */
} nbm_problem;

/* MLP surrogate (P:60 two networks, one per side).  sizes = [3, W, ..., W, 1]
 * with uniform hidden width W.  Supported (others return NBM_E_INVALID_ARCH):
 *   FP32 tanh: W <= 32 with 1..5 hidden layers, W <= 64 with 1..4 (padded to 16/32/64),
 *              W in {128, 256} with 2..4;
 *   FP32 sine: W <= 32 with 1..5 hidden layers (the paper's 5 x 10 nets);
 *   BF16 (tcgen05): W in {64, 128} tanh or SiLU, W = 256 tanh, 2..4 hidden layers;
 *   FP32X (tcgen05, three bf16 planes): W = 64 tanh, 2..4 hidden layers (4: streamed weights).
 * Variable mu (nbm_problem.mu_kind) runs on every direct-form kernel except FP32X.  stencil =
 * NBM_STENCIL_STABLE needs tanh with FP32 or BF16 (any of the widths above) and constant mu. */
typedef struct nbm_arch {
  int n_layers;                  /* entries of sizes[] (>= 3) */
  const int* sizes;              /* host */
  int act;                       /* NBM_ACT_* */
  int prec;                      /* NBM_PREC_* */
  int n_nets;                    /* 1 (shared) or 2 (net-, net+) */
  int stencil;                   /* NBM_STENCIL_* (0 = direct) */
} nbm_arch;

typedef struct nbm_handle nbm_handle;

/* ---- host-only helpers (no device work; usable without a GPU) ---- */
/* Number of parameters of the flat theta: sum_l (fan_in fan_out + fan_out) per net, times
 * n_nets.  Layout (G17): net- then net+; per layer W_l row-major
 * [fan_out][fan_in] then b_l.  Returns -1 for an invalid arch. */
int64_t nbm_arch_param_count(const nbm_arch* arch);
/* Validate descriptors exactly as nbm_create does: NBM_OK or NBM_E_INVALID_*. */
int nbm_check(const nbm_problem* problem, const nbm_arch* arch);
/* Library version string. */
const char* nbm_version(void);

/* ---- lifetime ---- */
/* Create a handle on `device`: validates and copies the descriptors, uploads the
 * problem constants, and allocates the workspace for up to max_points interior and
 * max_points boundary points per call.  *out is set only on NBM_OK. */
int nbm_create(const nbm_problem* problem, const nbm_arch* arch, int device,
               int64_t max_points, nbm_handle** out);
void nbm_destroy(nbm_handle* h);
int64_t nbm_param_count(const nbm_handle* h);
const char* nbm_last_error(const nbm_handle* h);
/* Synchronise `stream`, then return and clear the sticky device error word
 * (NBM_E_OUT_OF_DOMAIN / NBM_E_DEGENERATE / NBM_E_NONFINITE) or a CUDA error. */
int nbm_status(nbm_handle* h, void* stream);

/* ---- the hot path ---- */

/* Xavier/Glorot-uniform init, zero biases (G11; "fully determined by seed"):
 * theta_dev [P] fp32. */
int nbm_init_params(nbm_handle* h, uint64_t seed, float* theta_dev, void* stream);

/* Random collocation points ("randomly sampled points"; G9).
 * kind = NBM_POINTS_INTERIOR: uniform on the 2^-24 lattice in [-1+h, 1-h]^3;
 * NBM_POINTS_BOUNDARY: uniform on the six faces.  Point i of this call is global
 * index first_index + i, so shards drawn by different ranks form one global set.
 * h_cell must be a multiple of 2^-24 in (0, 1).  pts_dev: [n][3] fp32 (AoS). */
int nbm_sample(nbm_handle* h, uint64_t seed, uint64_t step, int kind, int64_t first_index,
               int64_t n, float h_cell, float* pts_dev, void* stream);
/* As nbm_sample, with the step word of the Philox counter read from device memory at run
 * time (*step_dev, int64, 0-based), so a captured CUDA graph replays successive steps
 * (SURVEY 7.3 hard part 9).  step_dev is caller-owned; the library only reads it. */
int nbm_sample_at(nbm_handle* h, uint64_t seed, const int64_t* step_dev, int kind,
                  int64_t first_index, int64_t n, float h_cell, float* pts_dev, void* stream);

/* Loss and gradient (G1-G3, G18).
 * For each interior point p (pts_dev [n][3]): place the implicit cell of width h_cell,
 * classify its 7 vertices by phi (tie -> Omega-), assemble the sharp-interface row,
 * evaluate the side-tagged networks at the 7 vertices, r = (A u - b)/d.  For each
 * boundary point (bpts_dev [nb][3]): r_b = u_side(p)(p) - g(p).
 *   loss_dev[0] = (1/n_global) sum r^2 + (lambda_b/nb_global) sum r_b^2   (this rank's share)
 *   grad_dev[P] = d loss / d theta                                         (this rank's share)
 * over the terms selected by `terms` (NBM_TERM_*).  With data parallelism each rank
 * passes its own shard and the global counts; all-reduce(sum) of [grad, loss] then
 * yields the global L and dL/dtheta exactly.  loss_dev and grad_dev are
 * overwritten.  Points must lie on the 2^-24 lattice with all arms inside the box
 * (else the sticky NBM_E_OUT_OF_DOMAIN is raised and those points contribute 0).
 * Deterministic: identical inputs give bitwise-identical outputs (G21). */
int nbm_loss_grad(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n,
                  const float* bpts_dev, int64_t nb, float h_cell, int64_t n_global,
                  int64_t nb_global, unsigned terms, float* loss_dev, float* grad_dev,
                  void* stream);

/* Multi-resolution loss ("placing implicit cells at multi-resolutions", "three
 * levels of implicit refinement").  The same centres
 * are evaluated at n_levels cell widths h_l = h0 / 2^l, l = 0..n_levels-1:
 *   loss = (1/n_global) sum_p sum_l w_l r_p(h_l)^2 + (lambda_b/nb_global) sum_b r_b^2
 * with level_weights (host, [n_levels]; NULL = all 1) and the boundary term counted
 * once.  h0 / 2^(n_levels-1) must stay on the 2^-24 lattice (else NBM_E_INVALID_PROBLEM);
 * 1 <= n_levels <= 8.  nbm_loss_grad is this call with n_levels = 1.  Deterministic like
 * nbm_loss_grad (the levels are added in level order). */
int nbm_loss_grad_ml(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n,
                     const float* bpts_dev, int64_t nb, float h0, int n_levels,
                     const float* level_weights, int64_t n_global, int64_t nb_global,
                     unsigned terms, float* loss_dev, float* grad_dev, void* stream);

/* Stencil classification alone ("calculating interface-cell crossings"):
 * for each interior point, mask_dev[i] bit 0 = side(p), bit j (1..6) = side(p + arm_j)
 * with arms +x,-x,+y,-y,+z,-z and side = (phi > 0) (tie -> Omega-); cls_dev[i] =
 * 0 all Omega-, 1 all Omega+, 2 mixed (crossed), 5 an arm left the box.  u8 outputs [n].
 * This is the same classification nbm_loss_grad runs internally (exposed for parity). */
int nbm_classify(nbm_handle* h, const float* pts_dev, int64_t n, float h_cell, uint8_t* mask_dev,
                 uint8_t* cls_dev, void* stream);

/* Surrogate evaluation: u_dev[i] = net_side(p_i)(p_i), side by phi. */
int nbm_eval(nbm_handle* h, const float* theta_dev, const float* pts_dev, int64_t n,
             float* u_dev, void* stream);

/* Error norms against the problem's closed-form solution (the RMSE and L-inf
 * columns of Table 1).  Over the (M+1)^3 nodal points p of the
 * box (coordinates -1 + 2 i / M in fp64 rounded to fp32, x fastest):
 * e(p) = u_side(p)(p) - u*_side(p)(p) with the network evaluated as nbm_eval does and u* in
 * fp64; out_dev (device, double[2]) receives rmse = sqrt(mean e^2) and linf = max |e|.
 * Runs in chunks of max_points through the eval path (overwrites the workspace's crossed-row
 * buffers; stream-ordered with nbm_loss_grad).  Deterministic (fixed-order reductions).
 * Errors: NBM_E_ARG (M outside 1..4096, null pointers), NBM_E_INVALID_PROBLEM (a source
 * without a closed-form solution: NBM_SRC_GAUSS). */
int nbm_error_norms(nbm_handle* h, const float* theta_dev, int M, double* out_dev, void* stream);

/* Adam (G19), in place on fp32 theta, m, v given grad, all [P]; t is the
 * 1-based step after increment.  Per element: m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
 * theta -= lr (m/bc1) / (sqrt(v/bc2) + eps) with bc_k = 1 - b_k^t computed in fp64. */
int nbm_adam_step(nbm_handle* h, float* theta_dev, float* m_dev, float* v_dev,
                  const float* grad_dev, int64_t t, float lr, float b1, float b2, float eps,
                  void* stream);
/* As nbm_adam_step with a device step counter (CUDA-graph replay): t = *t_dev + 1 is used
 * for the bias corrections (the same fp64 formula, one fp32 rounding), then *t_dev = t.
 * *t_dev is the number of completed steps, so nbm_sample_at(step_dev = t_dev) earlier in
 * the same step draws step t - 1, as the host-counter calls do.  Two kernel launches. */
int nbm_adam_step_at(nbm_handle* h, float* theta_dev, float* m_dev, float* v_dev,
                     const float* grad_dev, int64_t* t_dev, float lr, float b1, float b2,
                     float eps, void* stream);

/* ---- measurement hook (bench.py) ----
 * When enabled, nbm_loss_grad records CUDA events around its fused MLP kernel launches
 * on `stream`; nbm_timing_read synchronises and returns the accumulated milliseconds
 * and the number of calls timed since the last read. */
int nbm_timing_enable(nbm_handle* h, int enable);
int nbm_timing_read(nbm_handle* h, double* mlp_ms, double* total_ms, int64_t* calls);
/* number of CUDA kernels launched by the last nbm_loss_grad call */
int nbm_last_launch_count(const nbm_handle* h);

#ifdef __cplusplus
}
#endif
#endif
