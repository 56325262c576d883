/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the NBM
 * discretized-residual loss and its parameter gradient.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path (paper_2210_14907_b200/csrc, include/nbm.h); neither includes the
 * other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md
 * line n (see DESIGN.md for the readings G1..G22 taken where the paper is
 * silent or garbled).  Everything is fp64 unless a precision-emulation mode
 * is requested (those exist only to measure the noise floor of a correct
 * fp32 / bf16 implementation, SURVEY 8c "Conditioning").
 */
#ifndef NBM_ORACLE_H
#define NBM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* level-set kinds (configs in BASELINE.json) */
enum { ORC_LS_NONE = 0, ORC_LS_SPHERES = 1, ORC_LS_STAR = 2, ORC_LS_PLANE = 3, ORC_LS_GRID = 4 };
/* data families: manufactured or physical (BASELINE.json configs 1-4) */
enum { ORC_SRC_SINE3PI = 0, ORC_SRC_PAIR = 1, ORC_SRC_GAUSS = 2, ORC_SRC_POLY2 = 3, ORC_SRC_PAPER41 = 4 };
/* diffusion coefficient mu+-(x) ("k u - div(mu grad u) = f"): constants beta+-, the
 * paper's 4.1 fields (P:68 mu- = y^2 ln(x+2) + 4, mu+ = e^{-z}), or linear test fields */
enum { ORC_MU_CONST = 0, ORC_MU_PAPER41 = 1, ORC_MU_LINEAR = 2 };
/* activations */
enum { ORC_ACT_TANH = 0, ORC_ACT_SILU = 1, ORC_ACT_SINE = 2 };
/* arithmetic modes of the MLP: exact fp64 (the oracle proper) and two
 * emulations used only to measure noise floors. */
enum { ORC_MODE_F64 = 0, ORC_MODE_F32 = 1, ORC_MODE_BF16 = 2 };
/* loss terms (per-term parity, SURVEY 8c rule 1) */
enum { ORC_T_UNX_MINUS = 0, ORC_T_UNX_PLUS = 1, ORC_T_CROSSED = 2, ORC_T_BOUNDARY = 3 };

typedef struct {
  int ls_kind;
  int n_spheres;                 /* ORC_LS_SPHERES: union (min) of spheres */
  const double* centers;         /* [n_spheres][3] */
  const double* radii;           /* [n_spheres] */
  double star_r0, star_amp;      /* ORC_LS_STAR: r - r0 - amp sin(m th) cos(n ph) */
  int star_m, star_n;
  double plane_n[3], plane_c;    /* ORC_LS_PLANE: n.x - c (test geometry) */
  double beta[2];                /* beta-, beta+  (P:40 mu-+, renamed) */
  double k[2];                   /* k-, k+         */
  int source;
  int n_charges;                 /* ORC_SRC_GAUSS */
  const double* q;               /* [n_charges] */
  const double* charge_centers;  /* [n_charges][3] */
  double charge_sigma;
  const double* poly;            /* ORC_SRC_POLY2: [2][10] c, g[3], A00 A01 A02 A11 A12 A22 */
  double lambda_b;               /* boundary weight */
  int grid_n;                    /* ORC_LS_GRID: Nc cells per axis (S:82 Sampled variant) */
  const double* grid_phi;        /* [(Nc+1)^3] nodal values over [-1,1]^3, x fastest */
  int mu_kind;                   /* ORC_MU_* */
  const double* mu_lin;          /* ORC_MU_LINEAR: [2][4] m0, mx, my, mz per side */
} orc_problem;

typedef struct {
  int n_layers;                  /* entries in sizes[], e.g. 5 for 3-64-64-64-1 */
  const int* sizes;
  int act;
  int n_nets;                    /* 1 or 2 (one network per side) */
} orc_arch;

/* One assembled stencil row. pos[0] is the centre. */
typedef struct {
  float pos[7][3];
  int tag[7];                    /* 0 = net-, 1 = net+ : which side's network evaluates pos[j] */
  double coef[7];                /* A-row entries; coef[0] == d */
  double f;                      /* f_s(p) */
  double corr;                   /* sum of crossed-arm corrections; rhs = f - corr (G3) */
  double rhs;                    /* b_p */
  double d;                      /* diagonal d_p (Jacobi M) */
  int side;                      /* side of the centre: 0 = Omega-, 1 = Omega+ */
  int mask;                      /* bit0 side(p), bit j side(q_j) */
  int crossed;                   /* mask is mixed (class 2) */
  int n_crossed_arms;            /* crossed arms that were not snapped */
  int n_snapped;                 /* arms with theta outside [1e-6, 1-1e-6] */
  double theta[7];               /* theta per arm (0 if uncrossed) */
} orc_row;

/* ---- Philox4x32-10 counter-based generator (Salmon et al. 2011) ---- */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* ---- sampler (S:336-344 UniformRandom; lattice reading G9) ----
 * kind 0 = interior points on the 2^-24 lattice in [-1+h, 1-h]^3,
 * kind 1 = boundary points on the six faces.  H = h * 2^24 (integer).
 * point i uses global index first+i. */
void orc_sample(int kind, uint64_t seed, uint64_t step, int64_t first, int64_t n,
                int64_t H, float* pts);

/* ---- geometry ---- */
double orc_phi(const orc_problem* pb, const double x[3]);
int orc_side(const orc_problem* pb, const double x[3]);   /* 0 = Omega- (phi<=0), 1 = Omega+ */
/* crossing on segment a->b, closed form for spheres/plane, bisection for the star.
 * returns 1 if sides differ (theta, xg, nrm filled), 0 otherwise, <0 on error */
int orc_crossing(const orc_problem* pb, const double a[3], const double b[3],
                 double* theta, double xg[3], double nrm[3]);
/* plain 200-step bisection on the side function (independent cross-check) */
int orc_crossing_bisect(const orc_problem* pb, const double a[3], const double b[3], double* theta);
int orc_normal(const orc_problem* pb, const double x[3], double nrm[3]);

/* ---- problem data (P:40-41 jump problem, configs) ---- */
int orc_exact(const orc_problem* pb, int side, const double x[3], double* u, double grad[3]);
double orc_f(const orc_problem* pb, int side, const double x[3]);
double orc_mu(const orc_problem* pb, int side, const double x[3], double grad[3]);
double orc_alpha(const orc_problem* pb, const double x[3]);
double orc_sigma(const orc_problem* pb, const double x[3], const double n[3]);
double orc_g(const orc_problem* pb, const double x[3]);

/* ---- kernel assembly (S:252-258 with the sign reading G3) ----
 * returns 0, or -1 OutOfDomain (an arm leaves [-1,1]^3), -2 DegenerateGradient.
 * sign_mutation != 0 applies S:257's literal "add to rhs" (mutation test only). */
int orc_assemble(const orc_problem* pb, const float p[3], float h, int sign_mutation, orc_row* row);
int orc_classify(const orc_problem* pb, const float* pts, int64_t n, float h,
                 uint8_t* mask, uint8_t* cls);

/* ---- surrogate ---- */
int64_t orc_param_count(const orc_arch* a);              /* all nets */
void orc_init_params(const orc_arch* a, uint64_t seed, float* theta);  /* Xavier, G11 */
/* u = net_k(x) in the given mode.  theta is fp64: the CUDA path's fp32 theta is
 * promoted exactly by the caller; finite-difference pins perturb it in fp64.
 * bf16 mode rounds the hidden x hidden GEMM operands to bf16 (G16). */
double orc_forward(const orc_arch* a, const double* theta, int net, const double x[3], int mode);
/* grad += cot * d net_k(x) / d theta  (fp64 reverse accumulation) */
void orc_backward(const orc_arch* a, const double* theta, int net, const double x[3],
                  double cot, int mode, double* grad);

/* ---- loss and gradient (G1, G18) ----
 * loss_terms[4] and grad[P] are outputs (sum of the selected terms);
 * grad_terms may be NULL or [4][P].  Each interior point uses h; the global
 * means divide by n_glob and nb_glob.  terms = bitmask over ORC_T_*.
 * nthreads <= 0 means all OpenMP threads.  Returns 0 or an assembly error. */
int orc_loss_grad(const orc_problem* pb, const orc_arch* a, const double* theta,
                  const float* pts, int64_t n, const float* bpts, int64_t nb, float h,
                  int64_t n_glob, int64_t nb_glob, int mode, unsigned terms,
                  double* loss_terms, double* grad, double* grad_terms, int nthreads);

/* residuals (r per interior point, r_b per boundary point), fp64 */
int orc_residuals(const orc_problem* pb, const orc_arch* a, const double* theta,
                  const float* pts, int64_t n, const float* bpts, int64_t nb, float h,
                  int mode, double* r, double* rb);

/* raw and r = raw/d with the manufactured exact solution substituted for the
 * networks (S:263 truncation oracle); cls[i] = 0/1 uncrossed side, 2 crossed */
int orc_residual_exact(const orc_problem* pb, const float* pts, int64_t n, float h,
                       double* raw, double* r, uint8_t* cls);

/* u at points, network chosen by side(p) */
void orc_eval(const orc_problem* pb, const orc_arch* a, const double* theta,
              const float* pts, int64_t n, int mode, double* u);

/* rmse, linf of u_{side} - u* over the (M+1)^3 nodal grid; -1: no exact solution */
int orc_error_norms(const orc_problem* pb, const orc_arch* a, const double* theta, int M,
                    int mode, double out[2]);

/* ---- Adam ---- fp64 and an fp32 mirror with a fixed op order */
void orc_adam(int64_t P, double* theta, double* m, double* v, const double* g,
              int64_t t, double lr, double b1, double b2, double eps);
void orc_adam_f32(int64_t P, float* theta, float* m, float* v, const float* g,
                  int64_t t, float lr, float b1, float b2, float eps);

int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
