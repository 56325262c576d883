// geometry.cu -- K2: implicit cell placement, level-set classification, stable class
// partition, crossed-row assembly and the crossed rows' residual/cotangents.
//
// Compiled with -fmad=false: every fp64 operation of the level set is a single IEEE
// rounding in the written order, so side(x) (phi <= 0) is bit-identical to the
// oracle's and the stencil masks match exactly (SURVEY 8c "K2 masks: bit-exact").
//
// Passages: P:52 (Fig. 2 caption: "placing implicit cells ... calculating
// interface-cell crossings"), P:59-60 (sharp-interface kernel, level set, M^-1),
// S:76-149 (geometry), S:252-258 (assembly, sign reading G3), S:303 (snapping G6).
#include <math.h>

#include "nbm_internal.cuh"

namespace nbm {

constexpr int kClsBlock = 256;     // threads per classification block
constexpr int kClsPerThread = 4;   // items per thread
constexpr int kClsItems = kClsBlock * kClsPerThread;

// ------------------------------------------------------------------ level sets
__device__ double d_sphere_phi(const DevProblem& P, int k, const double x[3]) {
  double dx = x[0] - P.centers[k][0], dy = x[1] - P.centers[k][1], dz = x[2] - P.centers[k][2];
  return sqrt((dx * dx + dy * dy) + dz * dz) - P.radii[k];
}

// star (G13): r - r0 - amp * [sin(th) U_{m-1}(cos th)] * T_n(cos ph)
__device__ double d_star_phi(const DevProblem& P, const double x[3]) {
  double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
  double r = sqrt(rho * rho + x[2] * x[2]);
  if (r == 0.0) return -P.star_r0;
  if (rho == 0.0) return r - P.star_r0;
  double ct = x[2] / r, st = rho / r, cp = x[0] / rho;
  double um = 1.0;
  if (P.star_m > 1) {
    double ua = 1.0, ub = 2.0 * ct;
    for (int k = 2; k < P.star_m; ++k) {
      double uc = 2.0 * ct * ub - ua;
      ua = ub;
      ub = uc;
    }
    um = ub;
  }
  double tn = 1.0;
  if (P.star_n > 0) {
    double ta = 1.0, tb = cp;
    for (int k = 1; k < P.star_n; ++k) {
      double tc = 2.0 * cp * tb - ta;
      ta = tb;
      tb = tc;
    }
    tn = tb;
  }
  return (r - P.star_r0) - P.star_amp * ((st * um) * tn);
}

// Sampled level set (S:82, P:60 coarse mesh): trilinear interpolation of the nodal values with a
// fixed operation order (s = (x + 1) Nc/2 clamped to the cube, cell index, then seven
// a + t (b - a) along x, y, z), bit-identical to the oracle under -fmad=false.
__device__ __forceinline__ double d_lerp(double a, double b, double t) { return a + t * (b - a); }
__device__ double d_grid_phi(const DevProblem& P, const double x[3]) {
  const int nc = P.grid_n, n1 = nc + 1;
  const double half = 0.5 * (double)nc;
  int i[3];
  double t[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double sd = (x[d] + 1.0) * half;
    if (sd < 0.0) sd = 0.0;
    if (sd > (double)nc) sd = (double)nc;
    int id = (int)floor(sd);
    if (id > nc - 1) id = nc - 1;
    i[d] = id;
    t[d] = sd - (double)id;
  }
  const float* g = P.grid_phi + (int64_t)i[0] + (int64_t)n1 * ((int64_t)i[1] + (int64_t)n1 * i[2]);
  const int64_t sy = n1, sz = (int64_t)n1 * n1;
  const double c00 = d_lerp((double)__ldg(g), (double)__ldg(g + 1), t[0]);
  const double c10 = d_lerp((double)__ldg(g + sy), (double)__ldg(g + sy + 1), t[0]);
  const double c01 = d_lerp((double)__ldg(g + sz), (double)__ldg(g + sz + 1), t[0]);
  const double c11 = d_lerp((double)__ldg(g + sz + sy), (double)__ldg(g + sz + sy + 1), t[0]);
  const double c0 = d_lerp(c00, c10, t[1]), c1 = d_lerp(c01, c11, t[1]);
  return d_lerp(c0, c1, t[2]);
}

__device__ double d_phi(const DevProblem& P, const double x[3]) {
  switch (P.ls_kind) {
    case NBM_LS_SPHERES: {
      double m = d_sphere_phi(P, 0, x);
      for (int k = 1; k < P.n_spheres; ++k) m = fmin(m, d_sphere_phi(P, k, x));
      return m;
    }
    case NBM_LS_STAR:
      return d_star_phi(P, x);
    case NBM_LS_PLANE:
      return ((P.plane_n[0] * x[0] + P.plane_n[1] * x[1]) + P.plane_n[2] * x[2]) - P.plane_c;
    case NBM_LS_GRID:
      return d_grid_phi(P, x);
    default:
      return -1.0;
  }
}

__device__ __forceinline__ int d_side_exact(const DevProblem& P, const double x[3]) {
  return d_phi(P, x) <= 0.0 ? 0 : 1;
}

// side(x) = (phi(x) > 0), tie -> Omega- (S:84), identical to the fp64 definition: an fp32
// filter decides whenever its margin exceeds its error bound, else the fp64 formula runs.
//  spheres: |x-c|^2 vs r^2 in fp32 (relative error < 4e-7) with a 1e-5 relative margin;
//  star:    the fp32 formula with a margin above its error bound (>= 1e-5 (2 + r)).
// sphere filter over fp32 sphere data [n][4] = (cx, cy, cz, r) (shared-memory copy in K2a)
__device__ __forceinline__ int d_side_spheres(const DevProblem& P, const float4* __restrict__ sph, const double x[3]) {
  const float x0 = (float)x[0], x1 = (float)x[1], x2 = (float)x[2];
  bool unsure = false;
  for (int k = 0; k < P.n_spheres; ++k) {
    const float4 c = sph[k];
    const float dx = x0 - c.x, dy = x1 - c.y, dz = x2 - c.z;
    const float d2 = (dx * dx + dy * dy) + dz * dz;
    const float r2 = c.w * c.w;
    if (d2 < r2 * (1.0f - 1e-5f)) return 0;          // certainly inside sphere k
    if (d2 <= r2 * (1.0f + 1e-5f)) unsure = true;
  }
  if (!unsure) return 1;                              // certainly outside all spheres
  return d_side_exact(P, x);
}

__device__ __forceinline__ int d_side(const DevProblem& P, const double x[3]) {
  if (P.ls_kind == NBM_LS_SPHERES) {
    const float x0 = (float)x[0], x1 = (float)x[1], x2 = (float)x[2];
    bool unsure = false;
    for (int k = 0; k < P.n_spheres; ++k) {
      const float dx = x0 - P.centers_f[k][0], dy = x1 - P.centers_f[k][1], dz = x2 - P.centers_f[k][2];
      const float d2 = (dx * dx + dy * dy) + dz * dz;
      const float r2 = P.radii_f[k] * P.radii_f[k];
      if (d2 < r2 * (1.0f - 1e-5f)) return 0;          // certainly inside sphere k
      if (d2 <= r2 * (1.0f + 1e-5f)) unsure = true;
    }
    if (!unsure) return 1;                              // certainly outside all spheres
    return d_side_exact(P, x);
  }
  if (P.ls_kind == NBM_LS_STAR) {
    const float x0 = (float)x[0], x1 = (float)x[1], x2 = (float)x[2];
    const float rho = sqrtf(x0 * x0 + x1 * x1), r = sqrtf(rho * rho + x2 * x2);
    if (r > 1e-3f && rho > 1e-3f) {
      const float ct = x2 / r, st = rho / r, cp = x0 / rho;
      float um = 1.0f;
      if (P.star_m > 1) {
        float ua = 1.0f, ub = 2.0f * ct;
        for (int k = 2; k < P.star_m; ++k) { const float uc = 2.0f * ct * ub - ua; ua = ub; ub = uc; }
        um = ub;
      }
      float tn = 1.0f;
      if (P.star_n > 0) {
        float ta = 1.0f, tb = cp;
        for (int k = 1; k < P.star_n; ++k) { const float tc = 2.0f * cp * tb - ta; ta = tb; tb = tc; }
        tn = tb;
      }
      const float ph = (r - (float)P.star_r0) - (float)P.star_amp * ((st * um) * tn);
      const float mm = (float)(P.star_m + 1), nn = (float)(P.star_n + 1);
      const float margin = 1e-5f * (2.0f + r) + 1e-6f * fabsf((float)P.star_amp) * (mm * mm) * (nn * nn);
      if (ph > margin) return 1;
      if (ph < -margin) return 0;
    }
    return d_side_exact(P, x);
  }
  return d_side_exact(P, x);
}

// Unit normal Omega- -> Omega+ at x (G7). Returns false if degenerate.
__device__ bool d_normal(const DevProblem& P, const double x[3], double n[3]) {
  double g[3];
  if (P.ls_kind == NBM_LS_PLANE) {
    g[0] = P.plane_n[0]; g[1] = P.plane_n[1]; g[2] = P.plane_n[2];
  } else if (P.ls_kind == NBM_LS_SPHERES) {
    int best = 0;
    double m = d_sphere_phi(P, 0, x);
    for (int k = 1; k < P.n_spheres; ++k) {
      double v = d_sphere_phi(P, k, x);
      if (v < m) { m = v; best = k; }
    }
    for (int d = 0; d < 3; ++d) g[d] = x[d] - P.centers[best][d];
  } else {
    const double e = P.ls_kind == NBM_LS_GRID ? 1.0 / (double)P.grid_n : 1e-5;   // S:116 (Sampled: hc/2)
    for (int d = 0; d < 3; ++d) {
      double xp[3] = {x[0], x[1], x[2]}, xm[3] = {x[0], x[1], x[2]};
      xp[d] += e;
      xm[d] -= e;
      g[d] = (d_phi(P, xp) - d_phi(P, xm)) / (2.0 * e);
    }
  }
  double nn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  if (!(nn >= 1e-12)) return false;
  n[0] = g[0] / nn; n[1] = g[1] / nn; n[2] = g[2] / nn;
  return true;
}

// Crossing on the arm a -> b (sides differ); theta nearest to a (G8).
__device__ double d_crossing_theta(const DevProblem& P, const double a[3], const double b[3], int sa) {
  double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  if (P.ls_kind == NBM_LS_PLANE) {
    double nd = P.plane_n[0] * d[0] + P.plane_n[1] * d[1] + P.plane_n[2] * d[2];
    return -d_phi(P, a) / nd;
  }
  if (P.ls_kind == NBM_LS_GRID) {   // S:125 Sampled: root of the linear interpolant of the end values
    const double pa = d_phi(P, a), pb = d_phi(P, b);
    return pa / (pa - pb);
  }
  if (P.ls_kind == NBM_LS_SPHERES) {
    double best = -1.0;
    for (int k = 0; k < P.n_spheres; ++k) {
      double ac[3] = {a[0] - P.centers[k][0], a[1] - P.centers[k][1], a[2] - P.centers[k][2]};
      double A = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      double B = 2.0 * (ac[0] * d[0] + ac[1] * d[1] + ac[2] * d[2]);
      double C = (ac[0] * ac[0] + ac[1] * ac[1] + ac[2] * ac[2]) - P.radii[k] * P.radii[k];
      double disc = B * B - 4.0 * A * C;
      if (disc < 0.0 || A == 0.0) continue;
      double sq = sqrt(disc);
      double q = -0.5 * (B + (B >= 0.0 ? sq : -sq));
      double r1 = q / A, r2 = (q != 0.0) ? C / q : r1;
      double t[2] = {fmin(r1, r2), fmax(r1, r2)};
      for (int r = 0; r < 2; ++r) {
        double tc = t[r];
        if (!(tc >= 0.0 && tc <= 1.0)) continue;
        if (best >= 0.0 && tc >= best) continue;
        double x[3] = {a[0] + tc * d[0], a[1] + tc * d[1], a[2] + tc * d[2]};
        bool inside_other = false;   // the union's sign changes only outside the other spheres
        for (int j = 0; j < P.n_spheres && !inside_other; ++j)
          if (j != k && d_sphere_phi(P, j, x) < 0.0) inside_other = true;
        if (!inside_other) best = tc;
      }
    }
    if (best >= 0.0) return best;
  }
  double lo = 0.0, hi = 1.0;   // star (and the sphere rounding corner case): bisection
  const int iters = (P.ls_kind == NBM_LS_STAR) ? 60 : 200;
  for (int it = 0; it < iters; ++it) {
    double mid = 0.5 * (lo + hi);
    double x[3] = {a[0] + mid * d[0], a[1] + mid * d[1], a[2] + mid * d[2]};
    if (d_side(P, x) == sa) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

// ------------------------------------------------------------------ data
// manufactured solutions; returns false for the Gaussian source (no exact solution)
// diffusion coefficient of side s at x and its gradient (P:68 for the 4.1 fields)
__device__ double d_mu(const DevProblem& P, int s, const double x[3], double grad[3]) {
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, m;
  if (P.mu_kind == NBM_MU_PAPER41) {
    if (s == 0) {   // mu- = y^2 ln(x + 2) + 4
      const double lx = log(x[0] + 2.0);
      m = x[1] * x[1] * lx + 4.0;
      g0 = x[1] * x[1] / (x[0] + 2.0);
      g1 = 2.0 * x[1] * lx;
    } else {        // mu+ = e^{-z}
      m = exp(-x[2]);
      g2 = -m;
    }
  } else if (P.mu_kind == NBM_MU_LINEAR) {
    const double* c = P.mu_lin[s];
    m = c[0] + (c[1] * x[0] + c[2] * x[1]) + c[3] * x[2];
    g0 = c[1]; g1 = c[2]; g2 = c[3];
  } else {
    m = P.beta[s];
  }
  if (grad) { grad[0] = g0; grad[1] = g1; grad[2] = g2; }
  return m;
}

__device__ bool d_exact(const DevProblem& P, int s, const double x[3], double* u, double g[3]) {
  if (P.source == NBM_SRC_PAPER41) {   // u- = e^z, u+ = cos(x) sin(y)
    if (s == 0) {
      const double e = exp(x[2]);
      *u = e;
      g[0] = 0.0; g[1] = 0.0; g[2] = e;
    } else {
      const double cx = cos(x[0]), sx = sin(x[0]), cy = cos(x[1]), sy = sin(x[1]);
      *u = cx * sy;
      g[0] = -sx * sy; g[1] = cx * cy; g[2] = 0.0;
    }
    return true;
  }
  if (P.source == NBM_SRC_SINE3PI) {
    const double pi = 3.141592653589793;
    double sx = sin(pi * x[0]), sy = sin(pi * x[1]), sz = sin(pi * x[2]);
    double cx = cos(pi * x[0]), cy = cos(pi * x[1]), cz = cos(pi * x[2]);
    *u = sx * sy * sz;
    g[0] = pi * cx * sy * sz; g[1] = pi * sx * cy * sz; g[2] = pi * sx * sy * cz;
    return true;
  }
  if (P.source == NBM_SRC_PAIR) {
    if (s == 0) {
      double e = exp(x[0]), cy = cos(x[1]), sy = sin(x[1]);
      *u = e * cy * x[2];
      g[0] = e * cy * x[2]; g[1] = -e * sy * x[2]; g[2] = e * cy;
    } else {
      double t = x[0] + x[1] + x[2];
      double c = cos(t);
      *u = sin(t);
      g[0] = c; g[1] = c; g[2] = c;
    }
    return true;
  }
  return false;
}

__device__ double d_lap_exact(const DevProblem& P, int s, const double x[3]) {
  if (P.source == NBM_SRC_PAPER41) return s == 0 ? exp(x[2]) : -2.0 * cos(x[0]) * sin(x[1]);
  if (P.source == NBM_SRC_PAIR) return s == 0 ? 0.0 : -3.0 * sin(x[0] + x[1] + x[2]);
  const double pi = 3.141592653589793;   // SINE3PI
  return -3.0 * pi * pi * sin(pi * x[0]) * sin(pi * x[1]) * sin(pi * x[2]);
}

__device__ double d_source(const DevProblem& P, int s, const double x[3]) {
  double u, g[3];
  if (P.mu_kind != NBM_MU_CONST || P.source == NBM_SRC_PAPER41) {
    // f = k u - div(mu grad u) = k u - mu Lap u - grad mu . grad u
    if (!d_exact(P, s, x, &u, g)) return 0.0;
    double gm[3];
    const double m = d_mu(P, s, x, gm);
    return P.k[s] * u - m * d_lap_exact(P, s, x) - ((gm[0] * g[0] + gm[1] * g[1]) + gm[2] * g[2]);
  }
  if (P.source == NBM_SRC_SINE3PI) {
    d_exact(P, s, x, &u, g);
    const double pi = 3.141592653589793;
    return (P.k[s] + 3.0 * pi * pi * P.beta[s]) * u;   // -Lap u = 3 pi^2 u
  }
  if (P.source == NBM_SRC_PAIR) {
    d_exact(P, s, x, &u, g);
    return s == 0 ? P.k[0] * u : (P.k[1] + 3.0 * P.beta[1]) * u;   // u- harmonic (G12)
  }
  double s2 = P.charge_sigma * P.charge_sigma;
  double norm = pow(2.0 * 3.141592653589793 * s2, -1.5);
  double acc = 0.0;
  for (int k = 0; k < P.n_charges; ++k) {
    double dx = x[0] - P.charge_centers[k][0], dy = x[1] - P.charge_centers[k][1],
           dz = x[2] - P.charge_centers[k][2];
    acc += P.q[k] * norm * exp(-((dx * dx + dy * dy) + dz * dz) / (2.0 * s2));
  }
  return acc;
}

// ------------------------------------------------------------------ K2a classify
// Items 0..n-1: interior points -> class 0/1/2 (or skip); items n..n+nb-1: boundary
// points -> class 3/4 by side.  eval_only: items are evaluation points -> class 3/4.
__global__ void __launch_bounds__(kClsBlock) k_classify(
    const DevProblem* __restrict__ Pp, const float* __restrict__ pts, int64_t n,
    const float* __restrict__ bpts, int64_t nb, float hf, double d_minus, double d_plus,
    unsigned terms, int eval_only, uint8_t* __restrict__ cls, float* __restrict__ aux,
    int* __restrict__ blk_counts, int* __restrict__ err, uint8_t* __restrict__ mask_out,
    float* __restrict__ pcoef) {
  const DevProblem& P = *Pp;
  __shared__ int cnt[kNumCls];
  __shared__ float4 sph[kMaxSpheres];   // the sphere union's fp32 data, read by every side test
  if (threadIdx.x < kNumCls) cnt[threadIdx.x] = 0;
  if (P.ls_kind == NBM_LS_SPHERES && threadIdx.x < P.n_spheres)
    sph[threadIdx.x] = make_float4(P.centers_f[threadIdx.x][0], P.centers_f[threadIdx.x][1],
                                   P.centers_f[threadIdx.x][2], P.radii_f[threadIdx.x]);
  __syncthreads();
  auto side = [&](const double x[3]) {
    return P.ls_kind == NBM_LS_SPHERES ? d_side_spheres(P, sph, x) : d_side(P, x);
  };
  int64_t base = (int64_t)blockIdx.x * kClsItems;
  int64_t total = n + nb;
  for (int k = 0; k < kClsPerThread; ++k) {
    int64_t it = base + k * kClsBlock + threadIdx.x;
    if (it >= total) break;
    int c;
    float a = 0.0f;
    if (it < n && !eval_only) {
      const float* p = pts + 3 * it;
      double pd[3] = {p[0], p[1], p[2]};
      int s = side(pd);
      int mask = s;
      bool ood = false;
#pragma unroll 1
      for (int j = 1; j <= 6; ++j) {
        int dd = (j - 1) >> 1;
        float q[3] = {p[0], p[1], p[2]};
        q[dd] = (j & 1) ? __fadd_rn(p[dd], hf) : __fsub_rn(p[dd], hf);
        if (q[dd] < -1.0f || q[dd] > 1.0f) ood = true;
        double qd[3] = {q[0], q[1], q[2]};
        mask |= side(qd) << j;
      }
      if (mask_out) mask_out[it] = (uint8_t)mask;
      if (ood) {
        atomicOr(err, kErrOutOfDomain);
        c = kClsSkip;
      } else {
        c = (mask == 0) ? kClsUnxMinus : (mask == 0x7F) ? kClsUnxPlus : kClsCrossed;
        unsigned bit = (c == kClsUnxMinus) ? NBM_TERM_UNX_MINUS
                     : (c == kClsUnxPlus) ? NBM_TERM_UNX_PLUS : NBM_TERM_CROSSED;
        if (!(terms & bit)) c = kClsSkip;
        else if (c != kClsCrossed) {
          if (P.mu_kind == NBM_MU_CONST) {
            a = (float)(d_source(P, s, pd) / (s ? d_plus : d_minus));
          } else {   // variable mu: mu_s at the six face midpoints, d = k_s + sum mu_j / h^2
            const double h = hf, h2 = h * h;
            double mj[6], d = P.k[s];
#pragma unroll 1
            for (int j = 1; j <= 6; ++j) {
              const int dd = (j - 1) >> 1;
              double xf[3] = {pd[0], pd[1], pd[2]};
              xf[dd] = pd[dd] + ((j & 1) ? 0.5 * h : -0.5 * h);
              mj[j - 1] = d_mu(P, s, xf, nullptr);
              d += mj[j - 1] / h2;
            }
            for (int j = 0; j < 6; ++j) pcoef[6 * it + j] = (float)((-mj[j] / h2) / d);
            a = (float)(d_source(P, s, pd) / d);
          }
        }
      }
    } else {
      const float* p = eval_only ? pts + 3 * it : bpts + 3 * (it - n);
      double pd[3] = {p[0], p[1], p[2]};
      int s = side(pd);
      c = s ? kClsBndPlus : kClsBndMinus;
      if (!eval_only) {
        if (!(terms & NBM_TERM_BOUNDARY)) c = kClsSkip;
        double u, g[3];
        a = d_exact(P, s, pd, &u, g) ? (float)u : 0.0f;   // g = u_side (G10); 0 for config 3
      }
    }
    cls[it] = (uint8_t)c;
    aux[it] = a;
    atomicAdd(&cnt[c], 1);
  }
  __syncthreads();
  if (threadIdx.x < kNumCls) blk_counts[blockIdx.x * kNumCls + threadIdx.x] = cnt[threadIdx.x];
}

// K2s: exclusive scan of the block counts; class regions [0|1|2|3|4] in `list`.
// counts[0..5] = class totals, counts[6..11] = class starts.
__global__ void __launch_bounds__(1024) k_scan(const int* __restrict__ blk_counts, int nblk,
                                               int* __restrict__ blk_offsets, int* __restrict__ counts) {
  __shared__ int tot[kNumCls];
  __shared__ int wsum[32];
  __shared__ int carry;
  int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // pass 1: totals per class
  for (int c = 0; c < kNumCls; ++c) {
    int s = 0;
    for (int b = tid; b < nblk; b += 1024) s += blk_counts[b * kNumCls + c];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) wsum[wid] = s;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += wsum[w];
      tot[c] = t;
    }
    __syncthreads();
  }
  int start = 0;
  for (int c = 0; c < kNumCls; ++c) {
    if (tid == 0) { counts[c] = tot[c]; counts[kNumCls + c] = start; carry = start; }
    __syncthreads();
    for (int b0 = 0; b0 < nblk; b0 += 1024) {
      int b = b0 + tid;
      int v = b < nblk ? blk_counts[b * kNumCls + c] : 0;
      int x = v;   // inclusive warp scan
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wid] = x;
      __syncthreads();
      if (wid == 0) {
        int s = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, s, o);
          if (lane >= o) s += y;
        }
        wsum[lane] = s;
      }
      __syncthreads();
      int excl = carry + (wid ? wsum[wid - 1] : 0) + x - v;
      if (b < nblk) blk_offsets[b * kNumCls + c] = excl;
      __syncthreads();
      if (tid == 1023) carry = excl + v;
      __syncthreads();
    }
    start += tot[c];
  }
}

// K2c: stable scatter of item indices into the class regions.
__global__ void __launch_bounds__(kClsBlock) k_scatter(
    const uint8_t* __restrict__ cls, const float* __restrict__ aux, int64_t n, int64_t total,
    int eval_only, const int* __restrict__ blk_offsets, int* __restrict__ list,
    float* __restrict__ list_aux) {
  __shared__ int wcnt[kClsBlock / 32][kNumCls];
  __shared__ int run[kNumCls];
  int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < kNumCls) run[tid] = blk_offsets[blockIdx.x * kNumCls + tid];
  int64_t base = (int64_t)blockIdx.x * kClsItems;
  for (int k = 0; k < kClsPerThread; ++k) {
    int64_t it = base + k * kClsBlock + tid;
    int c = it < total ? cls[it] : -1;
    unsigned lt = (1u << lane) - 1u;
    int myrank = 0;
    __syncthreads();
    for (int cc = 0; cc < kNumCls; ++cc) {
      unsigned m = __ballot_sync(0xffffffffu, c == cc);
      if (c == cc) myrank = __popc(m & lt);
      if (lane == 0) wcnt[wid][cc] = __popc(m);
    }
    __syncthreads();
    if (c >= 0 && c != kClsSkip) {
      int off = run[c] + myrank;
      for (int w = 0; w < wid; ++w) off += wcnt[w][c];
      int idx = (int)((it < n || eval_only) ? it : it - n);
      list[off] = idx;
      list_aux[off] = aux[it];
    }
    __syncthreads();
    if (tid < kNumCls) {
      int s = 0;
      for (int w = 0; w < kClsBlock / 32; ++w) s += wcnt[w][tid];
      run[tid] += s;
    }
  }
}

cudaError_t launch_classify(const nbm_handle* h, const float* pts, int64_t n, const float* bpts,
                            int64_t nb, int64_t H, double d_minus, double d_plus, unsigned terms,
                            bool eval_only, cudaStream_t s, uint8_t* mask_out) {
  const Workspace& w = h->ws;
  int64_t total = n + nb;
  int nblk = (int)((total + kClsItems - 1) / kClsItems);
  if (nblk == 0) {
    return cudaMemsetAsync(w.counts, 0, 16 * sizeof(int), s);
  }
  float hf = (float)((double)H / kLattice);
  k_classify<<<nblk, kClsBlock, 0, s>>>(h->d_problem, pts, n, bpts, nb, hf, d_minus, d_plus, terms,
                                        eval_only ? 1 : 0, w.cls, w.aux_tmp, w.blk_counts, w.err,
                                        mask_out, w.pcoef);
  k_scan<<<1, 1024, 0, s>>>(w.blk_counts, nblk, w.blk_offsets, w.counts);
  k_scatter<<<nblk, kClsBlock, 0, s>>>(w.cls, w.aux_tmp, n, total, eval_only ? 1 : 0,
                                       w.blk_offsets, w.list, w.list_aux);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2x crossed rows
// One warp per crossed point, lane j < 7 owns stencil position j: the sharp-interface row in
// fp64 (G3, G6), normalised by the diagonal: chat_j = c_j / d (chat_0 = 1),
// rhs_hat = b / d, so the residual r = sum_j chat_j u_j - rhs_hat is M^-1 A u - M^-1 b
// (P:60).  Lane 0 sums the arm contributions in arm order.  Writes the 7 evaluation rows
// (position, network tag).
__global__ void __launch_bounds__(128) k_assemble_crossed(
    const DevProblem* __restrict__ Pp, const float* __restrict__ pts, float hf,
    const int* __restrict__ counts, const int* __restrict__ list, float* __restrict__ xrec,
    float* __restrict__ xrow_x, uint8_t* __restrict__ xrow_tag, int* __restrict__ err) {
  const DevProblem& P = *Pp;
  const int nx = counts[kClsCrossed];
  const int start = counts[kNumCls + kClsCrossed];
  const int lane = threadIdx.x & 31, j = lane;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ci < nx; ci += warps) {
    const float* p = pts + 3 * list[start + ci];
    const double pd[3] = {p[0], p[1], p[2]};
    const double h = hf, h2 = h * h;
    const int s = d_side(P, pd), so = 1 - s;
    const double bs = P.beta[s], bo = P.beta[so];
    // this lane's position
    float q[3] = {p[0], p[1], p[2]};
    const int dd = (j - 1) >> 1;
    if (j >= 1 && j <= 6) q[dd] = (j & 1) ? __fadd_rn(p[dd], hf) : __fsub_rn(p[dd], hf);
    double coef = 0.0, cc = 0.0, corr = 0.0;   // arm coefficient, centre contribution, rhs correction
    int tag = s;
    if (j >= 1 && j <= 6) {
      const double qd[3] = {q[0], q[1], q[2]};
      const int sq = d_side(P, qd);
      bool crossed = false;
      double th = 0.0, n[3] = {0, 0, 0}, xg[3];
      if (sq != s) {
        th = d_crossing_theta(P, pd, qd, s);
        if (th >= 1e-6 && th <= 1.0 - 1e-6) {   // snapping (G6)
          for (int c = 0; c < 3; ++c) xg[c] = pd[c] + th * (qd[c] - pd[c]);
          if (d_normal(P, xg, n)) crossed = true;
          else atomicOr(err, kErrDegenerate);
        }
      }
      if (!crossed) {                             // (a) uncrossed arm: mu_s at the face midpoint
        double mf = bs;
        if (P.mu_kind != NBM_MU_CONST) {
          double xf[3] = {pd[0], pd[1], pd[2]};
          xf[dd] = pd[dd] + ((j & 1) ? 0.5 * h : -0.5 * h);
          mf = d_mu(P, s, xf, nullptr);
        }
        coef = -mf / h2;
        cc = mf / h2;
      } else {                                    // (b) crossed arm, S:257 with rhs = f - corrections (G3)
        double mn = bs, mfar = bo;                // mu_near = mu_s(x_G), mu_far = mu_s'(x_G)
        if (P.mu_kind != NBM_MU_CONST) { mn = d_mu(P, s, xg, nullptr); mfar = d_mu(P, so, xg, nullptr); }
        const double muh = mn * mfar / (th * mfar + (1.0 - th) * mn);
        const double sg = (s == 0) ? 1.0 : -1.0;
        const double ne = (j & 1) ? n[dd] : -n[dd];   // n . e_j
        double um, up, gm[3], gp[3], alpha = 0.0, sigma = 0.0;
        if (d_exact(P, 0, xg, &um, gm)) {
          d_exact(P, 1, xg, &up, gp);
          alpha = up - um;
          const double dp = gp[0] * n[0] + gp[1] * n[1] + gp[2] * n[2];
          const double dm = gm[0] * n[0] + gm[1] * n[1] + gm[2] * n[2];
          sigma = d_mu(P, 1, xg, nullptr) * dp - d_mu(P, 0, xg, nullptr) * dm;
        }
        const double a = sg * alpha, ba = sg * sigma * ne;
        cc = muh / h2;
        coef = -muh / h2;
        tag = so;
        corr = muh * (a / h2 + (1.0 - th) * ba / (h * mfar));
      }
    }
    if (j < 7) {
      for (int c = 0; c < 3; ++c) xrow_x[(7 * (int64_t)ci + j) * 3 + c] = q[c];
      xrow_tag[7 * (int64_t)ci + j] = (uint8_t)tag;
    }
    // lane 0: d = k_s + sum_j cc_j, rhs = f_s(p) - sum_j corr_j (arm order), normalise
    double c0 = P.k[s], cs = 0.0, coefs[7];
    for (int a = 1; a <= 6; ++a) {
      c0 += __shfl_sync(0xffffffffu, cc, a);
      cs += __shfl_sync(0xffffffffu, corr, a);
      coefs[a] = __shfl_sync(0xffffffffu, coef, a);
    }
    if (lane == 0) {
      const double d = c0;
      const double rhs = d_source(P, s, pd) - cs;
      float* rec = xrec + 8 * (int64_t)ci;
      rec[0] = 1.0f;
      for (int a = 1; a < 7; ++a) rec[a] = (float)(coefs[a] / d);
      rec[7] = (float)(rhs / d);
    }
  }
}

// K2p: stable partition of the crossed rows by network (single CTA; ~1% of the work).
// counts[12 + net] = rows of that network.
__global__ void __launch_bounds__(1024) k_partition_xrows(const int* __restrict__ counts,
                                                          const uint8_t* __restrict__ tag,
                                                          int n_nets, int64_t xstride,
                                                          int* __restrict__ xlist,
                                                          int* __restrict__ counts_out) {
  __shared__ int wc[32][2];
  __shared__ int run[2];
  int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int nrows = 7 * counts[kClsCrossed];
  if (tid < 2) run[tid] = 0;
  for (int b0 = 0; b0 < nrows; b0 += 1024) {
    int r = b0 + tid;
    int net = r < nrows ? (n_nets == 1 ? 0 : (int)tag[r]) : -1;
    unsigned lt = (1u << lane) - 1u;
    unsigned m0 = __ballot_sync(0xffffffffu, net == 0);
    unsigned m1 = __ballot_sync(0xffffffffu, net == 1);
    __syncthreads();
    if (lane == 0) { wc[wid][0] = __popc(m0); wc[wid][1] = __popc(m1); }
    __syncthreads();
    if (net >= 0) {
      int off = run[net] + __popc((net ? m1 : m0) & lt);
      for (int w = 0; w < wid; ++w) off += wc[w][net];
      xlist[net * xstride + off] = r;
    }
    __syncthreads();
    if (tid < 2) {
      int s = 0;
      for (int w = 0; w < 32; ++w) s += wc[w][tid];
      run[tid] += s;
    }
  }
  __syncthreads();
  if (tid < 2) counts_out[12 + tid] = run[tid];
}

cudaError_t launch_assemble_crossed(const nbm_handle* h, const float* pts, int64_t n, int64_t H,
                                    cudaStream_t s) {
  const Workspace& w = h->ws;
  float hf = (float)((double)H / kLattice);
  int grid = 148 * 8;   // one warp per crossed point (grid-stride)
  k_assemble_crossed<<<grid, 128, 0, s>>>(h->d_problem, pts, hf, w.counts, w.list, w.xrec,
                                          w.xrow_x, w.xrow_tag, w.err);
  k_partition_xrows<<<1, 1024, 0, s>>>(w.counts, w.xrow_tag, h->arch.n_nets, 7 * w.xcap,
                                       w.xlist, w.counts);
  return cudaGetLastError();
}

// K2r: residual and cotangents of the crossed rows after the forward-only pass:
// r = sum_j chat_j u_j - rhs_hat (fp32), loss += r^2 / N, cot_j = (2/N) r chat_j.
__global__ void __launch_bounds__(1024) k_crossed_residual(const int* __restrict__ counts,
                                                           const float* __restrict__ xrec,
                                                           const float* __restrict__ xu,
                                                           float* __restrict__ xcot, float two_over_n,
                                                           double inv_n, double* __restrict__ lout) {
  __shared__ double ws[32];
  int nx = counts[kClsCrossed];
  double acc = 0.0;
  for (int ci = threadIdx.x; ci < nx; ci += 1024) {
    const float* rec = xrec + 8 * (int64_t)ci;
    const float* u = xu + 7 * (int64_t)ci;
    float r = u[0];
    for (int j = 1; j < 7; ++j) r = __fadd_rn(r, __fmul_rn(rec[j], u[j]));
    r = __fsub_rn(r, rec[7]);
    acc += (double)r * (double)r;
    float rc = __fmul_rn(two_over_n, r);
    xcot[7 * (int64_t)ci] = rc;
    for (int j = 1; j < 7; ++j) xcot[7 * (int64_t)ci + j] = __fmul_rn(rc, rec[j]);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += ws[w];
    *lout = t * inv_n;
  }
}

// ---- evaluation-grid error norms (Table 1) ----
// nodal points g = first .. first+n-1 of the (M+1)^3 grid over the box, x fastest:
// lo + (hi - lo) i / M in fp64, rounded to fp32
__global__ void k_nodal_points(int M, int64_t first, int64_t n, float* __restrict__ pts) {
  const int64_t m1 = (int64_t)M + 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = first + i;
    const int64_t idx[3] = {g % m1, (g / m1) % m1, g / (m1 * m1)};
#pragma unroll
    for (int c = 0; c < 3; ++c) pts[3 * i + c] = (float)(-1.0 + 2.0 * (double)idx[c] / (double)M);
  }
}

// e = u - u*_{side}: each block folds its points' sum e^2 and max |e| (fixed order: grid
// stride, warp butterfly, warps in order) into its slot; chunks run in stream order, so the
// result is deterministic
__global__ void __launch_bounds__(kErrThreads) k_error_accum(const DevProblem* __restrict__ Pp,
                                                             const float* __restrict__ pts,
                                                             const float* __restrict__ u, int64_t n,
                                                             double* __restrict__ slots, int init) {
  const DevProblem& P = *Pp;
  double sum = 0.0, mx = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double ue, g[3];
    d_exact(P, d_side_exact(P, x), x, &ue, g);
    const double e = (double)u[i] - ue;
    sum += e * e;
    mx = fmax(mx, fabs(e));
  }
  for (int o = 16; o; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double ws[2][kErrThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    ws[0][threadIdx.x >> 5] = sum;
    ws[1][threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, m = 0.0;
    for (int w = 0; w < kErrThreads / 32; ++w) {
      t += ws[0][w];
      m = fmax(m, ws[1][w]);
    }
    double* sl = slots + 2 * blockIdx.x;
    sl[0] = init ? t : sl[0] + t;
    sl[1] = init ? m : fmax(sl[1], m);
  }
}

__global__ void k_error_final(const double* __restrict__ slots, int nslots, double inv_total, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t = 0.0, m = 0.0;
  for (int b = 0; b < nslots; ++b) {
    t += slots[2 * b];
    m = fmax(m, slots[2 * b + 1]);
  }
  out[0] = sqrt(t * inv_total);
  out[1] = m;
}

cudaError_t launch_nodal_points(int M, int64_t first, int64_t n, float* pts, cudaStream_t s) {
  k_nodal_points<<<148 * 4, 256, 0, s>>>(M, first, n, pts);
  return cudaGetLastError();
}

cudaError_t launch_error_accum(const nbm_handle* h, const float* pts, const float* u, int64_t n, bool init,
                               cudaStream_t s) {
  k_error_accum<<<kErrBlocks, kErrThreads, 0, s>>>(h->d_problem, pts, u, n, h->ws.epart, init ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_error_final(const nbm_handle* h, int64_t total, double* out, cudaStream_t s) {
  k_error_final<<<1, 32, 0, s>>>(h->ws.epart, kErrBlocks, 1.0 / (double)total, out);
  return cudaGetLastError();
}

cudaError_t launch_crossed_residual(const nbm_handle* h, int64_t n_global, double weight, cudaStream_t s) {
  const Workspace& w = h->ws;   // weight: the resolution level's w_l, 1 for one level
  k_crossed_residual<<<1, 1024, 0, s>>>(w.counts, w.xrec, w.xrow_u, w.xrow_cot,
                                        (float)(2.0 * weight / (double)n_global), weight / (double)n_global,
                                        w.lpart + w.grid_mlp);
  return cudaGetLastError();
}

}  // namespace nbm
