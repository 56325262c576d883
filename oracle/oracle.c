/*
 * oracle.c -- plain fp64 CPU oracle of the NBM loss + gradient hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Each function cites the passage
 * it follows: P:n = PAPER.md line n, S:n = SPEC.md line n, Gk = the reading
 * k listed in DESIGN.md ("Readings of the paper").
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fopenmp -fPIC -shared
 * (no fast-math; no FMA contraction, so every fp op rounds once as written).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  Sampling is           */
/* "random collocation points"; the generator is our choice (G9) */
/* ------------------------------------------------------------------------ */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    if (round < 9) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_block(uint64_t seed, uint64_t counter, uint32_t word2, uint32_t stream,
                         uint32_t out[4]) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {(uint32_t)counter, (uint32_t)(counter >> 32), word2, stream};
  orc_philox(ctr, key, out);
}

static uint64_t mulhi64(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
}

/* S:339 UniformRandom: interior points uniform in the shrunken cube
 * [-1+h, 1-h]^3 (so all arms stay in the domain), boundary points
 * uniform on the 6 faces.  Reading G9: coordinates on the 2^-24 lattice. */
void orc_sample(int kind, uint64_t seed, uint64_t step, int64_t first, int64_t n,
                int64_t H, float* pts) {
  const int64_t L = (int64_t)1 << 24;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t gi = (uint64_t)(first + i);
    uint32_t w[8];
    philox_block(seed, 2 * gi + 0, (uint32_t)step, (uint32_t)kind, w);
    philox_block(seed, 2 * gi + 1, (uint32_t)step, (uint32_t)kind, w + 4);
    float* x = pts + 3 * i;
    if (kind == 0) {
      uint64_t M = (uint64_t)(2 * (L - H));
      for (int c = 0; c < 3; ++c) {
        uint64_t W = (uint64_t)w[2 * c] | ((uint64_t)w[2 * c + 1] << 32);
        int64_t m = (int64_t)mulhi64(W, M + 1);         /* uniform integer in [0, M] */
        x[c] = (float)(m - (L - H)) * 0x1p-24f;          /* exact */
      }
    } else {
      uint32_t f = (uint32_t)(((uint64_t)w[6] * 6u) >> 32); /* face in [0,5] */
      int axis = (int)(f >> 1);
      float sgn = (f & 1u) ? -1.0f : 1.0f;
      int slot = 0;
      for (int c = 0; c < 3; ++c) {
        if (c == axis) { x[c] = sgn; continue; }
        uint64_t W = (uint64_t)w[2 * slot] | ((uint64_t)w[2 * slot + 1] << 32);
        int64_t m = (int64_t)mulhi64(W, (uint64_t)(2 * L) + 1);  /* [0, 2^25] */
        x[c] = (float)(m - L) * 0x1p-24f;
        ++slot;
      }
    }
  }
}

/* ------------------------------------------------------------------------ */
/* geometry: level set phi, side, crossings, normals   */
/* ------------------------------------------------------------------------ */
static double sphere_phi(const orc_problem* pb, int k, const double x[3]) {
  const double* c = pb->centers + 3 * k;
  double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
  return sqrt((dx * dx + dy * dy) + dz * dz) - pb->radii[k];
}

/* star: r - r0 - amp * sin(m th) cos(n ph), th polar angle from +z,
 * ph = atan2(y, x) (G13).  sin(m th) = sin th * U_{m-1}(cos th) and
 * cos(n ph) = T_n(cos ph), Chebyshev recurrences, so only + - * / sqrt. */
static double star_phi(const orc_problem* pb, const double x[3]) {
  double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
  double r = sqrt(rho * rho + x[2] * x[2]);
  if (r == 0.0) return -pb->star_r0;
  if (rho == 0.0) return r - pb->star_r0;
  double ct = x[2] / r, st = rho / r, cp = x[0] / rho;
  double u0 = 1.0, u1 = 2.0 * ct;                 /* U_0, U_1 */
  double um;                                      /* U_{m-1} */
  if (pb->star_m <= 1) um = 1.0;
  else {
    for (int k = 2; k < pb->star_m; ++k) { double u2 = 2.0 * ct * u1 - u0; u0 = u1; u1 = u2; }
    um = u1;
  }
  double t0 = 1.0, t1 = cp;                       /* T_0, T_1 */
  double tn;
  if (pb->star_n == 0) tn = 1.0;
  else {
    for (int k = 1; k < pb->star_n; ++k) { double t2 = 2.0 * cp * t1 - t0; t0 = t1; t1 = t2; }
    tn = t1;
  }
  double ang = (st * um) * tn;
  return (r - pb->star_r0) - pb->star_amp * ang;
}

/* Sampled level set ("trilinear interpolation of nodal values", "a separate coarse
 * mesh encapsulates a level-set function"): nodes x_i = -1 + i hc, hc = 2/Nc, values x-fastest.
 * Cell index and local coordinate per axis from s = (x + 1) Nc/2 (clamped to the cube), then
 * seven linear interpolations a + t (b - a): along x, then y, then z. */
static double grid_lerp(double a, double b, double t) { return a + t * (b - a); }
static double grid_phi(const orc_problem* pb, const double x[3]) {
  const int nc = pb->grid_n, n1 = nc + 1;
  const double half = 0.5 * (double)nc;
  int i[3];
  double t[3];
  for (int d = 0; d < 3; ++d) {
    double sd = (x[d] + 1.0) * half;
    if (sd < 0.0) sd = 0.0;
    if (sd > (double)nc) sd = (double)nc;
    int id = (int)floor(sd);
    if (id > nc - 1) id = nc - 1;
    i[d] = id;
    t[d] = sd - (double)id;
  }
#define GV(a, b, c) pb->grid_phi[(int64_t)(i[0] + (a)) + (int64_t)n1 * ((int64_t)(i[1] + (b)) + (int64_t)n1 * (i[2] + (c)))]
  double c00 = grid_lerp(GV(0, 0, 0), GV(1, 0, 0), t[0]);
  double c10 = grid_lerp(GV(0, 1, 0), GV(1, 1, 0), t[0]);
  double c01 = grid_lerp(GV(0, 0, 1), GV(1, 0, 1), t[0]);
  double c11 = grid_lerp(GV(0, 1, 1), GV(1, 1, 1), t[0]);
#undef GV
  double c0 = grid_lerp(c00, c10, t[1]), c1 = grid_lerp(c01, c11, t[1]);
  return grid_lerp(c0, c1, t[2]);
}

double orc_phi(const orc_problem* pb, const double x[3]) {
  switch (pb->ls_kind) {
    case ORC_LS_NONE: return -1.0;                /* everything is Omega- (config 1) */
    case ORC_LS_SPHERES: {
      double m = sphere_phi(pb, 0, x);
      for (int k = 1; k < pb->n_spheres; ++k) { double v = sphere_phi(pb, k, x); if (v < m) m = v; }
      return m;
    }
    case ORC_LS_STAR: return star_phi(pb, x);
    case ORC_LS_PLANE:
      return ((pb->plane_n[0] * x[0] + pb->plane_n[1] * x[1]) + pb->plane_n[2] * x[2]) - pb->plane_c;
    case ORC_LS_GRID: return grid_phi(pb, x);
  }
  return -1.0;
}

/* Omega- iff phi <= 0 (tie rule G5) */
int orc_side(const orc_problem* pb, const double x[3]) { return orc_phi(pb, x) <= 0.0 ? 0 : 1; }

int orc_normal(const orc_problem* pb, const double x[3], double nrm[3]) {
  double g[3];
  if (pb->ls_kind == ORC_LS_PLANE) {
    g[0] = pb->plane_n[0]; g[1] = pb->plane_n[1]; g[2] = pb->plane_n[2];
  } else if (pb->ls_kind == ORC_LS_SPHERES) {
    /* closed-form normal of the sphere attaining the min (lowest index on ties), G7 */
    int best = 0; double m = sphere_phi(pb, 0, x);
    for (int k = 1; k < pb->n_spheres; ++k) { double v = sphere_phi(pb, k, x); if (v < m) { m = v; best = k; } }
    const double* c = pb->centers + 3 * best;
    g[0] = x[0] - c[0]; g[1] = x[1] - c[1]; g[2] = x[2] - c[2];
  } else {
    /* central differences, step 1e-5 (Analytic) or hc/2 = 1/Nc of the interpolant (Sampled) */
    const double e = pb->ls_kind == ORC_LS_GRID ? 1.0 / (double)pb->grid_n : 1e-5;
    for (int d = 0; d < 3; ++d) {
      double xp[3] = {x[0], x[1], x[2]}, xm[3] = {x[0], x[1], x[2]};
      xp[d] += e; xm[d] -= e;
      g[d] = (orc_phi(pb, xp) - orc_phi(pb, xm)) / (2.0 * e);
    }
  }
  double nn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  if (!(nn >= 1e-12)) return -2;                  /* DegenerateGradient */
  nrm[0] = g[0] / nn; nrm[1] = g[1] / nn; nrm[2] = g[2] / nn;
  return 0;
}

int orc_crossing_bisect(const orc_problem* pb, const double a[3], const double b[3], double* theta) {
  int sa = orc_side(pb, a);
  if (sa == orc_side(pb, b)) return 0;
  double lo = 0.0, hi = 1.0;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    double x[3] = {a[0] + mid * (b[0] - a[0]), a[1] + mid * (b[1] - a[1]), a[2] + mid * (b[2] - a[2])};
    if (orc_side(pb, x) == sa) lo = mid; else hi = mid;
  }
  *theta = 0.5 * (lo + hi);
  return 1;
}

/* roots of |a + t d - c|^2 = R^2 (numerically stable quadratic) */
static int sphere_roots(const orc_problem* pb, int k, const double a[3], const double d[3], double t[2]) {
  const double* c = pb->centers + 3 * k;
  double ac[3] = {a[0] - c[0], a[1] - c[1], a[2] - c[2]};
  double A = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  double B = 2.0 * (ac[0] * d[0] + ac[1] * d[1] + ac[2] * d[2]);
  double C = (ac[0] * ac[0] + ac[1] * ac[1] + ac[2] * ac[2]) - pb->radii[k] * pb->radii[k];
  double disc = B * B - 4.0 * A * C;
  if (disc < 0.0 || A == 0.0) return 0;
  double s = sqrt(disc);
  double q = -0.5 * (B + (B >= 0.0 ? s : -s));
  double r1 = q / A, r2 = (q != 0.0) ? C / q : r1;
  t[0] = r1 < r2 ? r1 : r2; t[1] = r1 < r2 ? r2 : r1;
  return 2;
}

/* Crossing of Gamma on the arm a->b ("calculating interface-cell
 * crossings" P:52).  Root nearest to a (G8): closed form for spheres (the
 * first per-sphere root where the union sign changes) and planes, fp64
 * bisection for the star. */
int orc_crossing(const orc_problem* pb, const double a[3], const double b[3],
                 double* theta, double xg[3], double nrm[3]) {
  int sa = orc_side(pb, a), sb = orc_side(pb, b);
  if (sa == sb) return 0;
  double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double th = -1.0;
  if (pb->ls_kind == ORC_LS_SPHERES) {
    for (int k = 0; k < pb->n_spheres; ++k) {
      double t[2];
      if (!sphere_roots(pb, k, a, d, t)) continue;
      for (int r = 0; r < 2; ++r) {
        double tc = t[r];
        if (!(tc >= 0.0 && tc <= 1.0)) continue;
        if (th >= 0.0 && tc >= th) continue;
        double x[3] = {a[0] + tc * d[0], a[1] + tc * d[1], a[2] + tc * d[2]};
        int inside_other = 0;                     /* the union changes sign only if no other sphere contains x */
        for (int j = 0; j < pb->n_spheres; ++j)
          if (j != k && sphere_phi(pb, j, x) < 0.0) { inside_other = 1; break; }
        if (!inside_other) th = tc;
      }
    }
    if (th < 0.0) orc_crossing_bisect(pb, a, b, &th);   /* rounding corner case */
  } else if (pb->ls_kind == ORC_LS_PLANE) {
    double nd = pb->plane_n[0] * d[0] + pb->plane_n[1] * d[1] + pb->plane_n[2] * d[2];
    th = -orc_phi(pb, a) / nd;
  } else if (pb->ls_kind == ORC_LS_GRID) {
    /* S:125 Sampled: root of the linear interpolant between phi(a) and phi(b) */
    double pa = orc_phi(pb, a), pbv = orc_phi(pb, b);
    th = pa / (pa - pbv);
  } else {
    double lo = 0.0, hi = 1.0;
    for (int it = 0; it < 60; ++it) {
      double mid = 0.5 * (lo + hi);
      double x[3] = {a[0] + mid * d[0], a[1] + mid * d[1], a[2] + mid * d[2]};
      if (orc_side(pb, x) == sa) lo = mid; else hi = mid;
    }
    th = 0.5 * (lo + hi);
  }
  *theta = th;
  xg[0] = a[0] + th * d[0]; xg[1] = a[1] + th * d[1]; xg[2] = a[2] + th * d[2];
  return orc_normal(pb, xg, nrm) < 0 ? -2 : 1;
}

/* diffusion coefficient of side s at x and its gradient (P:68 for the 4.1 fields) */
double orc_mu(const orc_problem* pb, int s, const double x[3], double grad[3]) {
  double g0 = 0.0, g1 = 0.0, g2 = 0.0, m;
  if (pb->mu_kind == ORC_MU_PAPER41) {
    if (s == 0) {                                  /* mu- = y^2 ln(x + 2) + 4 */
      double lx = log(x[0] + 2.0);
      m = x[1] * x[1] * lx + 4.0;
      g0 = x[1] * x[1] / (x[0] + 2.0);
      g1 = 2.0 * x[1] * lx;
    } else {                                       /* mu+ = e^{-z} */
      m = exp(-x[2]);
      g2 = -m;
    }
  } else if (pb->mu_kind == ORC_MU_LINEAR) {
    const double* c = pb->mu_lin + 4 * s;
    m = c[0] + (c[1] * x[0] + c[2] * x[1]) + c[3] * x[2];
    g0 = c[1]; g1 = c[2]; g2 = c[3];
  } else {
    m = pb->beta[s];
  }
  if (grad) { grad[0] = g0; grad[1] = g1; grad[2] = g2; }
  return m;
}

/* ------------------------------------------------------------------------ */
/* problem data: k u - div(beta grad u) = f, [u] = alpha, [beta d_n u] =     */
/* sigma; manufactured families of BASELINE.json configs           */
/* ------------------------------------------------------------------------ */
int orc_exact(const orc_problem* pb, int side, const double x[3], double* u, double g[3]) {
  switch (pb->source) {
    case ORC_SRC_SINE3PI: {                        /* config 1: u = sin(pi x) sin(pi y) sin(pi z) */
      double sx = sin(M_PI * x[0]), sy = sin(M_PI * x[1]), sz = sin(M_PI * x[2]);
      double cx = cos(M_PI * x[0]), cy = cos(M_PI * x[1]), cz = cos(M_PI * x[2]);
      *u = sx * sy * sz;
      if (g) { g[0] = M_PI * cx * sy * sz; g[1] = M_PI * sx * cy * sz; g[2] = M_PI * sx * sy * cz; }
      return 0;
    }
    case ORC_SRC_PAIR:                             /* configs 2,4,5: u- = e^x cos(y) z, u+ = sin(x+y+z) */
      if (side == 0) {
        double e = exp(x[0]), cy = cos(x[1]), sy = sin(x[1]);
        *u = e * cy * x[2];
        if (g) { g[0] = e * cy * x[2]; g[1] = -e * sy * x[2]; g[2] = e * cy; }
      } else {
        double s = x[0] + x[1] + x[2];
        *u = sin(s);
        if (g) { double c = cos(s); g[0] = c; g[1] = c; g[2] = c; }
      }
      return 0;
    case ORC_SRC_PAPER41:                          /* u- = e^z, u+ = cos(x) sin(y) */
      if (side == 0) {
        double e = exp(x[2]);
        *u = e;
        if (g) { g[0] = 0.0; g[1] = 0.0; g[2] = e; }
      } else {
        double cx = cos(x[0]), sx = sin(x[0]), cy = cos(x[1]), sy = sin(x[1]);
        *u = cx * sy;
        if (g) { g[0] = -sx * sy; g[1] = cx * cy; g[2] = 0.0; }
      }
      return 0;
    case ORC_SRC_POLY2: {                          /* test family: c + g.x + x^T A x per side */
      const double* p = pb->poly + 10 * side;
      double A[3][3] = {{p[4], p[5], p[6]}, {p[5], p[7], p[8]}, {p[6], p[8], p[9]}};
      double Ax[3];
      for (int i = 0; i < 3; ++i) Ax[i] = A[i][0] * x[0] + A[i][1] * x[1] + A[i][2] * x[2];
      *u = p[0] + (p[1] * x[0] + p[2] * x[1] + p[3] * x[2]) + (x[0] * Ax[0] + x[1] * Ax[1] + x[2] * Ax[2]);
      if (g) for (int i = 0; i < 3; ++i) g[i] = p[1 + i] + 2.0 * Ax[i];
      return 0;
    }
  }
  return -1;                                       /* no exact solution (config 3) */
}

/* Laplacian of the manufactured solutions */
static double lap_exact(const orc_problem* pb, int side, const double x[3]) {
  double u;
  switch (pb->source) {
    case ORC_SRC_SINE3PI: orc_exact(pb, side, x, &u, NULL); return -3.0 * M_PI * M_PI * u;
    case ORC_SRC_PAIR: return side == 0 ? 0.0 : -3.0 * sin(x[0] + x[1] + x[2]);
    case ORC_SRC_POLY2: { const double* p = pb->poly + 10 * side; return 2.0 * (p[4] + p[7] + p[9]); }
    case ORC_SRC_PAPER41: return side == 0 ? exp(x[2]) : -2.0 * cos(x[0]) * sin(x[1]);
  }
  return 0.0;
}

double orc_f(const orc_problem* pb, int side, const double x[3]) {
  double ks = pb->k[side], bs = pb->beta[side], u;
  if (pb->mu_kind != ORC_MU_CONST || pb->source == ORC_SRC_PAPER41) {
    /* f = k u - div(mu grad u) = k u - mu Lap u - grad mu . grad u */
    double gu[3], gm[3];
    if (orc_exact(pb, side, x, &u, gu) < 0) return 0.0;
    double m = orc_mu(pb, side, x, gm);
    return ks * u - m * lap_exact(pb, side, x) - ((gm[0] * gu[0] + gm[1] * gu[1]) + gm[2] * gu[2]);
  }
  switch (pb->source) {
    case ORC_SRC_SINE3PI:                          /* -Lap u = 3 pi^2 u */
      orc_exact(pb, side, x, &u, NULL);
      return (ks + 3.0 * M_PI * M_PI * bs) * u;
    case ORC_SRC_PAIR:
      orc_exact(pb, side, x, &u, NULL);
      if (side == 0) return ks * u;                /* u- harmonic (G12) */
      return (ks + 3.0 * bs) * u;                  /* -Lap sin(x+y+z) = 3 sin(x+y+z) */
    case ORC_SRC_GAUSS: {                          /* sum_k q_k N(x; c_k, s^2 I) (G13) */
      double s2 = pb->charge_sigma * pb->charge_sigma;
      double norm = pow(2.0 * M_PI * s2, -1.5);
      double acc = 0.0;
      for (int k = 0; k < pb->n_charges; ++k) {
        const double* c = pb->charge_centers + 3 * k;
        double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
        acc += pb->q[k] * norm * exp(-((dx * dx + dy * dy) + dz * dz) / (2.0 * s2));
      }
      return acc;
    }
    case ORC_SRC_POLY2: {
      const double* p = pb->poly + 10 * side;
      orc_exact(pb, side, x, &u, NULL);
      return ks * u - bs * 2.0 * (p[4] + p[7] + p[9]);
    }
  }
  return 0.0;
}

/* alpha = [u] = u+ - u- on Gamma */
double orc_alpha(const orc_problem* pb, const double x[3]) {
  double um, up;
  if (orc_exact(pb, 0, x, &um, NULL) < 0) return 0.0;
  orc_exact(pb, 1, x, &up, NULL);
  return up - um;
}

/* sigma = [beta d_n u] = beta+ grad u+ . n - beta- grad u- . n */
double orc_sigma(const orc_problem* pb, const double x[3], const double n[3]) {
  double um, up, gm[3], gp[3];
  if (orc_exact(pb, 0, x, &um, gm) < 0) return 0.0;
  orc_exact(pb, 1, x, &up, gp);
  double dp = gp[0] * n[0] + gp[1] * n[1] + gp[2] * n[2];
  double dm = gm[0] * n[0] + gm[1] * n[1] + gm[2] * n[2];
  return orc_mu(pb, 1, x, NULL) * dp - orc_mu(pb, 0, x, NULL) * dm;
}

/* Dirichlet data: the manufactured u of the side containing x (G10) */
double orc_g(const orc_problem* pb, const double x[3]) {
  double u;
  if (orc_exact(pb, orc_side(pb, x), x, &u, NULL) < 0) return 0.0;
  return u;
}

/* ------------------------------------------------------------------------ */
/* NBM kernel: implicit cell + sharp-interface row */
/* ------------------------------------------------------------------------ */
static const int ARM_DIM[7] = {0, 0, 0, 1, 1, 2, 2};
static const int ARM_SGN[7] = {0, +1, -1, +1, -1, +1, -1};

int orc_assemble(const orc_problem* pb, const float p[3], float hf, int sign_mutation, orc_row* row) {
  memset(row, 0, sizeof(*row));
  double pd[3] = {p[0], p[1], p[2]};
  double h = hf, h2 = h * h;
  int s = orc_side(pb, pd), so = 1 - s;
  row->side = s;
  row->mask = s;
  for (int c = 0; c < 3; ++c) row->pos[0][c] = p[c];
  row->tag[0] = s;
  double c0 = pb->k[s];                              /* k_s u_s(p) term */
  double corr = 0.0;
  double bs = pb->beta[s], bo = pb->beta[so];
  for (int j = 1; j <= 6; ++j) {
    int dd = ARM_DIM[j];
    float q[3] = {p[0], p[1], p[2]};
    q[dd] = (float)((double)p[dd] + ARM_SGN[j] * h);  /* fp32 arm, exact on the lattice */
    if (q[dd] < -1.0f || q[dd] > 1.0f) return -1;     /* OutOfDomain */
    for (int c = 0; c < 3; ++c) row->pos[j][c] = q[c];
    double qd[3] = {q[0], q[1], q[2]};
    int sq = orc_side(pb, qd);
    row->mask |= sq << j;
    /* mu_s at the arm's face midpoint p + (h/2) e (beta_s when mu is constant) */
    double xf[3] = {pd[0], pd[1], pd[2]};
    xf[dd] = pd[dd] + ARM_SGN[j] * 0.5 * h;
    const double mf = pb->mu_kind == ORC_MU_CONST ? bs : orc_mu(pb, s, xf, NULL);
    if (sq == s) {                                     /* (a) uncrossed arm */
      row->coef[j] = -mf / h2; c0 += mf / h2; row->tag[j] = s;
      continue;
    }
    double th, xg[3], n[3];
    int rc = orc_crossing(pb, pd, qd, &th, xg, n);
    if (rc < 0) return -2;
    row->theta[j] = th;
    if (th < 1e-6 || th > 1.0 - 1e-6) {                /* theta snapping (G6) */
      row->coef[j] = -mf / h2; c0 += mf / h2; row->tag[j] = s; row->n_snapped++;
      continue;
    }
    /* (b) crossed arm, S:257 with the sign reading G3; mu_near = mu_s(x_G), mu_far = mu_s'(x_G) */
    double mn = bs, mfar = bo;
    if (pb->mu_kind != ORC_MU_CONST) { mn = orc_mu(pb, s, xg, NULL); mfar = orc_mu(pb, so, xg, NULL); }
    double muh = mn * mfar / (th * mfar + (1.0 - th) * mn);
    double sg = (s == 0) ? 1.0 : -1.0;
    double e[3] = {0, 0, 0}; e[dd] = ARM_SGN[j];
    double a = sg * orc_alpha(pb, xg);
    double ba = sg * orc_sigma(pb, xg, n) * (n[0] * e[0] + n[1] * e[1] + n[2] * e[2]);
    c0 += muh / h2;
    row->coef[j] = -muh / h2;
    row->tag[j] = so;
    corr += muh * (a / h2 + (1.0 - th) * ba / (h * mfar));
    row->n_crossed_arms++;
  }
  row->coef[0] = c0;
  row->d = c0;
  row->f = orc_f(pb, s, pd);
  row->corr = corr;
  row->rhs = sign_mutation ? row->f + corr : row->f - corr;
  row->crossed = (row->mask != 0 && row->mask != 0x7F);
  return 0;
}

int orc_classify(const orc_problem* pb, const float* pts, int64_t n, float h,
                 uint8_t* mask, uint8_t* cls) {
  for (int64_t i = 0; i < n; ++i) {
    const float* p = pts + 3 * i;
    double pd[3] = {p[0], p[1], p[2]};
    int s = orc_side(pb, pd), m = s;
    for (int j = 1; j <= 6; ++j) {
      int dd = ARM_DIM[j];
      float q[3] = {p[0], p[1], p[2]};
      q[dd] = (float)((double)p[dd] + ARM_SGN[j] * (double)h);
      if (q[dd] < -1.0f || q[dd] > 1.0f) return -1;
      double qd[3] = {q[0], q[1], q[2]};
      m |= orc_side(pb, qd) << j;
    }
    mask[i] = (uint8_t)m;
    cls[i] = (uint8_t)((m == 0) ? 0 : (m == 0x7F) ? 1 : 2);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* surrogate: MLP per side, hand-written reverse accumulation     */
/* ------------------------------------------------------------------------ */
int64_t orc_param_count(const orc_arch* a) {
  int64_t p = 0;
  for (int l = 1; l < a->n_layers; ++l) p += (int64_t)a->sizes[l] * a->sizes[l - 1] + a->sizes[l];
  return p * a->n_nets;
}

/* G11: Glorot-uniform +-sqrt(6/(fan_in+fan_out)), zero biases; Philox stream 2.  Sine nets
 * (S:175): +-sqrt(6/fan_in). */
void orc_init_params(const orc_arch* a, uint64_t seed, float* theta) {
  uint64_t e = 0;
  int64_t off = 0;
  for (int net = 0; net < a->n_nets; ++net)
    for (int l = 1; l < a->n_layers; ++l) {
      int fi = a->sizes[l - 1], fo = a->sizes[l];
      float amp = a->act == ORC_ACT_SINE ? sqrtf(6.0f / (float)fi) : sqrtf(6.0f / (float)(fi + fo));
      for (int64_t k = 0; k < (int64_t)fi * fo; ++k, ++e) {
        uint32_t w[4];
        philox_block(seed, e >> 2, 0u, 2u, w);
        float u = (float)(w[e & 3] >> 8) * 0x1p-24f;
        theta[off++] = amp * (2.0f * u - 1.0f);
      }
      for (int k = 0; k < fo; ++k) theta[off++] = 0.0f;
    }
}

static inline double rnd(int mode, double x) { return mode == ORC_MODE_F64 ? x : (double)(float)x; }
/* round-to-nearest-even to bf16 (G16) */
static inline double rbf16(double xd) {
  float x = (float)xd;
  uint32_t u; memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return x;
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  float y; memcpy(&y, &u, 4);
  return y;
}

static inline double act_f(int act, double z) {
  switch (act) {
    case ORC_ACT_TANH: return tanh(z);
    case ORC_ACT_SILU: return z / (1.0 + exp(-z));
    default: return sin(z);
  }
}
static inline double act_d(int act, double z, double h) {
  switch (act) {
    case ORC_ACT_TANH: return 1.0 - h * h;
    case ORC_ACT_SILU: { double sg = 1.0 / (1.0 + exp(-z)); return sg * (1.0 + z * (1.0 - sg)); }
    default: return cos(z);
  }
}

#define MAXW 1024
#define MAXL 16
typedef struct { double z[MAXL][MAXW]; double h[MAXL][MAXW]; } tape_t;

static int64_t net_offset(const orc_arch* a, int net) {
  orc_arch one = *a; one.n_nets = 1;
  return net * orc_param_count(&one);
}

/* forward pass with tape; layer l (1..L-1): z_l = W_l h_{l-1} + b_l, hidden h_l = act(z_l),
 * output u = z_{L-1}.  bf16 mode rounds the operands of hidden x hidden
 * products (tensor-core GEMMs) to bf16 and keeps layer 1 / output in fp32 (G16). */
static double fwd_tape(const orc_arch* a, const double* theta, int net, const double x[3],
                       int mode, tape_t* T) {
  const double* P = theta + net_offset(a, net);
  int L = a->n_layers;
  for (int c = 0; c < 3; ++c) T->h[0][c] = rnd(mode, x[c]);
  for (int l = 1; l < L; ++l) {
    int fi = a->sizes[l - 1], fo = a->sizes[l];
    const double* W = P; const double* b = P + (int64_t)fi * fo;
    int gemm = (mode == ORC_MODE_BF16) && l >= 2 && l <= L - 2;
    for (int o = 0; o < fo; ++o) {
      double acc = 0.0;
      for (int i = 0; i < fi; ++i) {
        double w = W[(int64_t)o * fi + i], hv = T->h[l - 1][i];
        if (gemm) { w = rbf16(w); hv = rbf16(hv); }
        acc = rnd(mode, acc + rnd(mode, w * hv));
      }
      double z = rnd(mode, acc + (double)b[o]);
      T->z[l][o] = z;
      T->h[l][o] = (l < L - 1) ? rnd(mode, act_f(a->act, z)) : z;
    }
    P += (int64_t)fi * fo + fo;
  }
  return T->h[L - 1][0];
}

double orc_forward(const orc_arch* a, const double* theta, int net, const double x[3], int mode) {
  tape_t* T = (tape_t*)malloc(sizeof(tape_t));
  double u = fwd_tape(a, theta, net, x, mode, T);
  free(T);
  return u;
}

static void bwd_tape(const orc_arch* a, const double* theta, int net, double cot, int mode,
                     const tape_t* T, double* grad) {
  int L = a->n_layers;
  int64_t off[MAXL];
  int64_t o0 = net_offset(a, net);
  for (int l = 1; l < L; ++l) { off[l] = o0; o0 += (int64_t)a->sizes[l] * a->sizes[l - 1] + a->sizes[l]; }
  static __thread double dl[MAXW], dn[MAXW];
  dl[0] = rnd(mode, cot);                              /* delta_{L-1} = u-bar */
  for (int l = L - 1; l >= 1; --l) {
    int fi = a->sizes[l - 1], fo = a->sizes[l];
    const double* W = theta + off[l];
    double* gW = grad + off[l];
    double* gb = gW + (int64_t)fi * fo;
    int gemm = (mode == ORC_MODE_BF16) && l >= 2 && l <= L - 2;
    /* bf16 path (G16): the bias gradients of hidden layers 1..NH-1 and the layer-1 weight
     * gradient are tensor-core reductions of the bf16 delta; layer-1 inputs enter as a
     * two-term bf16 split x = bf16(x) + bf16(x - bf16(x)). */
    int tail = (mode == ORC_MODE_BF16) && l <= L - 3;
    for (int o = 0; o < fo; ++o) {                     /* dW_l += delta_l h_{l-1}^T, db_l += delta_l */
      double dv = (gemm || (tail && l == 1)) ? rbf16(dl[o]) : dl[o];
      for (int i = 0; i < fi; ++i) {
        double hv = gemm ? rbf16(T->h[l - 1][i]) : T->h[l - 1][i];
        if (tail && l == 1) { double hi = rbf16(hv); hv = hi + rbf16(hv - hi); }
        gW[(int64_t)o * fi + i] += rnd(mode, dv * hv);
      }
      gb[o] += tail ? rbf16(dl[o]) : dl[o];
    }
    if (l == 1) break;
    for (int i = 0; i < fi; ++i) {                     /* delta_{l-1} = (W_l^T delta_l) . act'(z_{l-1}) */
      double acc = 0.0;
      for (int o = 0; o < fo; ++o) {
        double w = W[(int64_t)o * fi + i], dv = dl[o];
        if (gemm) { w = rbf16(w); dv = rbf16(dv); }
        acc = rnd(mode, acc + rnd(mode, w * dv));
      }
      /* bf16 path (G16): tanh' of hidden layers 1..NH-1 from the bf16 operand copy of h;
       * SiLU' of hidden layers 2..NH-1 stored (rounded) in bf16; others exact */
      double hv = T->h[l - 1][i], ad;
      if (mode == ORC_MODE_BF16 && l - 1 <= L - 3 && a->act == ORC_ACT_TANH)
        ad = act_d(a->act, T->z[l - 1][i], rbf16(hv));
      else if (mode == ORC_MODE_BF16 && l - 1 >= 2 && l - 1 <= L - 3 && a->act == ORC_ACT_SILU)
        ad = rbf16(act_d(a->act, T->z[l - 1][i], hv));
      else
        ad = act_d(a->act, T->z[l - 1][i], hv);
      dn[i] = rnd(mode, acc * rnd(mode, ad));
    }
    memcpy(dl, dn, sizeof(double) * fi);
  }
}

void orc_backward(const orc_arch* a, const double* theta, int net, const double x[3],
                  double cot, int mode, double* grad) {
  tape_t* T = (tape_t*)malloc(sizeof(tape_t));
  fwd_tape(a, theta, net, x, mode, T);
  bwd_tape(a, theta, net, cot, mode, T, grad);
  free(T);
}

/* ------------------------------------------------------------------------ */
/* loss and gradient ("local L2-norm residual r_p = ||M^-1 A u - M^-1 b||", */
/* S:345-348; G1 loss = (1/N) sum r^2 + (lambda_b/N_b) sum r_b^2)            */
/* ------------------------------------------------------------------------ */
static int net_of(const orc_arch* a, int tag) { return a->n_nets == 1 ? 0 : tag; }

/* r for one assembled row. fp64: raw = sum coef u - rhs, r = raw / d (S:267,
 * S:248).  Emulation modes evaluate M^-1 A u - M^-1 b in fp32 with the
 * normalised coefficients (the product's arithmetic), to measure its noise. */
static double row_residual(const orc_row* row, const double u[7], int mode) {
  if (mode == ORC_MODE_F64) {
    double raw = 0.0;
    for (int j = 0; j < 7; ++j) raw += row->coef[j] * u[j];
    raw -= row->rhs;
    return raw / row->d;
  }
  float acc = (float)u[0];
  for (int j = 1; j < 7; ++j) acc = acc + (float)(row->coef[j] / row->d) * (float)u[j];
  acc = acc - (float)(row->rhs / row->d);
  return acc;
}

static int point_term(const orc_row* row) {
  return row->crossed ? ORC_T_CROSSED : (row->side == 0 ? ORC_T_UNX_MINUS : ORC_T_UNX_PLUS);
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int orc_loss_grad(const orc_problem* pb, const orc_arch* a, const double* theta,
                  const float* pts, int64_t n, const float* bpts, int64_t nb, float h,
                  int64_t n_glob, int64_t nb_glob, int mode, unsigned terms,
                  double* loss_terms, double* grad, double* grad_terms, int nthreads) {
  int64_t P = orc_param_count(a);
  int nt = nthreads > 0 ? nthreads : orc_num_threads();
  int nslots = grad_terms ? 4 : 1;
  double* part = (double*)calloc((size_t)nt * nslots * P, sizeof(double));
  double* lpart = (double*)calloc((size_t)nt * 4, sizeof(double));
  int err = 0;
  int64_t ntot = n + nb;
#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    int t = omp_get_thread_num();
#else
    int t = 0;
#endif
    tape_t* T = (tape_t*)malloc(sizeof(tape_t));
    int64_t lo = ntot * t / nt, hi = ntot * (t + 1) / nt;   /* static contiguous chunk */
    for (int64_t i = lo; i < hi; ++i) {
      if (i < n) {
        orc_row row;
        int rc = orc_assemble(pb, pts + 3 * i, h, 0, &row);
        if (rc) {
#pragma omp atomic write
          err = rc;
          continue;
        }
        int term = point_term(&row);
        if (!(terms & (1u << term))) continue;
        double u[7];
        for (int j = 0; j < 7; ++j) {
          double x[3] = {row.pos[j][0], row.pos[j][1], row.pos[j][2]};
          u[j] = fwd_tape(a, theta, net_of(a, row.tag[j]), x, mode, T);
        }
        double r = row_residual(&row, u, mode);
        lpart[4 * t + term] += r * r / (double)n_glob;
        double* g = part + ((size_t)t * nslots + (grad_terms ? term : 0)) * P;
        for (int j = 0; j < 7; ++j) {                      /* cotangents 2 r coef_j / d */
          double cj = (j == 0) ? 1.0 : row.coef[j] / row.d;
          double cot = 2.0 / (double)n_glob * r * cj;
          if (mode != ORC_MODE_F64) cot = (float)(2.0f / (float)n_glob * (float)r * (float)cj);
          double x[3] = {row.pos[j][0], row.pos[j][1], row.pos[j][2]};
          fwd_tape(a, theta, net_of(a, row.tag[j]), x, mode, T);
          bwd_tape(a, theta, net_of(a, row.tag[j]), cot, mode, T, g);
        }
      } else {
        if (!(terms & (1u << ORC_T_BOUNDARY))) continue;
        const float* pb3 = bpts + 3 * (i - n);
        double x[3] = {pb3[0], pb3[1], pb3[2]};
        int s = orc_side(pb, x);                           /* S:285 boundary_residual */
        double rb = fwd_tape(a, theta, net_of(a, s), x, mode, T) - orc_g(pb, x);
        if (mode != ORC_MODE_F64) rb = (float)rb;
        lpart[4 * t + ORC_T_BOUNDARY] += pb->lambda_b * rb * rb / (double)nb_glob;
        double cot = 2.0 * pb->lambda_b / (double)nb_glob * rb;
        double* g = part + ((size_t)t * nslots + (grad_terms ? ORC_T_BOUNDARY : 0)) * P;
        bwd_tape(a, theta, net_of(a, s), cot, mode, T, g);
      }
    }
    free(T);
  }
  for (int k = 0; k < 4; ++k) {
    double s = 0.0;
    for (int t = 0; t < nt; ++t) s += lpart[4 * t + k];       /* fixed thread order */
    loss_terms[k] = s;
  }
  for (int64_t p = 0; p < P; ++p) {
    double tot = 0.0;
    for (int k = 0; k < nslots; ++k) {
      double s = 0.0;
      for (int t = 0; t < nt; ++t) s += part[((size_t)t * nslots + k) * P + p];
      if (grad_terms) grad_terms[(size_t)k * P + p] = s;
      tot += s;
    }
    grad[p] = tot;
  }
  free(part); free(lpart);
  return err;
}

int orc_residuals(const orc_problem* pb, const orc_arch* a, const double* theta,
                  const float* pts, int64_t n, const float* bpts, int64_t nb, float h,
                  int mode, double* r, double* rb) {
  int err = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    tape_t* T = (tape_t*)malloc(sizeof(tape_t));
    orc_row row;
    int rc = orc_assemble(pb, pts + 3 * i, h, 0, &row);
    if (rc) {
#pragma omp atomic write
      err = rc;
    } else {
      double u[7];
      for (int j = 0; j < 7; ++j) {
        double x[3] = {row.pos[j][0], row.pos[j][1], row.pos[j][2]};
        u[j] = fwd_tape(a, theta, net_of(a, row.tag[j]), x, mode, T);
      }
      r[i] = row_residual(&row, u, mode);
    }
    free(T);
  }
  for (int64_t i = 0; i < nb; ++i) {
    double x[3] = {bpts[3 * i], bpts[3 * i + 1], bpts[3 * i + 2]};
    rb[i] = orc_forward(a, theta, net_of(a, orc_side(pb, x)), x, mode) - orc_g(pb, x);
  }
  return err;
}

int orc_residual_exact(const orc_problem* pb, const float* pts, int64_t n, float h,
                       double* raw, double* r, uint8_t* cls) {
  int err = 0;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    orc_row row;
    int rc = orc_assemble(pb, pts + 3 * i, h, 0, &row);
    if (rc) {
#pragma omp atomic write
      err = rc;
      continue;
    }
    double acc = 0.0;
    for (int j = 0; j < 7; ++j) {
      double x[3] = {row.pos[j][0], row.pos[j][1], row.pos[j][2]}, u;
      orc_exact(pb, row.tag[j], x, &u, NULL);
      acc += row.coef[j] * u;
    }
    raw[i] = acc - row.rhs;
    r[i] = raw[i] / row.d;
    cls[i] = (uint8_t)(row.crossed ? 2 : row.side);
  }
  return err;
}

void orc_eval(const orc_problem* pb, const orc_arch* a, const double* theta,
              const float* pts, int64_t n, int mode, double* u) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    u[i] = orc_forward(a, theta, net_of(a, orc_side(pb, x)), x, mode);
  }
}

/* ------------------------------------------------------------------------ */
/* Error norms on the evaluation grid (Table 1): over all     */
/* (M+1)^3 nodal points p of the box, e(p) = u_{side(p)}(p) - u*_{side(p)}(p),   */
/* rmse = sqrt(mean e^2), linf = max |e|.  Nodal coordinates lo + (hi-lo) i/M    */
/* in fp64, rounded to fp32 (the points the networks see), x fastest.    */
/* Returns -1 when the problem has no closed-form solution.                      */
/* ------------------------------------------------------------------------ */
int orc_error_norms(const orc_problem* pb, const orc_arch* a, const double* theta, int M,
                    int mode, double out[2]) {
  const int64_t m1 = (int64_t)M + 1, total = m1 * m1 * m1;
  double sum = 0.0, mx = 0.0;
  int bad = 0;
  for (int64_t g = 0; g < total; ++g) {
    const int64_t idx[3] = {g % m1, (g / m1) % m1, g / (m1 * m1)};
    double x[3];
    for (int c = 0; c < 3; ++c) {
      const double lo = -1.0, hi = 1.0;   /* the box (G23) */
      x[c] = (double)(float)(lo + (hi - lo) * (double)idx[c] / (double)M);
    }
    const int s = orc_side(pb, x);
    double ue, grad[3];
    if (orc_exact(pb, s, x, &ue, grad) != 0) { bad = 1; break; }   /* 0 = defined */
    const double e = orc_forward(a, theta, net_of(a, s), x, mode) - ue;
    sum += e * e;
    if (fabs(e) > mx) mx = fabs(e);
  }
  if (bad) return -1;
  out[0] = sqrt(sum / (double)total);
  out[1] = mx;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Adam: t <- t+1; m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2;      */
/* theta <- theta - lr mhat / (sqrt(vhat) + eps)                             */
/* ------------------------------------------------------------------------ */
void orc_adam(int64_t P, double* theta, double* m, double* v, const double* g,
              int64_t t, double lr, double b1, double b2, double eps) {
  double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
  for (int64_t i = 0; i < P; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    double mh = m[i] / bc1, vh = v[i] / bc2;
    theta[i] -= lr * mh / (sqrt(vh) + eps);
  }
}

/* fp32 mirror: bias corrections in fp64 then rounded; every op below is one
 * fp32 rounding in the written order. */
void orc_adam_f32(int64_t P, float* theta, float* m, float* v, const float* g,
                  int64_t t, float lr, float b1, float b2, float eps) {
  float bc1 = (float)(1.0 - pow((double)b1, (double)t));
  float bc2 = (float)(1.0 - pow((double)b2, (double)t));
  float ob1 = 1.0f - b1, ob2 = 1.0f - b2;
  for (int64_t i = 0; i < P; ++i) {
    float gi = g[i];
    float mi = b1 * m[i] + ob1 * gi;
    float vi = b2 * v[i] + ob2 * (gi * gi);
    m[i] = mi; v[i] = vi;
    float mh = mi / bc1, vh = vi / bc2;
    float den = sqrtf(vh) + eps;
    theta[i] = theta[i] - (lr * mh) / den;
  }
}
