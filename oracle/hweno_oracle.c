/* TEST INFRASTRUCTURE ONLY — see hweno_oracle.h.
 *
 * Every function restates the reference in fp64 (weights fp64 or fp32) and
 * cites the file:line it follows (paths relative to /root/reference/proj).
 * Expressions keep the reference's evaluation order; the build uses
 * -ffp-contract=off so no multiply-add is fused behind our back. */
#include "hweno_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define RG 4 /* kRadialGhost, evolve.hpp:14 */
#define AG 2 /* kAngularGhost, evolve.hpp:15 */
#define NC 4 /* kComponents,  evolve.hpp:16 */

static inline size_t lay_width(const orc_problem* p) { return (size_t)p->nrho + 2 * RG; }
static inline size_t lay_plane(const orc_problem* p) {
  return lay_width(p) * ((size_t)p->ntheta + 2 * AG);
}
/* FieldLayout::at, evolve.hpp:30-34 */
static inline size_t lay_at(const orc_problem* p, int c, int j, int k) {
  return (size_t)c * lay_plane(p) + (size_t)(k + AG) * lay_width(p) + (size_t)(j + RG);
}

size_t orc_state_size(int nrho, int ntheta) {
  return (size_t)NC * ((size_t)nrho + 2 * RG) * ((size_t)ntheta + 2 * AG);
}

/* EvolutionRhs ctor, evolve.cpp:19-30 */
int orc_prepare(orc_problem* p) {
  const double* lam = p->coef + (size_t)1 * p->nrho * p->ntheta;
  for (int k = 0; k < p->ntheta; ++k) {
    int sp = 0;
    while (sp < p->nrho && lam[sp + (size_t)p->nrho * k] < 0.0) ++sp;
    for (int j = sp; j < p->nrho; ++j)
      if (lam[j + (size_t)p->nrho * k] < 0.0) return -1;
    p->split[k] = sp;
  }
  return 0;
}

/* apply_boundaries, evolve.cpp:40-71 */
void orc_apply_boundaries(const orc_problem* p, double* u) {
  const int n = p->nrho, nt = p->ntheta;
  const long long w = (long long)lay_width(p);
  for (int k = 0; k < nt; ++k)
    for (int c = 0; c < NC; ++c) {
      double* q0 = u + lay_at(p, c, 0, k);
      for (int t = 1; t <= RG; ++t)
        q0[-t] = 4.0 * q0[-t + 1] - 6.0 * q0[-t + 2] + 4.0 * q0[-t + 3] - q0[-t + 4];
      double* q = q0 + n - 1;
      for (int t = 1; t <= RG; ++t)
        q[t] = 4.0 * q[t - 1] - 6.0 * q[t - 2] + 4.0 * q[t - 3] - q[t - 4];
    }
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < NC; ++c) {
      double* base = u + lay_at(p, c, j, 0);
      for (int t = 0; t < AG; ++t) {
        double north = base[(long long)t * w];
        double south = base[(long long)(nt - 1 - t) * w];
        base[-(long long)(1 + t) * w] = p->parity > 0 ? north : -north;
        base[(long long)(nt + t) * w] = p->parity > 0 ? south : -south;
      }
    }
}

/* weno5_weights_t<double>, spatial.hpp:29-65 */
void orc_weno5_weights_f64(const double a[5], double eps, double w[3]) {
  if (isinf(eps)) {
    w[0] = 1.0 / 10.0;
    w[1] = 6.0 / 10.0;
    w[2] = 3.0 / 10.0;
    return;
  }
  const double f0 = a[0], f1 = a[1], f2 = a[2], f3 = a[3], f4 = a[4];
  const double c1312 = 13.0 / 12.0, quarter = 1.0 / 4.0;
  double t = f0 - 2.0 * f1 + f2;
  double s = f0 - 4.0 * f1 + 3.0 * f2;
  double is0 = c1312 * t * t + quarter * s * s;
  t = f1 - 2.0 * f2 + f3;
  s = f1 - f3;
  double is1 = c1312 * t * t + quarter * s * s;
  t = f2 - 2.0 * f3 + f4;
  s = 3.0 * f2 - 4.0 * f3 + f4;
  double is2 = c1312 * t * t + quarter * s * s;
  double e0 = eps + is0, e1 = eps + is1, e2 = eps + is2;
  double a0 = (1.0 / 10.0) / (e0 * e0);
  double a1 = (6.0 / 10.0) / (e1 * e1);
  double a2 = (3.0 / 10.0) / (e2 * e2);
  double inv = 1.0 / (a0 + a1 + a2);
  w[0] = a0 * inv;
  w[1] = a1 * inv;
  w[2] = a2 * inv;
}

/* weno5_weights_t<float>: the paper's mixed mode with the window demoted to
 * fp32 (spatial.hpp:40-42 demotes to the weight scalar). */
void orc_weno5_weights_f32(const double a[5], float eps, float w[3]) {
  if (isinf(eps)) {
    w[0] = 1.0f / 10.0f;
    w[1] = 6.0f / 10.0f;
    w[2] = 3.0f / 10.0f;
    return;
  }
  const float f0 = (float)a[0], f1 = (float)a[1], f2 = (float)a[2],
              f3 = (float)a[3], f4 = (float)a[4];
  const float c1312 = 13.0f / 12.0f, quarter = 1.0f / 4.0f;
  float t = f0 - 2.0f * f1 + f2;
  float s = f0 - 4.0f * f1 + 3.0f * f2;
  float is0 = c1312 * t * t + quarter * s * s;
  t = f1 - 2.0f * f2 + f3;
  s = f1 - f3;
  float is1 = c1312 * t * t + quarter * s * s;
  t = f2 - 2.0f * f3 + f4;
  s = 3.0f * f2 - 4.0f * f3 + f4;
  float is2 = c1312 * t * t + quarter * s * s;
  float e0 = eps + is0, e1 = eps + is1, e2 = eps + is2;
  float a0 = (1.0f / 10.0f) / (e0 * e0);
  float a1 = (6.0f / 10.0f) / (e1 * e1);
  float a2 = (3.0f / 10.0f) / (e2 * e2);
  float inv = 1.0f / (a0 + a1 + a2);
  w[0] = a0 * inv;
  w[1] = a1 * inv;
  w[2] = a2 * inv;
}

/* weno5_interface + weno5_combine, spatial.hpp:68-92 */
double orc_weno5_interface(const double a[5], int mode, double eps) {
  double w[3];
  if (mode == ORC_MIXED) {
    float wf[3];
    orc_weno5_weights_f32(a, (float)eps, wf);
    w[0] = (double)wf[0];
    w[1] = (double)wf[1];
    w[2] = (double)wf[2];
  } else {
    orc_weno5_weights_f64(a, eps, w);
  }
  double inv = 1.0 / (w[0] + w[1] + w[2]);
  w[0] = w[0] * inv;
  w[1] = w[1] * inv;
  w[2] = w[2] * inv;
  const double sixth = 1.0 / 6.0;
  double q0 = (2.0 * a[0] - 7.0 * a[1] + 11.0 * a[2]);
  double q1 = (-a[1] + 5.0 * a[2] + 2.0 * a[3]);
  double q2 = (2.0 * a[2] + 5.0 * a[3] - a[4]);
  return sixth * (w[0] * q0 + w[1] * q1 + w[2] * q2);
}

static inline double w5(double a0, double a1, double a2, double a3, double a4,
                        int mode, double eps) {
  const double a[5] = {a0, a1, a2, a3, a4};
  return orc_weno5_interface(a, mode, eps);
}

/* weno5_row_derivative, spatial.hpp:140-155 */
void orc_weno5_row_derivative(const double* u, int n, double drho, int mode,
                              double eps, int minus, double* du) {
  double inv = 1.0 / drho;
  double prev = minus ? w5(u[2], u[1], u[0], u[-1], u[-2], mode, eps)
                      : w5(u[-3], u[-2], u[-1], u[0], u[1], mode, eps);
  for (int j = 0; j < n; ++j) {
    double cur = minus ? w5(u[j + 3], u[j + 2], u[j + 1], u[j], u[j - 1], mode, eps)
                       : w5(u[j - 2], u[j - 1], u[j], u[j + 1], u[j + 2], mode, eps);
    du[j] = (cur - prev) * inv;
    prev = cur;
  }
}

/* weno3_weights_t / weno3_interface, spatial.hpp:94-130 */
static double w3(double a0, double a1, double a2, int mode, double eps) {
  double w0, w1;
  if (isinf(eps)) {
    if (mode == ORC_MIXED) {
      w0 = (double)(1.0f / 3.0f);
      w1 = (double)(2.0f / 3.0f);
    } else {
      w0 = 1.0 / 3.0;
      w1 = 2.0 / 3.0;
    }
  } else if (mode == ORC_MIXED) {
    float f0 = (float)a0, f1 = (float)a1, f2 = (float)a2, e = (float)eps;
    float d0 = f1 - f0, d1 = f2 - f1;
    float e0 = e + d0 * d0, e1 = e + d1 * d1;
    float x0 = (1.0f / 3.0f) / (e0 * e0);
    float x1 = (2.0f / 3.0f) / (e1 * e1);
    float inv = 1.0f / (x0 + x1);
    w0 = (double)(x0 * inv);
    w1 = (double)(x1 * inv);
  } else {
    double d0 = a1 - a0, d1 = a2 - a1;
    double e0 = eps + d0 * d0, e1 = eps + d1 * d1;
    double x0 = (1.0 / 3.0) / (e0 * e0);
    double x1 = (2.0 / 3.0) / (e1 * e1);
    double inv = 1.0 / (x0 + x1);
    w0 = x0 * inv;
    w1 = x1 * inv;
  }
  double inv = 1.0 / (w0 + w1);
  w0 = w0 * inv;
  w1 = w1 * inv;
  const double half = 1.0 / 2.0;
  double q0 = half * (3.0 * a1 - a0);
  double q1 = half * (a1 + a2);
  return w0 * q0 + w1 * q1;
}

/* weno3_row_derivative, spatial.hpp:157-169 */
static void weno3_row(const double* u, int n, double drho, int mode,
                      double eps, int minus, double* du) {
  double inv = 1.0 / drho;
  double prev = minus ? w3(u[1], u[0], u[-1], mode, eps)
                      : w3(u[-2], u[-1], u[0], mode, eps);
  for (int j = 0; j < n; ++j) {
    double cur = minus ? w3(u[j + 2], u[j + 1], u[j], mode, eps)
                       : w3(u[j - 1], u[j], u[j + 1], mode, eps);
    du[j] = (cur - prev) * inv;
    prev = cur;
  }
}

/* fd6_derivative, spatial.hpp:178-182 */
static inline double fd6(const double* u, double drho) {
  return (u[3] - u[-3] - 9.0 * (u[2] - u[-2]) + 45.0 * (u[1] - u[-1])) / (60.0 * drho);
}

/* ko8_dissipation, spatial.hpp:184-191 */
static inline double ko8(const double* u, double sigma, double h) {
  double d8 = u[-4] + u[4] - 8.0 * (u[-3] + u[3]) + 28.0 * (u[-2] + u[2]) -
              56.0 * (u[-1] + u[1]) + 70.0 * u[0];
  return sigma * d8 / (256.0 * h);
}

/* run_rhs<TW>, evolve.cpp:73-179 (phases 1-3) */
static void run_rhs(const orc_problem* p, const double* u, double* du) {
  const int n = p->nrho, nt = p->ntheta;
  const size_t P = (size_t)n * nt;
  const long long w = (long long)lay_width(p);
  double* scratch = (double*)malloc(sizeof(double) * 6 * P);
  double *dps_r = scratch, *dps_i = scratch + P, *dpi_r = scratch + 2 * P,
         *dpi_i = scratch + 3 * P, *ang_r = scratch + 4 * P, *ang_i = scratch + 5 * P;
  /* phase 1, evolve.cpp:88-122 */
  for (int k = 0; k < nt; ++k) {
    const double* rows[NC];
    for (int c = 0; c < NC; ++c) rows[c] = u + lay_at(p, c, 0, k);
    double* out[NC] = {dps_r + (size_t)k * n, dps_i + (size_t)k * n,
                       dpi_r + (size_t)k * n, dpi_i + (size_t)k * n};
    if (p->scheme == ORC_FD6KO) {
      for (int c = 0; c < NC; ++c)
        for (int j = 0; j < n; ++j) out[c][j] = fd6(rows[c] + j, p->drho);
      continue;
    }
    const int sp = p->split[k];
    if (p->scheme == ORC_WENO5) {
      orc_weno5_row_derivative(rows[0], n, p->drho, p->mode, p->eps, 1, out[0]);
      orc_weno5_row_derivative(rows[1], n, p->drho, p->mode, p->eps, 1, out[1]);
      for (int c = 2; c < NC; ++c) {
        if (sp > 0) orc_weno5_row_derivative(rows[c], sp, p->drho, p->mode, p->eps, 1, out[c]);
        if (sp < n)
          orc_weno5_row_derivative(rows[c] + sp, n - sp, p->drho, p->mode, p->eps, 0, out[c] + sp);
      }
    } else {
      weno3_row(rows[0], n, p->drho, p->mode, p->eps, 1, out[0]);
      weno3_row(rows[1], n, p->drho, p->mode, p->eps, 1, out[1]);
      for (int c = 2; c < NC; ++c) {
        if (sp > 0) weno3_row(rows[c], sp, p->drho, p->mode, p->eps, 1, out[c]);
        if (sp < n) weno3_row(rows[c] + sp, n - sp, p->drho, p->mode, p->eps, 0, out[c] + sp);
      }
    }
  }
  /* phase 2, evolve.cpp:125-136 with theta_derivatives_column,
   * spatial.hpp:208-222 */
  const double inv1 = 1.0 / (12.0 * p->dtheta);
  const double inv2 = 1.0 / (12.0 * p->dtheta * p->dtheta);
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < 2; ++c) {
      const double* col = u + lay_at(p, c, j, 0);
      double* ang = c == 0 ? ang_r : ang_i;
      for (int k = 0; k < nt; ++k) {
        const double* q = col + (long long)k * w;
        double m2 = q[-2 * w], m1 = q[-w], p1 = q[w], p2 = q[2 * w];
        double d1 = (m2 - 8.0 * m1 + 8.0 * p1 - p2) * inv1;
        double d2 = (-m2 + 16.0 * m1 - 30.0 * q[0] + 16.0 * p1 - p2) * inv2;
        ang[j + (size_t)k * n] = d2 + p->cotth[k] * d1;
      }
    }
  /* phase 3, evolve.cpp:139-178 */
  for (int k = 0; k < nt; ++k) {
    const size_t ci = (size_t)k * n;
    const double *psr = u + lay_at(p, 0, 0, k), *psi = u + lay_at(p, 1, 0, k),
                 *pir = u + lay_at(p, 2, 0, k), *pii = u + lay_at(p, 3, 0, k);
    double *d0 = du + lay_at(p, 0, 0, k), *d1 = du + lay_at(p, 1, 0, k),
           *d2 = du + lay_at(p, 2, 0, k), *d3 = du + lay_at(p, 3, 0, k);
    const double* cs = p->coef;
    const double *b = cs + 0 * P + ci, *lam = cs + 1 * P + ci, *wre = cs + 2 * P + ci,
                 *wim = cs + 3 * P + ci, *btr = cs + 4 * P + ci, *bti = cs + 5 * P + ci,
                 *cre = cs + 6 * P + ci, *cim = cs + 7 * P + ci, *ath = cs + 8 * P + ci;
    const double *Dsr = dps_r + ci, *Dsi = dps_i + ci, *Dpr = dpi_r + ci,
                 *Dpi = dpi_i + ci, *Ar = ang_r + ci, *Ai = ang_i + ci;
    for (int j = 0; j < n; ++j) {
      d0[j] = pir[j] - b[j] * Dsr[j];
      d1[j] = pii[j] - b[j] * Dsi[j];
      d2[j] = -lam[j] * Dpr[j] + wre[j] * Dsr[j] - wim[j] * Dsi[j] + btr[j] * pir[j] -
              bti[j] * pii[j] + cre[j] * psr[j] - cim[j] * psi[j] + ath[j] * Ar[j];
      d3[j] = -lam[j] * Dpi[j] + wre[j] * Dsi[j] + wim[j] * Dsr[j] + btr[j] * pii[j] +
              bti[j] * pir[j] + cre[j] * psi[j] + cim[j] * psr[j] + ath[j] * Ai[j];
    }
    if (p->scheme == ORC_FD6KO) {
      const double* rows[NC] = {psr, psi, pir, pii};
      double* outs[NC] = {d0, d1, d2, d3};
      for (int c = 0; c < NC; ++c)
        for (int j = 0; j < n; ++j)
          outs[c][j] = outs[c][j] - ko8(rows[c] + j, p->sigma, p->drho);
    }
  }
  free(scratch);
}

/* EvolutionRhs::operator(), evolve.cpp:181-187 */
void orc_rhs(const orc_problem* p, double* u, double* du) {
  orc_apply_boundaries(p, u);
  run_rhs(p, u, du);
}

/* ssprk33_step, timestep.hpp:54-71 */
void orc_ssprk33_step(const orc_problem* p, double* u, double dt) {
  const size_t n = orc_state_size(p->nrho, p->ntheta);
  double* s1 = (double*)calloc(n, sizeof(double));
  double* f = (double*)calloc(n, sizeof(double));
  const double c34 = 3.0 / 4.0, c14 = 1.0 / 4.0, c13 = 1.0 / 3.0, c23 = 2.0 / 3.0;
  orc_rhs(p, u, f);
  for (size_t i = 0; i < n; ++i) s1[i] = u[i] + dt * f[i];
  orc_rhs(p, s1, f);
  for (size_t i = 0; i < n; ++i) s1[i] = c34 * u[i] + c14 * (s1[i] + dt * f[i]);
  orc_rhs(p, s1, f);
  for (size_t i = 0; i < n; ++i) u[i] = c13 * u[i] + c23 * (s1[i] + dt * f[i]);
  free(s1);
  free(f);
}

/* ssprk104_step (reference low-storage form), timestep.hpp:78-109 */
void orc_ssprk104_step(const orc_problem* p, double* u, double dt) {
  const size_t n = orc_state_size(p->nrho, p->ntheta);
  double* s1 = (double*)calloc(n, sizeof(double));
  double* s2 = (double*)calloc(n, sizeof(double));
  double* f = (double*)calloc(n, sizeof(double));
  double* f4 = (double*)calloc(n, sizeof(double));
  const double dt6 = dt / 6.0;
  memcpy(s1, u, n * sizeof(double));
  for (int i = 1; i <= 4; ++i) {
    orc_rhs(p, s1, f);
    for (size_t q = 0; q < n; ++q) s1[q] = s1[q] + dt6 * f[q];
  }
  memcpy(s2, s1, n * sizeof(double));
  orc_rhs(p, s1, f4);
  const double c35 = 3.0 / 5.0, c25 = 2.0 / 5.0, dt15 = dt / 15.0;
  for (size_t q = 0; q < n; ++q) s1[q] = c35 * u[q] + c25 * s1[q] + dt15 * f4[q];
  for (int i = 6; i <= 9; ++i) {
    orc_rhs(p, s1, f);
    for (size_t q = 0; q < n; ++q) s1[q] = s1[q] + dt6 * f[q];
  }
  orc_rhs(p, s1, f);
  const double c125 = 1.0 / 25.0, c925 = 9.0 / 25.0, c350 = 3.0 / 50.0, c110 = 1.0 / 10.0;
  for (size_t q = 0; q < n; ++q)
    u[q] = c125 * u[q] + c925 * s2[q] + c35 * s1[q] + dt * (c350 * f4[q] + c110 * f[q]);
  free(s1);
  free(s2);
  free(f);
  free(f4);
}

/* state_admissible, evolve.cpp:217-235 */
int orc_state_admissible(const orc_problem* p, const double* u, double limit) {
  for (int c = 0; c < NC; ++c)
    for (int k = 0; k < p->ntheta; ++k) {
      const double* row = u + lay_at(p, c, 0, k);
      for (int j = 0; j < p->nrho; ++j)
        if (!(fabs(row[j]) <= limit)) return 0;
    }
  return 1;
}

/* advance_steps without hook, evolve.cpp:237-265 */
void orc_advance(const orc_problem* p, int stepper, double dt, long s0,
                 long s1, double* u, long* stats) {
  stats[0] = 0;
  stats[1] = 0;
  stats[2] = -1;
  for (long s = s0; s < s1; ++s) {
    if (stepper == ORC_SSPRK33)
      orc_ssprk33_step(p, u, dt);
    else
      orc_ssprk104_step(p, u, dt);
    stats[0] = s + 1 - s0;
    if (!orc_state_admissible(p, u, 1e30)) {
      stats[1] = 1;
      stats[2] = s + 1;
      break;
    }
  }
}
