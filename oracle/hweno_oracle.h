/* TEST INFRASTRUCTURE ONLY — the CPU checker for the GPU hot path.
 *
 * Plain-C restatement of the reference hot path in fp64 work precision with
 * fp64 ("f64" mode) or fp32 ("mixed" mode) WENO weights.  It keeps the
 * reference's data layout (FieldLayout, proj/include/hweno/evolve.hpp:23-35:
 * 4 component planes of (nrho+8) x (ntheta+4), rho fastest) and its operation
 * order, so the only difference from the reference is the scalar type
 * (double instead of DDReal; the GPU modes are one precision tier below the
 * reference's full/mixed modes).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. */
#ifndef HWENO_ORACLE_H
#define HWENO_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_WENO5 = 0, ORC_WENO3 = 1, ORC_FD6KO = 2 };
enum { ORC_F64 = 0, ORC_MIXED = 1 };
enum { ORC_SSPRK33 = 0, ORC_SSPRK104 = 1 };

typedef struct {
  int nrho, ntheta;
  double drho, dtheta;
  int parity;            /* theta ghost sign (-1)^(m+s), evolve.cpp:18 */
  const double* coef;    /* 9 planes b,lam,w_re,w_im,bt_re,bt_im,c_re,c_im,ath */
  const double* cotth;   /* ntheta */
  int scheme;            /* ORC_WENO5 | ORC_FD6KO | ORC_WENO3 */
  int mode;              /* ORC_F64 | ORC_MIXED */
  double eps, sigma;
  int* split;            /* ntheta, filled by orc_prepare */
} orc_problem;

size_t orc_state_size(int nrho, int ntheta);
/* evolve.cpp:19-30: per-row first j with lam >= 0; returns -1 if lam changes
 * sign more than once along a row (the reference throws runtime_error). */
int orc_prepare(orc_problem* p);
void orc_apply_boundaries(const orc_problem* p, double* u);
/* EvolutionRhs::operator(): fills u's ghosts, writes du's interior. */
void orc_rhs(const orc_problem* p, double* u, double* du);
void orc_ssprk33_step(const orc_problem* p, double* u, double dt);
void orc_ssprk104_step(const orc_problem* p, double* u, double dt);
int orc_state_admissible(const orc_problem* p, const double* u, double limit);
/* advance_steps with no hook: stats = {steps_done, blew_up, blowup_step} */
void orc_advance(const orc_problem* p, int stepper, double dt, long s0,
                 long s1, double* u, long* stats);

void orc_weno5_weights_f64(const double a[5], double eps, double w[3]);
void orc_weno5_weights_f32(const double a[5], float eps, float w[3]);
double orc_weno5_interface(const double a[5], int mode, double eps);
void orc_weno5_row_derivative(const double* u, int n, double drho, int mode,
                              double eps, int minus, double* du);

#ifdef __cplusplus
}
#endif
#endif
