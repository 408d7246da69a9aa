// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A flat C ABI over the *unmodified* reference library (libhweno built from
// /root/reference/proj/src by oracle/Makefile).  It lets the Python tests and
// bench.py's cpu_baseline / --impl reference leg drive the reference's own
// setup and hot path:
//   make_grid / assemble_coefficients      proj/src/geometry.cpp:73-168
//   EvolutionRhs (ctor, operator())        proj/src/evolve.cpp:10-187
//   initial_data                           proj/src/evolve.cpp:189-215
//   select_dt / stepper_step               proj/include/hweno/timestep.hpp:25-118
//   advance_steps                          proj/src/evolve.cpp:237-265
//   HorizonSampler / multipole_project     proj/src/diagnostics.cpp:128-283
// No reference source is copied here; only its public headers are included.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "hweno/angular.hpp"
#include "hweno/coeff_kernels.hpp"
#include "hweno/diagnostics.hpp"
#include "hweno/evolve.hpp"
#include "hweno/geometry.hpp"
#include "hweno/io.hpp"
#include "hweno/parallel.hpp"
#include "hweno/timestep.hpp"
#include "hweno_gpu_setup.hpp"  // the reference's assembly on host threads (sub-grids)

using namespace hweno;

namespace {

thread_local std::string g_err;

struct RefHandle {
  PhysicalParams p;
  Grid g;
  CoefficientSet cs;
  SchemeSpec spec;
  std::unique_ptr<WorkerPool> pool;
  std::unique_ptr<EvolutionRhs> rhs;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void to_dd(const StateVec& u, double* out) {
  for (size_t i = 0; i < u.size(); ++i) {
    out[2 * i] = u[i].hi;
    out[2 * i + 1] = u[i].lo;
  }
}

StateVec from_dd(const double* in, size_t n) {
  StateVec u(n);
  for (size_t i = 0; i < n; ++i) u[i] = DDReal(in[2 * i], in[2 * i + 1]);
  return u;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// scheme: 0 weno5, 1 weno3, 2 fd6ko; mode: 0 full (DD weights), 1 mixed
// (fp64 weights).  eps may be +inf (frozen linear weights).
// deeper > 0: the excision sits `deeper` cells below the default grid of
// nrho - deeper points, same spacing (make_grid's rho_min overload, as in
// proj/tests/test_evolve.cpp:397-410)
int ref_create_deeper(double M, double a, int spin, int mmode, double S, int nrho,
                      int ntheta, int scheme, int mode, double eps, double sigma,
                      int workers, int deeper, void** out);

int ref_create(double M, double a, int spin, int mmode, double S, int nrho,
               int ntheta, int scheme, int mode, double eps, double sigma,
               int workers, void** out) {
  return ref_create_deeper(M, a, spin, mmode, S, nrho, ntheta, scheme, mode, eps, sigma,
                           workers, 0, out);
}

int ref_create_deeper(double M, double a, int spin, int mmode, double S, int nrho,
                      int ntheta, int scheme, int mode, double eps, double sigma,
                      int workers, int deeper, void** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<RefHandle>();
    h->p.M = WorkReal(M);
    h->p.a = WorkReal(a);
    h->p.spin = spin;
    h->p.mmode = mmode;
    h->p.S = WorkReal(S);
    if (deeper > 0) {
      const Grid g0 = make_grid(nrho - deeper, ntheta, h->p);
      h->g = make_grid(nrho, ntheta, h->p, g0.rho_min - WorkReal(double(deeper)) * g0.drho);
    } else {
      h->g = make_grid(nrho, ntheta, h->p);
    }
    // the unmodified assemble_coefficients, serial or (workers > 1) on theta-row
    // sub-grids from `workers` threads — bitwise the same planes
    h->cs = workers > 1 ? hweno_gpu::assemble_coefficients_parallel(h->g, h->p, workers)
                        : assemble_coefficients(h->g, h->p);
    h->spec.scheme = scheme == 0 ? Scheme::weno5
                     : scheme == 1 ? Scheme::weno3
                                   : Scheme::fd6ko;
    h->spec.mode = mode == 0 ? PrecisionMode::full : PrecisionMode::mixed;
    h->spec.eps = WorkReal(eps);
    h->spec.sigma = WorkReal(sigma);
    h->pool = std::make_unique<WorkerPool>(workers);
    h->rhs = std::make_unique<EvolutionRhs>(h->g, h->cs, h->p, h->spec,
                                            *h->pool);
    *out = h.release();
  });
}

void ref_destroy(void* hv) { delete static_cast<RefHandle*>(hv); }

// dbl[0..] = drho, dtheta, rho_min, max_speed, horizon_rho, S  (hi parts)
// dlo[..]  = the matching lo parts
// ints[0..] = nrho, ntheta, parity, horizon_index, state_size
int ref_info(void* hv, double* dbl, double* dlo, long long* ints) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    WorkReal v[6] = {h->g.drho, h->g.dtheta, h->g.rho_min, h->cs.max_speed,
                     horizon_rho(h->p), h->p.S};
    for (int i = 0; i < 6; ++i) {
      dbl[i] = v[i].hi;
      if (dlo) dlo[i] = v[i].lo;
    }
    ints[0] = h->g.nrho;
    ints[1] = h->g.ntheta;
    ints[2] = ((h->p.mmode + h->p.spin) % 2 == 0) ? 1 : -1;
    ints[3] = h->g.horizon_index;
    ints[4] = (long long)h->rhs->layout().size();
  });
}

// planes: 9*P doubles in the order b, lam, w_re, w_im, bt_re, bt_im, c_re,
// c_im, ath, each indexed j + nrho*k (the reference's CoefficientSet order).
// lo (optional) receives the low limbs.  cotth: ntheta.  rho/theta: grids.
int ref_coeffs(void* hv, double* planes, double* lo, double* cotth,
               double* rho, double* theta) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    const std::vector<WorkReal>* src[9] = {
        &h->cs.b,     &h->cs.lam,   &h->cs.w_re, &h->cs.w_im, &h->cs.bt_re,
        &h->cs.bt_im, &h->cs.c_re,  &h->cs.c_im, &h->cs.ath};
    size_t P = size_t(h->g.nrho) * h->g.ntheta;
    for (int q = 0; q < 9; ++q)
      for (size_t i = 0; i < P; ++i) {
        planes[q * P + i] = (*src[q])[i].hi;
        if (lo) lo[q * P + i] = (*src[q])[i].lo;
      }
    if (cotth)
      for (int k = 0; k < h->g.ntheta; ++k) cotth[k] = h->cs.cotth[k].hi;
    if (rho)
      for (int j = 0; j < h->g.nrho; ++j) rho[j] = h->g.rho[j].hi;
    if (theta)
      for (int k = 0; k < h->g.ntheta; ++k) theta[k] = h->g.theta[k].hi;
  });
}

// Grid::rho / Grid::costh as DD pairs (inputs of hwg_assemble_coefficients)
int ref_grid_dd(void* hv, double* rho_dd, double* costh_dd) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    for (int j = 0; j < h->g.nrho; ++j) {
      rho_dd[2 * j] = h->g.rho[j].hi;
      rho_dd[2 * j + 1] = h->g.rho[j].lo;
    }
    for (int k = 0; k < h->g.ntheta; ++k) {
      costh_dd[2 * k] = h->g.costh[k].hi;
      costh_dd[2 * k + 1] = h->g.costh[k].lo;
    }
  });
}

// all 14 CoefficientSet planes (geometry.hpp:73-90 order: b, lam, w_re,
// w_im, bt_re, bt_im, c_re, c_im, ath, p_mix, r_rad, br_re, br_im, bprime)
// as DD pairs, 14 x P x 2 doubles, and max_speed
int ref_coeffs_all_dd(void* hv, double* planes_dd, double* max_speed_dd) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    const std::vector<WorkReal>* src[14] = {
        &h->cs.b,     &h->cs.lam,   &h->cs.w_re,  &h->cs.w_im,  &h->cs.bt_re,
        &h->cs.bt_im, &h->cs.c_re,  &h->cs.c_im,  &h->cs.ath,   &h->cs.p_mix,
        &h->cs.r_rad, &h->cs.br_re, &h->cs.br_im, &h->cs.bprime};
    const size_t P = size_t(h->g.nrho) * h->g.ntheta;
    for (int q = 0; q < 14; ++q)
      for (size_t i = 0; i < P; ++i) {
        planes_dd[2 * (q * P + i)] = (*src[q])[i].hi;
        planes_dd[2 * (q * P + i) + 1] = (*src[q])[i].lo;
      }
    max_speed_dd[0] = h->cs.max_speed.hi;
    max_speed_dd[1] = h->cs.max_speed.lo;
  });
}

// wave_op_coeffs<DDReal> (coeff_kernels.hpp:661-666) at n points:
// in = n x {rho, cth, M, a, S} DD pairs, sm = n x {spin, mmode},
// out = n x 11 DD pairs (a_tr a_rr bt_re bt_im br_re br_im c_re c_im a_th da_tr da_rr)
int ref_wave_op_coeffs(int n, const double* in, const int* sm, double* out) {
  return guarded([&] {
    for (int i = 0; i < n; ++i) {
      const double* x = in + 10 * i;
      auto w = wave_op_coeffs<WorkReal>(DDReal(x[0], x[1]), DDReal(x[2], x[3]), DDReal(x[4], x[5]),
                                        DDReal(x[6], x[7]), DDReal(x[8], x[9]), sm[2 * i],
                                        sm[2 * i + 1]);
      const WorkReal v[11] = {w.a_tr, w.a_rr, w.bt_re, w.bt_im, w.br_re, w.br_im,
                              w.c_re, w.c_im, w.a_th,  w.da_tr, w.da_rr};
      for (int q = 0; q < 11; ++q) {
        out[22 * i + 2 * q] = v[q].hi;
        out[22 * i + 2 * q + 1] = v[q].lo;
      }
    }
  });
}

// DDReal(p) / DDReal(q) (the reference tests' rat(), test_geometry.cpp)
int ref_rat(long long p, long long q, double* out_dd) {
  return guarded([&] {
    const DDReal r = DDReal(p) / DDReal(q);
    out_dd[0] = r.hi;
    out_dd[1] = r.lo;
  });
}

// low limbs of cot(theta_k) (CoefficientSet::cotth)
int ref_cotth_lo(void* hv, double* lo) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    for (int k = 0; k < h->g.ntheta; ++k) lo[k] = h->cs.cotth[k].lo;
  });
}

// u_dd: 2*state_size doubles ({hi, lo} pairs, reference FieldLayout)
int ref_initial_data(void* hv, int ell, double center, double width,
                     double amplitude, double* u_dd) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    InitialDataSpec id;
    id.ell = ell;
    id.center = WorkReal(center);
    id.width = WorkReal(width);
    id.amplitude = WorkReal(amplitude);
    to_dd(initial_data(h->g, h->cs, h->p, id), u_dd);
  });
}

// EvolutionRhs::operator(): u_dd's ghosts are filled in place, du_dd gets
// the interior RHS (its ghosts are zeroed).
int ref_rhs(void* hv, double* u_dd, double* du_dd) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    size_t n = h->rhs->layout().size();
    StateVec u = from_dd(u_dd, n);
    StateVec du(n);
    (*h->rhs)(u, du);
    to_dd(u, u_dd);
    to_dd(du, du_dd);
  });
}

int ref_apply_boundaries(void* hv, double* u_dd) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    size_t n = h->rhs->layout().size();
    StateVec u = from_dd(u_dd, n);
    h->rhs->apply_boundaries(u);
    to_dd(u, u_dd);
  });
}

// stepper: 0 ssprk33, 1 ssprk104
int ref_select_dt(void* hv, int stepper, double cfl, double* dt_dd) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    StepperSpec st;
    st.kind = stepper == 0 ? StepperSpec::ssprk33 : StepperSpec::ssprk104;
    st.cfl = WorkReal(cfl);
    WorkReal dt = select_dt(h->g, h->cs, st);
    dt_dd[0] = dt.hi;
    dt_dd[1] = dt.lo;
  });
}

// advance_steps with the hook disabled, or (ktheta >= 0) with a hook that
// records the HorizonSampler observables (phi, dphi1..3; re, im each: 8
// doubles hi) plus tau.hi per sample into obs (capacity max_obs rows of 9).
// stats: steps_done, blew_up, blowup_step, n_obs; wall seconds in *wall.
int ref_advance(void* hv, int stepper, double cfl, const double* dt_dd,
                long s0, long s1, double* u_dd, long hook_every, int ktheta,
                double* obs, long max_obs, long* stats, double* wall) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    StepperSpec st;
    st.kind = stepper == 0 ? StepperSpec::ssprk33 : StepperSpec::ssprk104;
    st.cfl = WorkReal(cfl);
    size_t n = h->rhs->layout().size();
    StateVec u = from_dd(u_dd, n);
    WorkReal dt(dt_dd[0], dt_dd[1]);
    SampleHook hook;
    long n_obs = 0;
    std::unique_ptr<HorizonSampler> hs;
    if (ktheta >= 0) {
      hs = std::make_unique<HorizonSampler>(h->g, h->p, h->rhs->layout(),
                                            ktheta);
      hook.every = hook_every;
      hook.fn = [&](long, const WorkReal& tau, const StateVec& s) {
        if (n_obs >= max_obs) return;
        HorizonObservables ob = hs->sample(s);
        double* row = obs + 9 * n_obs;
        row[0] = tau.hi;
        row[1] = ob.phi.re.hi;
        row[2] = ob.phi.im.hi;
        for (int d = 0; d < 3; ++d) {
          row[3 + 2 * d] = ob.dphi[d].re.hi;
          row[4 + 2 * d] = ob.dphi[d].im.hi;
        }
        ++n_obs;
      };
    }
    RunStats rs =
        advance_steps(*h->rhs, st, u, dt, s0, s1, hook, *h->pool);
    to_dd(u, u_dd);
    stats[0] = rs.steps_done;
    stats[1] = rs.blew_up ? 1 : 0;
    stats[2] = rs.blowup_step;
    stats[3] = n_obs;
    if (wall) *wall = rs.wall_seconds;
  });
}

// advance_steps [s0, s1) with the hook disabled except for a timestamp at
// every step (SampleHook every = 1: fired before each step and at s1), so
// stamps[i] - stamps[i-1] is the wall time of step s0 + i - 1 inside ONE
// advance_steps call — the reference's own bench-scaling harness
// (proj/tools/main.cpp:168-221) times one call the same way.  stamps: s1 - s0
// + 1 seconds since the call began.  stats as ref_advance.
int ref_advance_timed(void* hv, int stepper, double cfl, const double* dt_dd, long s0,
                      long s1, double* u_dd, double* stamps, long* stats) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    StepperSpec st;
    st.kind = stepper == 0 ? StepperSpec::ssprk33 : StepperSpec::ssprk104;
    st.cfl = WorkReal(cfl);
    StateVec u = from_dd(u_dd, h->rhs->layout().size());
    WorkReal dt(dt_dd[0], dt_dd[1]);
    SampleHook hook;
    hook.every = 1;
    const auto t0 = std::chrono::steady_clock::now();
    hook.fn = [&](long s, const WorkReal&, const StateVec&) {
      stamps[s - s0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    RunStats rs = advance_steps(*h->rhs, st, u, dt, s0, s1, hook, *h->pool);
    to_dd(u, u_dd);
    stats[0] = rs.steps_done;
    stats[1] = rs.blew_up ? 1 : 0;
    stats[2] = rs.blowup_step;
  });
}

// A production-style run (driver.cpp:22-93 without files): initial data,
// select_dt, steps_for, sample_stride, and advance_steps with the driver's
// observer hook.  Per sample (row of 15): tau, phi, dphi1, dphi2, dphi3, obs
// (state_sample at j_obs), proj (multipole_project of Psi_R, Psi_I at j_obs),
// scri (state_sample at nrho-1); re/im pairs, .hi limbs.  k_obs = ntheta/2,
// j_obs = nearest_rho_index(observer_rho).  stats: steps_done, blew_up,
// blowup_step, n_obs, planned steps.
int ref_run_series(void* hv, int ell, double center, double width, double amplitude,
                   int stepper, double cfl, double tau_end, double cadence,
                   double observer_rho, double* out, long max_rows, long* stats,
                   double* wall) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    InitialDataSpec id;
    id.ell = ell;
    id.center = WorkReal(center);
    id.width = WorkReal(width);
    id.amplitude = WorkReal(amplitude);
    StateVec u = initial_data(h->g, h->cs, h->p, id);
    StepperSpec st;
    st.kind = stepper == 0 ? StepperSpec::ssprk33 : StepperSpec::ssprk104;
    st.cfl = WorkReal(cfl);
    WorkReal dt = select_dt(h->g, h->cs, st);
    const long steps = steps_for(dt, tau_end);
    const FieldLayout& lay = h->rhs->layout();
    const int kobs = h->g.ntheta / 2;
    long jobs = std::lround((observer_rho - h->g.rho_min.hi) / h->g.drho.hi);
    jobs = std::max(0L, std::min(jobs, long(h->g.nrho - 1)));
    HorizonSampler hs(h->g, h->p, lay, kobs);
    long n = 0;
    SampleHook hook;
    hook.every = sample_stride(dt, cadence);
    hook.fn = [&](long, const WorkReal& tau, const StateVec& s) {
      if (n >= max_rows) return;
      double* r = out + 15 * n;
      HorizonObservables ob = hs.sample(s);
      CxW o = state_sample(s, lay, int(jobs), kobs);
      CxW sc = state_sample(s, lay, lay.nrho - 1, kobs);
      r[0] = tau.hi;
      r[1] = ob.phi.re.hi; r[2] = ob.phi.im.hi;
      for (int d = 0; d < 3; ++d) { r[3 + 2 * d] = ob.dphi[d].re.hi; r[4 + 2 * d] = ob.dphi[d].im.hi; }
      r[9] = o.re.hi; r[10] = o.im.hi;
      if (h->p.mmode == 0) {
        r[11] = multipole_project(theta_slice(s, lay, 0, int(jobs)), h->p.spin, 0, ell).hi;
        r[12] = multipole_project(theta_slice(s, lay, 1, int(jobs)), h->p.spin, 0, ell).hi;
      } else {
        r[11] = r[12] = 0.0;
      }
      r[13] = sc.re.hi; r[14] = sc.im.hi;
      ++n;
    };
    RunStats rs = advance_steps(*h->rhs, st, u, dt, 0, steps, hook, *h->pool);
    stats[0] = rs.steps_done;
    stats[1] = rs.blew_up ? 1 : 0;
    stats[2] = rs.blowup_step;
    stats[3] = n;
    stats[4] = steps;
    if (wall) *wall = rs.wall_seconds;
  });
}

// execute_run's setup from an INI text (parse_config_text, io.cpp), then the
// same observer hook as ref_run_series.  workers overrides [parallel].
int ref_run_config(const char* ini, int workers, double* out, long max_rows, long* stats,
                   double* wall, double* dt_out) {
  return guarded([&] {
    RunConfig cfg = parse_config_text(ini, "inline");
    auto h = std::make_unique<RefHandle>();
    h->p = cfg.phys;
    h->g = make_grid(cfg.nrho, cfg.ntheta, h->p);
    // the unmodified assemble_coefficients, serial or (workers > 1) on theta-row
    // sub-grids from `workers` threads — bitwise the same planes
    h->cs = workers > 1 ? hweno_gpu::assemble_coefficients_parallel(h->g, h->p, workers)
                        : assemble_coefficients(h->g, h->p);
    h->spec = cfg.scheme;
    h->pool = std::make_unique<WorkerPool>(workers > 0 ? workers : cfg.workers);
    h->rhs = std::make_unique<EvolutionRhs>(h->g, h->cs, h->p, h->spec, *h->pool);
    StateVec u = initial_data(h->g, h->cs, h->p, cfg.init);
    WorkReal dt = select_dt(h->g, h->cs, cfg.stepper);
    const long steps = steps_for(dt, cfg.tau_end);
    const FieldLayout& lay = h->rhs->layout();
    const int kobs = cfg.ntheta / 2;
    long jobs = std::lround((to_double(cfg.output.observer_rho) - h->g.rho_min.hi) / h->g.drho.hi);
    jobs = std::max(0L, std::min(jobs, long(h->g.nrho - 1)));
    HorizonSampler hs(h->g, h->p, lay, kobs);
    long n = 0;
    SampleHook hook;
    hook.every = sample_stride(dt, cfg.output.series_cadence);
    hook.fn = [&](long, const WorkReal& tau, const StateVec& s) {
      if (n >= max_rows) return;
      double* r = out + 15 * n;
      HorizonObservables ob = hs.sample(s);
      CxW o = state_sample(s, lay, int(jobs), kobs);
      CxW sc = state_sample(s, lay, lay.nrho - 1, kobs);
      r[0] = tau.hi;
      r[1] = ob.phi.re.hi; r[2] = ob.phi.im.hi;
      for (int d = 0; d < 3; ++d) { r[3 + 2 * d] = ob.dphi[d].re.hi; r[4 + 2 * d] = ob.dphi[d].im.hi; }
      r[9] = o.re.hi; r[10] = o.im.hi;
      if (h->p.mmode == 0) {
        r[11] = multipole_project(theta_slice(s, lay, 0, int(jobs)), h->p.spin, 0, cfg.init.ell).hi;
        r[12] = multipole_project(theta_slice(s, lay, 1, int(jobs)), h->p.spin, 0, cfg.init.ell).hi;
      } else {
        r[11] = r[12] = 0.0;
      }
      r[13] = sc.re.hi; r[14] = sc.im.hi;
      ++n;
    };
    RunStats rs = advance_steps(*h->rhs, cfg.stepper, u, dt, 0, steps, hook, *h->pool);
    stats[0] = rs.steps_done;
    stats[1] = rs.blew_up ? 1 : 0;
    stats[2] = rs.blowup_step;
    stats[3] = n;
    stats[4] = steps;
    if (wall) *wall = rs.wall_seconds;
    dt_out[0] = dt.hi;
    dt_out[1] = dt.lo;
  });
}

// HorizonSampler weights for row ktheta, extracted through the sampler's
// public sample() with unit states (so they are exactly the reference's):
// w[d*8 + i] multiplies Psi(j0 + i) for derivative order d (widths 5..8;
// unused tail entries are 0).  *j0 = base index.
int ref_horizon_weights(void* hv, int ktheta, int* j0, double* w) {
  auto* h = static_cast<RefHandle*>(hv);
  return guarded([&] {
    const FieldLayout& lay = h->rhs->layout();
    HorizonSampler hs(h->g, h->p, lay, ktheta);
    *j0 = hs.base_index();
    StateVec u(lay.size());
    for (int i = 0; i < 8; ++i) {
      std::fill(u.begin(), u.end(), WorkReal(0));
      u[lay.at(0, *j0 + i, ktheta)] = WorkReal(1);
      HorizonObservables ob = hs.sample(u);
      w[0 * 8 + i] = ob.phi.re.hi;
      for (int d = 0; d < 3; ++d) w[(d + 1) * 8 + i] = ob.dphi[d].re.hi;
    }
  });
}

// Linear weights of multipole_project over a staggered theta slice of
// length ntheta (projection of the unit slices e_k).
int ref_projection_weights(int ntheta, int spin, int mmode, int ell,
                           double* w) {
  return guarded([&] {
    std::vector<WorkReal> slice(ntheta);
    for (int k = 0; k < ntheta; ++k) {
      std::fill(slice.begin(), slice.end(), WorkReal(0));
      slice[k] = WorkReal(1);
      w[k] = multipole_project(slice, spin, mmode, ell).hi;
    }
  });
}

int ref_multipole_project(const double* slice_hi, int ntheta, int spin,
                          int mmode, int ell, double* out) {
  return guarded([&] {
    std::vector<WorkReal> slice(ntheta);
    for (int k = 0; k < ntheta; ++k) slice[k] = WorkReal(slice_hi[k]);
    *out = multipole_project(slice, spin, mmode, ell).hi;
  });
}

// Row-level stencil KATs (proj/include/hweno/spatial.hpp): one weno5 row
// derivative in full (mode 0) or mixed (mode 1) precision.  u_dd holds
// n + 8 values (4 ghosts each side).
int ref_weno5_row(const double* u_dd, int n, double drho, double eps,
                  int mode, int minus, double* du_dd) {
  return guarded([&] {
    StateVec u = from_dd(u_dd, size_t(n) + 8);
    StateVec du(n);
    if (mode == 0)
      weno5_row_derivative<WorkReal>(u.data() + 4, n, WorkReal(drho),
                                     WorkReal(eps), minus != 0, du.data());
    else
      weno5_row_derivative<WeightReal>(u.data() + 4, n, WorkReal(drho), eps,
                                       minus != 0, du.data());
    to_dd(du, du_dd);
  });
}

// weno5 weights (proj/include/hweno/spatial.hpp:29-65), mode 0 DD / 1 fp64
int ref_weno5_weights(const double* a5, double eps, int mode, double* w3) {
  return guarded([&] {
    WorkReal a[5];
    for (int i = 0; i < 5; ++i) a[i] = WorkReal(a5[i]);
    if (mode == 0) {
      WorkReal w[3];
      weno5_weights_t<WorkReal>(a[0], a[1], a[2], a[3], a[4], WorkReal(eps),
                                w);
      for (int i = 0; i < 3; ++i) w3[i] = w[i].hi;
    } else {
      double w[3];
      weno5_weights_t<WeightReal>(a[0], a[1], a[2], a[3], a[4], eps, w);
      for (int i = 0; i < 3; ++i) w3[i] = w[i];
    }
  });
}

int ref_nthreads_hint(void) { return (int)std::thread::hardware_concurrency(); }

}  // extern "C"
