// hweno_gpu_dropin.hpp — header-only C++ drop-in for the reference solver.
//
// A reference maintainer includes this next to the reference's own headers
// (proj/include/hweno/*.hpp) and links libhwgpu.so.  It keeps the reference's
// types and call shapes, so driver code (proj/src/driver.cpp:22-137,
// proj/tools/main.cpp:168-221) changes only in the two lines that construct
// the RHS and call the time loop:
//
//   hweno::EvolutionRhs rhs(g, cs, p, spec, pool);            // reference
//   hweno_gpu::GpuEvolutionRhs rhs(g, cs, p, spec);           // GPU
//
//   advance_steps(rhs, stepper, u, dt, 0, n, hook, pool);      // reference
//   hweno_gpu::advance_steps(rhs, stepper, u, dt, 0, n, hook); // GPU
//
// Semantics follow proj/src/evolve.cpp:10-265: operator() fills u's ghosts and
// writes du's interior; advance_steps fires the hook at s % every == 0, at the
// first and at the last step (with tau = s * dt in double-double), stops at
// the first inadmissible state and reports RunStats.  Errors surface as the
// reference's exception types.
//
// Precision: Tier::exact (default) runs the double-double GPU tiers, which
// reproduce the reference's full / mixed modes BIT FOR BIT (SchemeSpec::mode
// full -> HWG_DD_FULL, mixed -> HWG_DD_MIXED).  Tier::fast runs one tier
// below: full -> HWG_F64, mixed -> HWG_MIXED (fp32 weights),
// ~10-20x faster and within 1e-12 / 1e-6 of the reference.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hweno/evolve.hpp"
#include "hweno/geometry.hpp"
#include "hweno/timestep.hpp"
#include "hweno_gpu.h"
#include "hweno_gpu_setup.hpp"

namespace hweno_gpu {

inline void check(int rc, const hwg_solver* s) {
  if (rc == HWG_OK) return;
  std::string msg = hwg_last_error(s);
  if (rc == HWG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

enum class Tier { exact, fast };

// assemble_coefficients (proj/src/geometry.cpp:118-168) on the GPU
// (SURVEY.md §8f-2): every CoefficientSet plane and max_speed bitwise equal to
// the reference's serial loop (hwg_assemble_coefficients evaluates the
// reference's own generated wave_op_coeffs<DDReal> in double-double, one
// thread per point); cotth is the reference's host loop (geometry.cpp:
// 131-132).  The hyperbolicity error is the reference's runtime_error.
//
//   hweno::CoefficientSet cs = assemble_coefficients(g, p);                // reference
//   hweno::CoefficientSet cs = hweno_gpu::assemble_coefficients_device(g, p);  // GPU
inline hweno::CoefficientSet assemble_coefficients_device(const hweno::Grid& g,
                                                          const hweno::PhysicalParams& p,
                                                          int device = 0) {
  using hweno::WorkReal;
  static_assert(sizeof(WorkReal) == 2 * sizeof(double), "DDReal is {double hi, lo}");
  hweno::CoefficientSet c;
  c.nrho = g.nrho;
  c.ntheta = g.ntheta;
  const size_t n = size_t(g.nrho) * g.ntheta;
  std::vector<WorkReal>* planes[14] = {&c.b,     &c.lam,   &c.w_re,  &c.w_im,  &c.bt_re,
                                       &c.bt_im, &c.c_re,  &c.c_im,  &c.ath,   &c.p_mix,
                                       &c.r_rad, &c.br_re, &c.br_im, &c.bprime};
  double* out[14];
  for (int q = 0; q < 14; ++q) {
    planes[q]->resize(n);
    out[q] = reinterpret_cast<double*>(planes[q]->data());
  }
  c.cotth.resize(g.ntheta);
  for (int k = 0; k < g.ntheta; ++k) c.cotth[k] = g.costh[k] / g.sinth[k];
  const double M[2] = {p.M.hi, p.M.lo}, a[2] = {p.a.hi, p.a.lo}, S[2] = {p.S.hi, p.S.lo};
  double vmax[2];
  int bad[2];
  const int rc = hwg_assemble_coefficients(
      device, reinterpret_cast<const double*>(g.rho.data()), g.nrho,
      reinterpret_cast<const double*>(g.costh.data()), g.ntheta, M, a, S, p.spin, p.mmode, out,
      vmax, bad);
  if (rc == HWG_ERUNTIME && bad[0] >= 0)  // geometry.cpp:146-149, its message
    throw std::runtime_error("hyperbolicity violated at rho=" + std::to_string(g.rho[bad[0]].hi) +
                             " theta=" + std::to_string(g.theta[bad[1]].hi));
  check(rc, nullptr);
  c.max_speed = WorkReal(vmax[0], vmax[1]);
  return c;
}

class GpuEvolutionRhs {
 public:
  GpuEvolutionRhs(const hweno::Grid& g, const hweno::CoefficientSet& cs,
                  const hweno::PhysicalParams& p, const hweno::SchemeSpec& spec,
                  int device = 0, Tier tier = Tier::exact)
      : lay_{g.nrho, g.ntheta}, spec_(spec) {
    const size_t P = size_t(g.nrho) * g.ntheta;
    const std::vector<hweno::WorkReal>* src[9] = {&cs.b,     &cs.lam,   &cs.w_re,
                                                  &cs.w_im,  &cs.bt_re, &cs.bt_im,
                                                  &cs.c_re,  &cs.c_im,  &cs.ath};
    std::vector<double> planes(9 * P), planes_lo(9 * P), cot(g.ntheta), cot_lo(g.ntheta);
    for (int q = 0; q < 9; ++q)
      for (size_t i = 0; i < P; ++i) {
        planes[q * P + i] = (*src[q])[i].hi;
        planes_lo[q * P + i] = (*src[q])[i].lo;
      }
    for (int k = 0; k < g.ntheta; ++k) {
      cot[k] = cs.cotth[k].hi;
      cot_lo[k] = cs.cotth[k].lo;
    }
    hwg_desc d{};
    d.nrho = g.nrho;
    d.ntheta = g.ntheta;
    d.drho = g.drho.hi;
    d.dtheta = g.dtheta.hi;
    d.parity = ((p.mmode + p.spin) % 2 == 0) ? 1 : -1;  // evolve.cpp:18
    d.scheme = spec.scheme == hweno::Scheme::weno5   ? HWG_WENO5
               : spec.scheme == hweno::Scheme::weno3 ? HWG_WENO3
                                                     : HWG_FD6KO;
    const bool full = spec.mode == hweno::PrecisionMode::full;
    if (tier == Tier::exact) d.precision = full ? HWG_DD_FULL : HWG_DD_MIXED;
    else d.precision = full ? HWG_F64 : HWG_MIXED;
    d.eps = spec.eps.hi;
    d.sigma = spec.sigma.hi;
    d.drho_lo = g.drho.lo;
    d.dtheta_lo = g.dtheta.lo;
    d.eps_lo = spec.eps.lo;
    d.sigma_lo = spec.sigma.lo;
    d.device = device;
    d.rho_offset = 0;
    d.nrho_global = g.nrho;
    d.coef_ld = g.nrho;
    d.coef_row0 = 0;
    if (tier == Tier::exact)
      check(hwg_create_dd(&d, planes.data(), planes_lo.data(), cot.data(), cot_lo.data(), &h_),
            nullptr);
    else
      check(hwg_create(&d, planes.data(), cot.data(), &h_), nullptr);
  }
  ~GpuEvolutionRhs() { hwg_destroy(h_); }
  GpuEvolutionRhs(const GpuEvolutionRhs&) = delete;
  GpuEvolutionRhs& operator=(const GpuEvolutionRhs&) = delete;

  // EvolutionRhs::operator() (evolve.hpp:61): DDReal is {double hi, lo}
  void operator()(hweno::StateVec& u, hweno::StateVec& du) {
    check(hwg_rhs_dd(h_, reinterpret_cast<double*>(u.data()),
                     reinterpret_cast<double*>(du.data())),
          h_);
  }

  const hweno::FieldLayout& layout() const { return lay_; }
  const hweno::SchemeSpec& scheme() const { return spec_; }
  hwg_solver* handle() { return h_; }

 private:
  hweno::FieldLayout lay_;
  hweno::SchemeSpec spec_;
  hwg_solver* h_ = nullptr;
};

namespace detail {
struct HookCtx {
  GpuEvolutionRhs* rhs;
  const hweno::SampleHook* hook;
  hweno::StateVec* u;
  std::exception_ptr err;  // thrown by the hook: rethrown once hwg_advance returns
};
inline void trampoline(long long step, double tau_hi, double tau_lo, const hwg_observables*,
                       void* user) noexcept {
  auto* c = static_cast<HookCtx*>(user);
  try {
    // the reference hook sees the full state (driver.cpp:64-91): bring it back
    check(hwg_get_state_dd(c->rhs->handle(), reinterpret_cast<double*>(c->u->data())),
          c->rhs->handle());
    c->hook->fn(long(step), hweno::WorkReal(tau_hi, tau_lo), *c->u);
  } catch (...) {  // no exception crosses the C ABI; stop the run as the reference would
    c->err = std::current_exception();
    hwg_abort_advance(c->rhs->handle());
  }
}
}  // namespace detail

// advance_steps (evolve.hpp:109-112) on the GPU.  u is uploaded once, stays
// on the device for the whole call and is written back at the end (and at
// hook steps, for the hook).
inline hweno::RunStats advance_steps(GpuEvolutionRhs& rhs, const hweno::StepperSpec& stepper,
                                     hweno::StateVec& u, const hweno::WorkReal& dt,
                                     long step_begin, long step_end,
                                     const hweno::SampleHook& hook) {
  hwg_solver* h = rhs.handle();
  check(hwg_set_state_dd(h, reinterpret_cast<const double*>(u.data())), h);
  detail::HookCtx ctx{&rhs, &hook, &u, nullptr};
  hwg_run_stats st{};
  const int kind = stepper.kind == hweno::StepperSpec::ssprk33 ? HWG_SSPRK33 : HWG_SSPRK104;
  const int rc = hwg_advance(h, kind, dt.hi, dt.lo, step_begin, step_end,
                             hook.fn ? hook.every : 1, hook.fn ? detail::trampoline : nullptr,
                             &ctx, &st);
  if (ctx.err) std::rethrow_exception(ctx.err);  // the hook's own exception
  check(rc, h);
  check(hwg_get_state_dd(h, reinterpret_cast<double*>(u.data())), h);
  hweno::RunStats rs;
  rs.steps_done = long(st.steps_done);
  rs.wall_seconds = st.wall_seconds;
  rs.blew_up = st.blew_up != 0;
  rs.blowup_step = long(st.blowup_step);
  return rs;
}

}  // namespace hweno_gpu
