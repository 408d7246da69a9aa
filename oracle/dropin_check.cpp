// TEST INFRASTRUCTURE ONLY — end-to-end check of the C++ drop-in
// (include/hweno_gpu_dropin.hpp) inside the reference's own setup code.
//
// The reference builds the grid, coefficients and initial data
// (proj/src/geometry.cpp, proj/src/evolve.cpp:189-215) and runs its own
// advance_steps with a driver-style hook (proj/src/driver.cpp:64-80); the same
// driver code then runs hweno_gpu::advance_steps.  Exit 0 iff the final states,
// the hook cadence and the hook's horizon observables agree.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include <chrono>
#include <filesystem>

#include "hweno/diagnostics.hpp"
#include "hweno/evolve.hpp"
#include "hweno/io.hpp"
#include "hweno_gpu_dropin.hpp"

using namespace hweno;

struct Run {
  std::vector<long> steps;
  std::vector<double> charge;  // Aretakis charge dphi[0].re
  StateVec u;
  RunStats st;
};

template <class Rhs, class Adv>
Run drive(Rhs& rhs, const Grid& g, const PhysicalParams& p, StateVec u0, const WorkReal& dt,
          long nsteps, Adv&& adv) {
  Run r;
  HorizonSampler hs(g, p, rhs.layout(), g.ntheta / 2);
  SampleHook hook;
  hook.every = 10;
  hook.fn = [&](long s, const WorkReal&, const StateVec& u) {
    r.steps.push_back(s);
    r.charge.push_back(hs.sample(u).dphi[0].re.hi);
  };
  r.u = u0;
  r.st = adv(rhs, r.u, dt, nsteps, hook);
  return r;
}

int main(int argc, char** argv) {
  int device = argc > 1 ? std::atoi(argv[1]) : 0;
  int bad = 0;
  for (int tier = 0; tier < 2; ++tier)
  for (int mode = 0; mode < 2; ++mode) {
    const bool exact = tier == 0;  // exact: DD tiers, bitwise; fast: fp64/fp32 tiers
    PhysicalParams p;
    p.M = WorkReal(1);
    p.a = WorkReal(0.9);
    p.spin = -2;
    p.mmode = 0;
    p.S = WorkReal(20);
    Grid g = make_grid(256, 16, p);
    CoefficientSet cs = assemble_coefficients(g, p);
    SchemeSpec spec;
    spec.mode = mode == 0 ? PrecisionMode::full : PrecisionMode::mixed;
    InitialDataSpec id;
    id.center = WorkReal(3.0);
    id.width = WorkReal(0.3);
    StateVec u0 = initial_data(g, cs, p, id);
    StepperSpec st;
    st.kind = StepperSpec::ssprk104;
    WorkReal dt = select_dt(g, cs, st);
    const long nsteps = 45;

    WorkerPool pool(4);
    EvolutionRhs ref(g, cs, p, spec, pool);
    Run a = drive(ref, g, p, u0, dt, nsteps,
                  [&](EvolutionRhs& r, StateVec& u, const WorkReal& d, long n,
                      const SampleHook& h) {
                    return advance_steps(r, st, u, d, 0, n, h, pool);
                  });
    hweno_gpu::GpuEvolutionRhs gpu(g, cs, p, spec, device,
                                   exact ? hweno_gpu::Tier::exact : hweno_gpu::Tier::fast);
    Run b = drive(gpu, g, p, u0, dt, nsteps,
                  [&](hweno_gpu::GpuEvolutionRhs& r, StateVec& u, const WorkReal& d, long n,
                      const SampleHook& h) {
                    return hweno_gpu::advance_steps(r, st, u, d, 0, n, h);
                  });
    double num = 0, den = 0;
    long nbits = 0;  // interior values whose hi or lo limb differs
    const FieldLayout& lay = ref.layout();
    for (int c = 0; c < kComponents; ++c)
      for (int k = 0; k < g.ntheta; ++k)
        for (int j = 0; j < g.nrho; ++j) {
          size_t i = lay.at(c, j, k);
          num = std::fmax(num, std::fabs(a.u[i].hi - b.u[i].hi));
          den = std::fmax(den, std::fabs(a.u[i].hi));
          nbits += std::memcmp(&a.u[i], &b.u[i], sizeof(DDReal)) != 0;
        }
    const double tol = exact ? 0.0 : (mode == 0 ? 1e-12 : 1e-6);
    double cerr = 0;
    for (size_t q = 0; q < a.charge.size() && q < b.charge.size(); ++q)
      cerr = std::fmax(cerr, std::fabs(a.charge[q] - b.charge[q]) /
                                 std::fmax(std::fabs(a.charge[q]), 1e-12));
    const bool ok = a.steps == b.steps && b.st.steps_done == nsteps && !b.st.blew_up &&
                    num / den <= tol && (!exact || (nbits == 0 && cerr == 0.0)) &&
                    cerr <= (mode == 0 ? 1e-9 : 1e-4);
    std::printf("%s %s: state rel %.3e (%ld values differ bitwise)  hooks %zu/%zu  charge rel %.3e"
                "  steps %ld  %s\n",
                exact ? "exact" : "fast", mode == 0 ? "full" : "mixed", num / den, nbits,
                a.steps.size(), b.steps.size(), cerr, b.st.steps_done, ok ? "OK" : "FAIL");
    bad += !ok;

    // EvolutionRhs::operator() on the same state
    StateVec u1 = u0, u2 = u0, d1(lay.size()), d2(lay.size());
    ref(u1, d1);
    gpu(u2, d2);
    double rn = 0, rd = 0, gh = 0;
    for (size_t i = 0; i < lay.size(); ++i) {
      rn = std::fmax(rn, std::fabs(d1[i].hi - d2[i].hi));
      rd = std::fmax(rd, std::fabs(d1[i].hi));
    }
    for (int c = 0; c < kComponents; ++c)
      for (int k = 0; k < g.ntheta; ++k)
        for (int t = 1; t <= kRadialGhost; ++t)
          gh = std::fmax(gh, std::fabs(u1[lay.at(c, -t, k)].hi - u2[lay.at(c, -t, k)].hi));
    const bool ok2 = rn / rd <= (exact ? 0.0 : (mode == 0 ? 1e-13 : 1e-6)) && gh <= 1e-13;
    std::printf("  rhs rel %.3e ghost diff %.3e %s\n", rn / rd, gh, ok2 ? "OK" : "FAIL");
    bad += !ok2;
  }
  // ---- §8f-2: threaded coefficient assembly, bitwise vs the serial reference
  {
    PhysicalParams p;
    p.M = WorkReal(1);
    p.a = WorkReal(1);
    p.spin = -2;
    p.mmode = 2;
    p.S = WorkReal(20);
    Grid g = make_grid(2048, 64, p);
    auto t0 = std::chrono::steady_clock::now();
    CoefficientSet a = assemble_coefficients(g, p);
    auto t1 = std::chrono::steady_clock::now();
    CoefficientSet b = hweno_gpu::assemble_coefficients_parallel(g, p);
    auto t2 = std::chrono::steady_clock::now();
    CoefficientSet d = hweno_gpu::assemble_coefficients_device(g, p);
    auto t3 = std::chrono::steady_clock::now();
    auto ndiff = [&](const CoefficientSet& x) {
      const std::vector<WorkReal>* pa[14] = {&a.b, &a.lam, &a.w_re, &a.w_im, &a.bt_re, &a.bt_im, &a.c_re,
                                             &a.c_im, &a.ath, &a.p_mix, &a.r_rad, &a.br_re, &a.br_im, &a.bprime};
      const std::vector<WorkReal>* pb[14] = {&x.b, &x.lam, &x.w_re, &x.w_im, &x.bt_re, &x.bt_im, &x.c_re,
                                             &x.c_im, &x.ath, &x.p_mix, &x.r_rad, &x.br_re, &x.br_im, &x.bprime};
      long diff = 0;
      for (int q = 0; q < 14; ++q)
        diff += std::memcmp(pa[q]->data(), pb[q]->data(), pa[q]->size() * sizeof(WorkReal)) != 0;
      diff += std::memcmp(a.cotth.data(), x.cotth.data(), a.cotth.size() * sizeof(WorkReal)) != 0;
      diff += std::memcmp(&a.max_speed, &x.max_speed, sizeof(WorkReal)) != 0;
      return diff;
    };
    const long diff = ndiff(b), ddiff = ndiff(d);
    const double ts = std::chrono::duration<double>(t1 - t0).count();
    const double tp = std::chrono::duration<double>(t2 - t1).count();
    const double td = std::chrono::duration<double>(t3 - t2).count();
    std::printf("coefficients 2048x64: serial %.3f s, threaded %.3f s (%.1fx), planes differing %ld %s\n",
                ts, tp, ts / tp, diff, diff == 0 ? "OK" : "FAIL");
    std::printf("coefficients 2048x64 on the GPU: %.3f s (%.1fx serial), planes differing %ld %s\n", td,
                ts / td, ddiff, ddiff == 0 ? "OK" : "FAIL");
    bad += diff != 0;
    bad += ddiff != 0;
  }
  // ---- §8f-3: checkpoint / restart through the GPU state (test_io.cpp:320-360)
  {
    RunConfig c = parse_config_text("[grid]\nnrho = 128\nntheta = 8\n[time]\ntau_end = 2\n", "inline");
    const PhysicalParams& p = c.phys;
    Grid g = make_grid(c.nrho, c.ntheta, p);
    CoefficientSet cs = hweno_gpu::assemble_coefficients_parallel(g, p);
    FieldLayout lay{g.nrho, g.ntheta};
    WorkerPool pool(2);
    WorkReal dt = select_dt(g, cs, c.stepper);
    SampleHook none;
    StateVec unbroken = initial_data(g, cs, p, c.init);
    EvolutionRhs rref(g, cs, p, c.scheme, pool);
    advance_steps(rref, c.stepper, unbroken, dt, 0, 30, none, pool);  // reference, unbroken
    hweno_gpu::GpuEvolutionRhs gA(g, cs, p, c.scheme, device);
    StateVec first = initial_data(g, cs, p, c.init);
    hweno_gpu::advance_steps(gA, c.stepper, first, dt, 0, 15, none);
    const std::string path =
        (std::filesystem::temp_directory_path() / "hwg_dropin_restart.txt").string();
    write_checkpoint(path, c, 15, WorkReal(15) * dt, lay, first);
    Checkpoint cp = read_checkpoint(path, c, lay);
    hweno_gpu::GpuEvolutionRhs gB(g, cs, p, c.scheme, device);
    StateVec resumed = cp.state;
    hweno_gpu::advance_steps(gB, c.stepper, resumed, dt, cp.step, 30, none);
    long mism = 0;
    for (int comp = 0; comp < kComponents; ++comp)
      for (int j = 0; j < g.nrho; ++j)
        for (int k = 0; k < g.ntheta; ++k)
          mism += std::memcmp(&unbroken[lay.at(comp, j, k)], &resumed[lay.at(comp, j, k)],
                              sizeof(WorkReal)) != 0;
    std::printf("checkpoint at step 15 -> GPU restart -> step 30 vs unbroken reference: %ld values differ %s\n",
                mism, mism == 0 ? "OK" : "FAIL");
    bad += mism != 0;
    std::filesystem::remove(path);
  }
  std::printf(bad ? "DROPIN FAIL\n" : "DROPIN OK\n");
  return bad ? 1 : 0;
}
