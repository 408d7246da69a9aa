// hweno_gpu_setup.hpp — reference-side setup helper (header-only, no GPU
// dependency): the reference's coefficient assembly on host threads.
//
// Included by the drop-in (hweno_gpu_dropin.hpp) and usable on its own next
// to the reference's headers (proj/include/hweno/*.hpp).
#pragma once

#include <algorithm>
#include <atomic>
#include <exception>
#include <thread>
#include <vector>

#include "hweno/geometry.hpp"

namespace hweno_gpu {

// assemble_coefficients (proj/src/geometry.cpp:118-168) off the serial host
// path.  The reference's own, unmodified
// hweno::assemble_coefficients runs on theta-row sub-grids from a pool of
// host threads (rows handed out one at a time by an atomic counter), and the
// rows are scattered into one CoefficientSet.  A sub-grid is the full Grid
// with ntheta = 1 and that row's theta / cos / sin: assemble_coefficients
// evaluates each point from (rho_j, cos theta_k) alone, so every entry is
// bitwise the serial one, and max_speed — an exact max over the same values
// — is the max of the rows' maxima.  The first error in the serial (k, j)
// order is rethrown (rows are evaluated in full; a row's first failing point
// is the serial order's within that row).
inline hweno::CoefficientSet assemble_coefficients_parallel(const hweno::Grid& g,
                                                            const hweno::PhysicalParams& p,
                                                            int threads = 0) {
  using hweno::WorkReal;
  hweno::CoefficientSet out;
  out.nrho = g.nrho;
  out.ntheta = g.ntheta;
  const size_t n = size_t(g.nrho) * g.ntheta;
  using Plane = std::vector<WorkReal> hweno::CoefficientSet::*;
  static constexpr Plane kPlanes[] = {
      &hweno::CoefficientSet::b,     &hweno::CoefficientSet::lam,
      &hweno::CoefficientSet::w_re,  &hweno::CoefficientSet::w_im,
      &hweno::CoefficientSet::bt_re, &hweno::CoefficientSet::bt_im,
      &hweno::CoefficientSet::c_re,  &hweno::CoefficientSet::c_im,
      &hweno::CoefficientSet::ath,   &hweno::CoefficientSet::p_mix,
      &hweno::CoefficientSet::r_rad, &hweno::CoefficientSet::br_re,
      &hweno::CoefficientSet::br_im, &hweno::CoefficientSet::bprime};
  for (Plane m : kPlanes) (out.*m).resize(n);
  out.cotth.resize(g.ntheta);
  std::vector<WorkReal> row_max(g.ntheta, WorkReal(0));
  std::vector<std::exception_ptr> err(g.ntheta);
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  threads = std::max(1, std::min(threads, g.ntheta));
  std::atomic<int> next{0};
  auto worker = [&] {
    hweno::Grid row = g;  // rho data shared by value; theta data replaced per row
    row.ntheta = 1;
    for (int k; (k = next.fetch_add(1)) < g.ntheta;) {
      row.theta.assign(1, g.theta[k]);
      row.costh.assign(1, g.costh[k]);
      row.sinth.assign(1, g.sinth[k]);
      try {
        const hweno::CoefficientSet c = hweno::assemble_coefficients(row, p);
        const size_t o = size_t(g.nrho) * k;
        for (Plane m : kPlanes) std::copy((c.*m).begin(), (c.*m).end(), (out.*m).begin() + o);
        out.cotth[k] = c.cotth[0];
        row_max[k] = c.max_speed;
      } catch (...) {
        err[k] = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  for (int k = 0; k < g.ntheta; ++k)
    if (err[k]) std::rethrow_exception(err[k]);
  WorkReal vmax(0);
  for (int k = 0; k < g.ntheta; ++k)  // the serial loop's comparison order
    if (vmax < row_max[k]) vmax = row_max[k];
  out.max_speed = vmax;
  return out;
}

}  // namespace hweno_gpu
