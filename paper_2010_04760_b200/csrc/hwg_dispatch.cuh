// Compile-time dispatch (scheme, mode, epilogue) -> kernel instantiation,
// shared by the two stage translation units.
#pragma once

#include <type_traits>

#include "hwg_kernels.cuh"

namespace hwg {

template <template <int, int, int> class L, int SCH, int MODE, class Args>
void dispatch_epi(const Args& a, int epi, int blocks, int wpb, cudaStream_t st) {
  switch (epi) {
    case EPI_RHS: L<SCH, MODE, EPI_RHS>::run(a, blocks, wpb, st); break;
    case EPI_AXPY: L<SCH, MODE, EPI_AXPY>::run(a, blocks, wpb, st); break;
    case EPI_RK3: L<SCH, MODE, EPI_RK3>::run(a, blocks, wpb, st); break;
    case EPI_RK3C: L<SCH, MODE, EPI_RK3C>::run(a, blocks, wpb, st); break;
    case EPI_RK104_5: L<SCH, MODE, EPI_RK104_5>::run(a, blocks, wpb, st); break;
    default: L<SCH, MODE, EPI_RK104_10>::run(a, blocks, wpb, st); break;
  }
}

template <template <int, int, int> class L, class Args>
void dispatch(const Args& a, int scheme, int mode, int epi, int blocks, int wpb,
              cudaStream_t st) {
  auto by_mode = [&](auto sch) {
    constexpr int SCH = decltype(sch)::value;
    if constexpr (SCH == FD6KO) {
      dispatch_epi<L, SCH, F64>(a, epi, blocks, wpb, st);  // no weights
    } else {
      if (mode == MIXED) dispatch_epi<L, SCH, MIXED>(a, epi, blocks, wpb, st);
      else if (mode == LIN) dispatch_epi<L, SCH, LIN>(a, epi, blocks, wpb, st);
      else dispatch_epi<L, SCH, F64>(a, epi, blocks, wpb, st);
    }
  };
  if (scheme == WENO5) by_mode(std::integral_constant<int, WENO5>{});
  else if (scheme == WENO3) by_mode(std::integral_constant<int, WENO3>{});
  else by_mode(std::integral_constant<int, FD6KO>{});
}

// call L<SCH, MODE, EPI>::attr() for every instantiation dispatch() can reach
template <template <int, int, int> class L, int SCH, int MODE>
void attr_epi() {
  L<SCH, MODE, EPI_RHS>::attr(); L<SCH, MODE, EPI_AXPY>::attr(); L<SCH, MODE, EPI_RK3>::attr();
  L<SCH, MODE, EPI_RK3C>::attr(); L<SCH, MODE, EPI_RK104_5>::attr();
  L<SCH, MODE, EPI_RK104_10>::attr();
}
template <template <int, int, int> class L>
void attr_all() {
  attr_epi<L, WENO5, F64>(); attr_epi<L, WENO5, MIXED>(); attr_epi<L, WENO5, LIN>();
  attr_epi<L, WENO3, F64>(); attr_epi<L, WENO3, MIXED>(); attr_epi<L, WENO3, LIN>();
  attr_epi<L, FD6KO, F64>();
}

}  // namespace hwg
