// Launchers of the stage-kernel instantiations.  Each tier is compiled in its
// own translation unit (hwg_stage_fast.cu, hwg_stage_dd.cu) so the build
// parallelises; hwg_solver.cu only sees these entry points.
#pragma once

#include <string>

#include "hwg_dd.cuh"
#include "hwg_kernels.cuh"

namespace hwg {
// fp64 / mixed / linear tiers (stage_kernel)
void launch_stage_fast(const StageArgs& a, int scheme, int mode, int epi, int blocks, int wpb,
                       cudaStream_t stream);
// resident blocks per SM of the tier's kernels (they differ by mode); also
// sets every kernel's smem attribute
cudaError_t occupancy_fast(int* blocks_per_sm, int mode);
void init_attributes_fast();
// double-double tiers (stage_kernel_dd)
void launch_stage_dd(const StageArgsDD& a, int scheme, int mode, int epi, int blocks, int wpb,
                     cudaStream_t stream);
cudaError_t occupancy_dd(int* blocks_per_sm);
// warps per 32-column theta chunk of the DD stage kernel (1, or 2 in the
// lane = (column, component) form)
int dd_warps_per_chunk();
// self-test of the DD tier's branch-free division vs IEEE division
cudaError_t div_selftest(long long n, unsigned long long seed, long long* mismatches,
                         long long* guard_fails);
void init_attributes_dd();
// multi-slab emulation of the fused halo push in one cooperative launch
// (hwg_peer_emu.cu): slab k owns blocks [block0, block0 + blocks) and runs
// the stage sequence args[gi % period] (a device array), epilogues epi[]
constexpr int kMaxEmuSlabs = 8;
constexpr int kMaxEmuPeriod = 20;  // two SSP-RK(10,4) steps
struct EmuSlab {
  const StageArgs* args;
  int block0, blocks;
  unsigned long long* bar;  // slab-local stage barrier (monotonic counter)
};
struct EmuArgs {
  int nslabs, nstages, period;
  long long skew_ns;  // odd slabs start every stage this much later (forces waits)
  int epi[kMaxEmuPeriod];
  EmuSlab s[kMaxEmuSlabs];
};
// capacity: co-resident blocks of the emulation kernel on this device
cudaError_t launch_peer_emu(const EmuArgs& m, int scheme, int mode, int blocks,
                            cudaStream_t stream, int* capacity);
// hwg_last_error(NULL) for the handle-less entry points (coefficient assembly)
void set_global_error(const std::string& msg);
}  // namespace hwg
