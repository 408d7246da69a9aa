// fp64 / mixed / linear instantiations of hwg::stage_kernel.
#include "hwg_dispatch.cuh"
#include "hwg_launch.h"

namespace hwg {
namespace {
template <int SCH, int MODE, int EPI>
struct FastLauncher {
  static void run(const StageArgs& a, int blocks, cudaStream_t st) {
    static bool attr = [] {
      cudaFuncSetAttribute(stage_kernel<SCH, MODE, EPI>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)stage_smem_bytes<EPI>());
      return true;
    }();
    (void)attr;
    stage_kernel<SCH, MODE, EPI><<<blocks, kWarpsPerBlock * 32, stage_smem_bytes<EPI>(), st>>>(a);
  }
};
}  // namespace

void launch_stage_fast(const StageArgs& a, int scheme, int mode, int epi, int blocks,
                       cudaStream_t stream) {
  dispatch<FastLauncher>(a, scheme, mode, epi, blocks, stream);
}

cudaError_t occupancy_fast(int* occ) {
  cudaError_t e = cudaFuncSetAttribute(stage_kernel<WENO5, F64, EPI_RK3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)stage_smem_bytes<EPI_RK3>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stage_kernel<WENO5, F64, EPI_RK3>,
                                                       kWarpsPerBlock * 32,
                                                       stage_smem_bytes<EPI_RK3>());
}
}  // namespace hwg
