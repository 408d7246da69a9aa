// Double-double instantiations of hwg::stage_kernel_dd (reference-exact tiers).
#include "hwg_dispatch.cuh"
#include "hwg_launch.h"

namespace hwg {
namespace {
template <int SCH, int MODE, int EPI>
struct DDLauncher {
  static void run(const StageArgsDD& a, int blocks, cudaStream_t st) {
    static bool attr = [] {
      cudaFuncSetAttribute(stage_kernel_dd<SCH, MODE, EPI>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)stage_smem_bytes_dd<EPI>());
      return true;
    }();
    (void)attr;
    stage_kernel_dd<SCH, MODE, EPI><<<blocks, kWarpsPerBlock * 32, stage_smem_bytes_dd<EPI>(),
                                      st>>>(a);
  }
};
}  // namespace

void launch_stage_dd(const StageArgsDD& a, int scheme, int mode, int epi, int blocks,
                     cudaStream_t stream) {
  dispatch<DDLauncher>(a, scheme, mode, epi, blocks, stream);
}

cudaError_t occupancy_dd(int* occ) {
  cudaError_t e = cudaFuncSetAttribute(stage_kernel_dd<WENO5, F64, EPI_RK3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)stage_smem_bytes_dd<EPI_RK3>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stage_kernel_dd<WENO5, F64, EPI_RK3>,
                                                       kWarpsPerBlock * 32,
                                                       stage_smem_bytes_dd<EPI_RK3>());
}
}  // namespace hwg
