// Double-double instantiations of hwg::stage_kernel_dd (reference-exact tiers).
#include "hwg_dispatch.cuh"
#include "hwg_launch.h"

namespace hwg {
namespace {
template <int SCH, int MODE, int EPI>
struct DDLauncher {
  static void attr() {
    cudaFuncSetAttribute(stage_kernel_dd<SCH, MODE, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)stage_smem_bytes_dd<EPI>());
  }
  static void run(const StageArgsDD& a, int blocks, int wpb, cudaStream_t st) {
    stage_kernel_dd<SCH, MODE, EPI><<<blocks, wpb * 32, stage_smem_bytes_dd<EPI>(wpb), st>>>(a);
  }
};
}  // namespace

void launch_stage_dd(const StageArgsDD& a, int scheme, int mode, int epi, int blocks,
                     int wpb, cudaStream_t stream) {
  dispatch<DDLauncher>(a, scheme, mode, epi, blocks, wpb, stream);
}

void init_attributes_dd() {
  static bool done = [] {
    attr_all<DDLauncher>();
    return true;
  }();
  (void)done;
}

cudaError_t occupancy_dd(int* occ) {
  init_attributes_dd();
  cudaError_t e = cudaFuncSetAttribute(stage_kernel_dd<WENO5, F64, EPI_RK3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)stage_smem_bytes_dd<EPI_RK3>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stage_kernel_dd<WENO5, F64, EPI_RK3>,
                                                       kWarpsPerBlock * 32,
                                                       stage_smem_bytes_dd<EPI_RK3>());
}
}  // namespace hwg
