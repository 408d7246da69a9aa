// fp64 / mixed / linear instantiations of hwg::stage_kernel.
#include "hwg_dispatch.cuh"
#include "hwg_launch.h"

namespace hwg {
namespace {
template <int SCH, int MODE, int EPI>
struct FastLauncher {
  static void attr() {
    cudaFuncSetAttribute(stage_kernel<SCH, MODE, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)stage_smem_bytes<EPI>());
  }
  static void run(const StageArgs& a, int blocks, int wpb, cudaStream_t st) {
    if (!a.pdl) {
      stage_kernel<SCH, MODE, EPI><<<blocks, wpb * 32, stage_smem_bytes<EPI>(wpb), st>>>(a);
      return;
    }
    // programmatic dependent launch: this stage's blocks may start (barrier
    // set-up, coefficient prefetch) while the previous stage drains; the
    // kernel waits for the previous grid (griddepcontrol.wait) before it
    // reads any state
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(wpb * 32);
    cfg.dynamicSmemBytes = stage_smem_bytes<EPI>(wpb);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, stage_kernel<SCH, MODE, EPI>, a);
  }
};
}  // namespace

void launch_stage_fast(const StageArgs& a, int scheme, int mode, int epi, int blocks,
                       int wpb, cudaStream_t stream) {
  dispatch<FastLauncher>(a, scheme, mode, epi, blocks, wpb, stream);
}

void init_attributes_fast() {
  static bool done = [] {
    attr_all<FastLauncher>();
    return true;
  }();
  (void)done;
}

template <int MODE>
static cudaError_t occupancy_mode(int* occ) {
  const size_t sm = stage_smem_bytes<EPI_RK3>();
  cudaError_t e = cudaFuncSetAttribute(stage_kernel<WENO5, MODE, EPI_RK3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stage_kernel<WENO5, MODE, EPI_RK3>,
                                                       kWarpsPerBlock * 32, sm);
}

cudaError_t occupancy_fast(int* occ, int mode) {
  init_attributes_fast();
  if (mode == F64) return occupancy_mode<F64>(occ);
  if (mode == MIXED) return occupancy_mode<MIXED>(occ);
  return occupancy_mode<LIN>(occ);
}
}  // namespace hwg
