// Multi-slab emulation of the fused NVLink halo push on ONE GPU
// (validation of the multi-GPU protocol).
//
// On an 8-GPU box every slab's stage kernels run on their own GPU, unordered
// with respect to the neighbours: a boundary warp may spin on its arrival
// counter while the neighbour's kernel is still computing the rows it will
// push.  Separate launches on one GPU cannot reproduce that safely (nothing
// guarantees they are co-resident, B200_PROFILING.md), so this kernel runs
// ALL slabs' stages in ONE cooperative launch (every block resident): the
// blocks of a slab run the slab's stage sequence back to back, separated only
// by a slab-local barrier (what a kernel boundary is on the slab's own GPU);
// between slabs there is no ordering except the production protocol itself
// — the in-kernel pushes into the neighbours' halo rows, their release
// counters and the boundary warps' bounded acquire spins (stage_body,
// hwg_kernels.cuh).  Slabs of different sizes drift apart, so boundary warps
// genuinely wait on counters bumped by concurrently running blocks (with
// skew_ns > 0 the odd slabs also start every stage late, so the even slabs'
// boundary warps must wait); the spins are counted (flag[8], hwg_peer_stats).
#include "hwg_launch.h"

namespace hwg {

// one stage of one slab, epilogue EPI
template <int SCH, int MODE, int EPI>
__device__ __forceinline__ void emu_run(const StageArgs& a, int bid, unsigned long long nw) {
  unsigned char* ring;
  uint32_t bar0;
  double2* trow;
  stage_layout<EPI>(ring, bar0, trow);
  if (!stage_body<SCH, MODE, EPI>(a, ring, bar0, trow, [] {}, bid)) return;  // frozen
  if (a.tick != nullptr)
    launch_ticket(a.tick, a.flag, (a.px.on_lo | a.px.on_hi) ? a.px.epoch : nullptr, nw);
}

template <int SCH, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 1) peer_emu_kernel(const EmuArgs m) {
  int sl = 0;
  while (sl + 1 < m.nslabs && (int)blockIdx.x >= m.s[sl + 1].block0) ++sl;
  const EmuSlab S = m.s[sl];
  const int bid = (int)blockIdx.x - S.block0;
  const unsigned long long nw = (unsigned long long)S.blocks * (blockDim.x >> 5);
  for (int gi = 0; gi < m.nstages; ++gi) {
    if (m.skew_ns > 0 && (sl & 1)) {  // a late neighbour (test knob)
      if (threadIdx.x == 0) {
        const unsigned long long t0 = globaltimer();
        while ((long long)(globaltimer() - t0) < m.skew_ns) __nanosleep(256);
      }
      __syncthreads();
    }
    const StageArgs& a = S.args[gi % m.period];  // device copy (global memory)
    switch (m.epi[gi % m.period]) {
      case EPI_AXPY: emu_run<SCH, MODE, EPI_AXPY>(a, bid, nw); break;
      case EPI_RK3: emu_run<SCH, MODE, EPI_RK3>(a, bid, nw); break;
      case EPI_RK3C: emu_run<SCH, MODE, EPI_RK3C>(a, bid, nw); break;
      case EPI_RK104_5: emu_run<SCH, MODE, EPI_RK104_5>(a, bid, nw); break;
      default: emu_run<SCH, MODE, EPI_RK104_10>(a, bid, nw); break;
    }
    // slab-local barrier: every block of this slab has finished stage gi
    // (and its writes are visible, also to the next stage's bulk copies)
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(S.bar, 1ull);
      const unsigned long long want = (unsigned long long)S.blocks * (unsigned long long)(gi + 1);
      while (ld_acquire_sys(S.bar) < want) __nanosleep(64);
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
}

namespace {
template <int SCH, int MODE>
cudaError_t run_emu(const EmuArgs& m, int blocks, cudaStream_t st, int* capacity) {
  size_t smem = 0;
  for (size_t b : {stage_smem_bytes<EPI_AXPY>(), stage_smem_bytes<EPI_RK3>(),
                   stage_smem_bytes<EPI_RK3C>(), stage_smem_bytes<EPI_RK104_5>(),
                   stage_smem_bytes<EPI_RK104_10>()})
    smem = b > smem ? b : smem;
  cudaError_t e = cudaFuncSetAttribute(peer_emu_kernel<SCH, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0, dev = 0, nsm = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, peer_emu_kernel<SCH, MODE>,
                                                         kWarpsPerBlock * 32, smem)) != cudaSuccess)
    return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  *capacity = occ * nsm;
  if (blocks > *capacity) return cudaErrorCooperativeLaunchTooLarge;
  void* args[] = {const_cast<EmuArgs*>(&m)};
  return cudaLaunchCooperativeKernel((const void*)peer_emu_kernel<SCH, MODE>, dim3(blocks),
                                     dim3(kWarpsPerBlock * 32), args, smem, st);
}
}  // namespace

cudaError_t launch_peer_emu(const EmuArgs& m, int scheme, int mode, int blocks,
                            cudaStream_t stream, int* capacity) {
  if (scheme == WENO5) {
    if (mode == MIXED) return run_emu<WENO5, MIXED>(m, blocks, stream, capacity);
    if (mode == F64) return run_emu<WENO5, F64>(m, blocks, stream, capacity);
  } else if (scheme == FD6KO) {
    return run_emu<FD6KO, F64>(m, blocks, stream, capacity);
  } else if (scheme == WENO3 && mode == MIXED) {
    return run_emu<WENO3, MIXED>(m, blocks, stream, capacity);
  }
  return cudaErrorNotSupported;
}

}  // namespace hwg
