// Double-double instantiations of hwg::stage_kernel_dd (reference-exact tiers).
#include "hwg_dispatch.cuh"
#include "hwg_launch.h"

namespace hwg {
namespace {
template <int SCH, int MODE, int EPI>
struct DDLauncher {
  // the full tier has no INL instantiation (its interfaces always stay out of line)
  static constexpr bool HAS_INL = MODE != F64;
  static void attr() {
    cudaFuncSetAttribute(stage_kernel_dd<SCH, MODE, EPI, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_smem_bytes_dd<EPI>());
    if constexpr (HAS_INL)
      cudaFuncSetAttribute(stage_kernel_dd<SCH, MODE, EPI, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)stage_smem_bytes_dd<EPI>());
  }
  static void run(const StageArgsDD& a, int blocks, int wpb, cudaStream_t st) {
    if constexpr (HAS_INL) {
      if (a.inl) {
        stage_kernel_dd<SCH, MODE, EPI, true><<<blocks, wpb * 32, stage_smem_bytes_dd<EPI>(wpb), st>>>(a);
        return;
      }
    }
    stage_kernel_dd<SCH, MODE, EPI, false><<<blocks, wpb * 32, stage_smem_bytes_dd<EPI>(wpb), st>>>(a);
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

int dd_warps_per_chunk() { return kDDWarpsPerChunk; }

cudaError_t occupancy_dd(int* occ) {
  init_attributes_dd();
  cudaError_t e = cudaFuncSetAttribute(stage_kernel_dd<WENO5, F64, EPI_RK3, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)stage_smem_bytes_dd<EPI_RK3>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stage_kernel_dd<WENO5, F64, EPI_RK3, false>,
                                                       kWarpsPerBlock * 32,
                                                       stage_smem_bytes_dd<EPI_RK3>());
}
}  // namespace hwg

// ---------------------------------------------------------------------------
// Self-test of the branch-free division (hwg_dd.cuh: rcp_div / div_y) against
// the compiler's IEEE division on n pseudo-random operand pairs: random
// exponents over the whole range (incl. subnormals, zeros, powers of two,
// all-ones mantissas) and the magnitudes the WENO weights produce.  Counts
// pairs where the guard passed but the quotient differs (must be 0) and
// pairs where the guard failed (the exact fallback path).
namespace hwg {
namespace {
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}
__device__ double rand_double(unsigned long long r, unsigned long long r2) {
  const int kind = (int)(r2 % 8);
  unsigned long long mant = r & ((1ull << 52) - 1);
  if (kind == 0) mant = (1ull << 52) - 1;                       // all-ones mantissa
  if (kind == 1) mant = 0;                                       // power of two
  int e;
  if (kind == 2) e = 0;                                          // subnormal / zero
  else if (kind < 6) e = 1023 + (int)((r2 >> 8) % 80) - 40;      // |x| ~ 2^-40 .. 2^40
  else e = 1 + (int)((r2 >> 8) % 2046);                          // any normal exponent
  const unsigned long long sign = (r2 >> 40) & 1ull;
  return __longlong_as_double((long long)((sign << 63) | ((unsigned long long)e << 52) | mant));
}
__global__ void div_selftest_kernel(long long n, unsigned long long seed,
                                    unsigned long long* out) {
  unsigned long long bad = 0, fails = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = mix64(seed ^ (unsigned long long)i * 0x9e3779b97f4a7c15ull);
    const double a = rand_double(mix64(k), mix64(k + 1));
    double b = rand_double(mix64(k + 2), mix64(k + 3));
    if (b == 0.0) b = 1.0;
    bool ok = true;
    const double q = div_y(a, b, rcp_div(b), ok);
    const double ref = a / b;
    if (!ok) ++fails;
    else if (__double_as_longlong(q) != __double_as_longlong(ref) && !(q != q && ref != ref)) ++bad;
  }
  atomicAdd(out, bad);
  atomicAdd(out + 1, fails);
}
}  // namespace

cudaError_t div_selftest(long long n, unsigned long long seed, long long* mismatches,
                         long long* guard_fails) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  div_selftest_kernel<<<148 * 8, 256>>>(n, seed, d);
  unsigned long long h[2] = {0, 0};
  e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  *mismatches = (long long)h[0];
  *guard_fails = (long long)h[1];
  return e;
}
}  // namespace hwg
