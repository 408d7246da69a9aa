// Achievable FP64-pipe rate of double-double code on this B200: the DD
// tiers' dominant routine (one WENO5 interface component in the reference's
// DDReal operations, hwg_dd.cuh weno5_dd — 446 FP64 instructions in the
// mixed mode, 1288 in the full mode, cuobjdump of this build) run in
// isolation, register-resident, at several occupancies (8 / 12 / 16 warps
// per SM via __launch_bounds__) and with 1 or 2 independent interface chains
// per thread (ILP), plus plain dd + dd and dd * dd chains.  Reported as FP64
// lane-operations/s and as a fraction of the measured DFMA peak
// (profiles/r02_fp_peaks.json, 1.8139e13): the ceiling the stage kernel's
// "fraction of the FP64 pipe" is to be read against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -I paper_2010_04760_b200/csrc -o tools/_build/dd_peak tools/dd_peak.cu
//   tools/_build/dd_peak > profiles/<round>_dd_peak.json
#include <cuda_runtime.h>

#include <cstdio>

#include "hwg_dd.cuh"

using namespace hwg;

constexpr double kPeak = 1.8139e13;  // measured DFMA lane-ops/s (r02_fp_peaks.json)

template <int MODE, int NCH, int MINB>
__global__ void __launch_bounds__(128, MINB) k_iface(dd* out, const DDConsts* Kp, double eps,
                                                     int iters) {
  const DDConsts K = *Kp;
  dd x[NCH][5];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int m = 0; m < 5; ++m)
      x[c][m] = {1.0 + 0.01 * m * m + 1e-6 * (threadIdx.x + c), 1e-18 * m};
  bool ok = true;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const dd r = weno5_dd<MODE, true>(x[c][0], x[c][1], x[c][2], x[c][3], x[c][4], K, eps, ok);
      x[c][0] = x[c][1]; x[c][1] = x[c][2]; x[c][2] = x[c][3]; x[c][3] = x[c][4];
      x[c][4] = r;
    }
  }
  double s = ok ? 0.0 : 1.0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += x[c][4].hi;
  if (s == 12345.678) out[0] = x[0][4];
}

// plain chains: acc = acc + y (dd + dd, 20 DADD) or acc = acc * y (dd * dd, 9)
template <int OP, int NCH>
__global__ void __launch_bounds__(128, 4) k_chain(dd* out, int iters) {
  dd a[NCH];
  const dd y = {OP == 0 ? 1e-3 : 0.9999999, 1e-20};
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = {1.0 + c + 1e-6 * threadIdx.x, 0.0};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < NCH; ++c) a[c] = OP == 0 ? a[c] + y : a[c] * y;
  double s = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += a[c].hi;
  if (s == 12345.678) out[0] = a[0];
}

template <class F>
float time_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) launch();
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  dd* out;
  DDConsts* Kd;
  cudaMalloc(&out, 64);
  cudaMalloc(&Kd, sizeof(DDConsts));
  DDConsts K{};
  K.c1312 = {13.0 / 12.0, 0.0};
  K.d0 = {0.1, 0.0}; K.d1 = {0.6, 0.0}; K.d2 = {0.3, 0.0};
  K.one = {1.0, 0.0};
  K.sixth = {1.0 / 6.0, 9.25185853854297e-18};
  K.eps = {1e-6, 0.0};
  cudaMemcpy(Kd, &K, sizeof K, cudaMemcpyHostToDevice);
  std::printf("{\"source\": \"tools/dd_peak.cu\", \"dfma_peak_lane_ops\": %.4e,\n \"runs\": [\n", kPeak);
  bool first = true;
  auto report = [&](const char* name, int warps_per_sm, int nch, double fp64_per_unit,
                    double units_per_thread, float ms, int threads) {
    const double lane_ops = fp64_per_unit * units_per_thread * threads / (ms * 1e-3);
    std::printf("%s  {\"kernel\": \"%s\", \"warps_per_sm\": %d, \"chains_per_thread\": %d, "
                "\"ms\": %.3f, \"fp64_lane_ops_per_s\": %.4e, \"frac_of_dfma_peak\": %.3f}",
                first ? " " : ",\n ", name, warps_per_sm, nch, ms, lane_ops, lane_ops / kPeak);
    first = false;
  };
  const int iters = 2000;
#define IFACE(MODE, OPS, NCH, MINB)                                                        \
  {                                                                                        \
    const int blocks = nsm * MINB, threads = blocks * 128;                                 \
    const float ms = time_ms([&] { k_iface<MODE, NCH, MINB><<<blocks, 128>>>(out, Kd, 1e-6, iters); }); \
    report(MODE == MIXED ? "weno5_dd mixed" : "weno5_dd full", MINB * 4, NCH, OPS, (double)iters * NCH, \
           ms, threads);                                                                   \
  }
  IFACE(MIXED, 446, 1, 2) IFACE(MIXED, 446, 1, 3) IFACE(MIXED, 446, 1, 4)
  IFACE(MIXED, 446, 2, 2) IFACE(MIXED, 446, 2, 3) IFACE(MIXED, 446, 2, 4)
  IFACE(F64, 1288, 1, 2) IFACE(F64, 1288, 1, 3) IFACE(F64, 1288, 2, 2)
#define CHAIN(OP, OPS, NCH)                                                                \
  {                                                                                        \
    const int blocks = nsm * 4, threads = blocks * 128;                                    \
    const float ms = time_ms([&] { k_chain<OP, NCH><<<blocks, 128>>>(out, iters * 8); });  \
    report(OP == 0 ? "dd+dd chain" : "dd*dd chain", 16, NCH, OPS, (double)iters * 8 * NCH, ms, threads); \
  }
  CHAIN(0, 20, 1) CHAIN(0, 20, 2) CHAIN(0, 20, 4) CHAIN(1, 9, 1) CHAIN(1, 9, 2) CHAIN(1, 9, 4)
  std::printf("\n]}\n");
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
