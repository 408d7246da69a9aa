// FP64 / FP32 pipe peaks of this B200 (the double-double tiers
// need a compute roofline, MEASURED_PEAKS.json has only HBM and bf16).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/fp_peaks tools/fp_peaks.cu
//   tools/_build/fp_peaks > profiles/<round>_fp_peaks.json
//
// Throughput kernels: every thread runs NCH independent dependency chains of
// one instruction (DFMA, DADD, DMUL, FFMA, packed FFMA2), enough resident
// warps to cover the pipe latency, grid = 148 SMs x blocks per SM; timed
// with CUDA events over several launches after warm-up.  Latency kernels:
// one chain, one warp.  Reported as instructions/s (warp-instructions x 32
// lanes) and, for the FMAs, FLOP/s (2 per lane).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));               \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

constexpr int NCH = 8;
constexpr int ITERS = 4096;

template <int OP>
__global__ void k_f64(double* out, double s) {
  double a[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = s + threadIdx.x * 1e-9 + c;
  const double m = 0.999999, q = 1e-7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (OP == 0) a[c] = fma(a[c], m, q);
      else if (OP == 1) a[c] = a[c] + q;
      else a[c] = a[c] * m;
    }
  }
  double r = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) r += a[c];
  if (r == 12345.678) out[0] = r;  // never true: keeps the chains live
}

template <int OP>
__global__ void k_f32(float* out, float s) {
  float a[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = s + threadIdx.x * 1e-6f + c;
  const float m = 0.9999f, q = 1e-4f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) a[c] = fmaf(a[c], m, q);
  }
  float r = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) r += a[c];
  if (r == 12345.678f) out[0] = r;
}

__global__ void k_f32x2(float* out, float s) {
  float2 a[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = make_float2(s + threadIdx.x * 1e-6f + c, s - c);
  const float2 m = make_float2(0.9999f, 0.9998f), q = make_float2(1e-4f, 2e-4f);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) a[c] = __ffma2_rn(a[c], m, q);
  }
  float r = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) r += a[c].x + a[c].y;
  if (r == 12345.678f) out[0] = r;
}

// latency: one dependent DFMA chain
__global__ void k_lat64(double* out, double s, long long* cyc) {
  double a = s;
  const double m = 0.999999, q = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) a = fma(a, m, q);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (a == 12345.678) out[0] = a;
}

template <class K, class... Args>
float time_kernel(K k, int blocks, int threads, Args... args) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<<<blocks, threads>>>(args...);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) k<<<blocks, threads>>>(args...);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms / reps;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* d64;
  float* d32;
  long long* dc;
  CK(cudaMalloc(&d64, 64));
  CK(cudaMalloc(&d32, 64));
  CK(cudaMalloc(&dc, 64));
  const int threads = 256, bps = 8;  // 64 warps per SM
  const int blocks = nsm * bps;
  const double lanes = (double)blocks * threads;
  const double ops = lanes * ITERS * NCH;  // per-lane instructions
  std::printf("{\"device_sms\": %d, \"clock_khz_attr\": %d, \"threads\": %d, \"blocks\": %d,\n", nsm,
              clk, threads, blocks);
  const char* names64[3] = {"dfma", "dadd", "dmul"};
  float t;
  t = time_kernel(k_f64<0>, blocks, threads, d64, 1.0);
  std::printf(" \"%s\": {\"ms\": %.4f, \"lane_ops_per_s\": %.4e, \"tflops\": %.3f},\n", names64[0], t,
              ops / (t * 1e-3), 2 * ops / (t * 1e-3) / 1e12);
  t = time_kernel(k_f64<1>, blocks, threads, d64, 1.0);
  std::printf(" \"%s\": {\"ms\": %.4f, \"lane_ops_per_s\": %.4e},\n", names64[1], t, ops / (t * 1e-3));
  t = time_kernel(k_f64<2>, blocks, threads, d64, 1.0);
  std::printf(" \"%s\": {\"ms\": %.4f, \"lane_ops_per_s\": %.4e},\n", names64[2], t, ops / (t * 1e-3));
  t = time_kernel(k_f32<0>, blocks, threads, d32, 1.0f);
  std::printf(" \"ffma\": {\"ms\": %.4f, \"lane_ops_per_s\": %.4e, \"tflops\": %.3f},\n", t,
              ops / (t * 1e-3), 2 * ops / (t * 1e-3) / 1e12);
  t = time_kernel(k_f32x2, blocks, threads, d32, 1.0f);
  std::printf(" \"ffma2\": {\"ms\": %.4f, \"lane_ops_per_s\": %.4e, \"tflops\": %.3f},\n", t,
              ops / (t * 1e-3), 4 * ops / (t * 1e-3) / 1e12);
  k_lat64<<<1, 32>>>(d64, 1.0, dc);
  CK(cudaDeviceSynchronize());
  long long cyc = 0;
  CK(cudaMemcpy(&cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost));
  std::printf(" \"dfma_latency_cycles\": %.2f,\n", (double)cyc / ITERS);
  std::printf(" \"note\": \"%d independent chains per lane, %d warps per SM; lane_ops = warp instructions x 32\"}\n",
              NCH, threads / 32 * bps);
  return 0;
}
