// Host runtime + C ABI of libhwgpu.so (include/hweno_gpu.h).
//
// The handle mirrors EvolutionRhs (proj/src/evolve.cpp:10-38) and the time
// loop advance_steps (evolve.cpp:237-265); the steppers' stage sequences are
// those of ssprk33_step / ssprk104_step (proj/include/hweno/timestep.hpp:54-109)
// with each stage one fused launch of hwg::stage_kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hweno_gpu.h"
#include "hwg_kernels.cuh"

using namespace hwg;

namespace {
thread_local std::string g_create_err;

struct DD {  // minimal double-double for host-side constants (precision.hpp:16-115)
  double hi, lo;
};
inline double two_sum(double a, double b, double& e) {
  double s = a + b, bb = s - a;
  e = (a - (s - bb)) + (b - bb);
  return s;
}
inline double quick_two_sum(double a, double b, double& e) {
  double s = a + b;
  e = b - (s - a);
  return s;
}
inline DD dd_mul(DD a, DD b) {
  double p2;
  double p1 = a.hi * b.hi;
  p2 = std::fma(a.hi, b.hi, -p1);
  p2 += a.hi * b.lo + a.lo * b.hi;
  p1 = quick_two_sum(p1, p2, p2);
  return {p1, p2};
}
inline DD dd_sub(DD a, DD b) {
  double s2, t2;
  double s1 = two_sum(a.hi, -b.hi, s2);
  double t1 = two_sum(a.lo, -b.lo, t2);
  s2 += t1;
  s1 = quick_two_sum(s1, s2, s2);
  s2 += t2;
  s1 = quick_two_sum(s1, s2, s2);
  return {s1, s2};
}
inline DD dd_div(DD a, DD b) {  // precision.hpp operator/
  double q1 = a.hi / b.hi;
  DD r = dd_sub(a, dd_mul(b, {q1, 0.0}));
  double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul(b, {q2, 0.0}));
  double q3 = r.hi / b.hi;
  double s2;
  double s1 = quick_two_sum(q1, q2, s2);
  double e;
  double t = two_sum(s1, q3, e);
  e += s2;
  t = quick_two_sum(t, e, e);
  return {t, e};
}
inline double ddq(double num, double den) { return dd_div({num, 0.0}, {den, 0.0}).hi; }
}  // namespace

struct hwg_solver {
  hwg_desc d{};
  int n = 0, nt = 0, ntp = 0, phys_lo = 1, phys_hi = 1;
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own = nullptr;
  double2* coef = nullptr;   // coefficient blocks (row, chunk) x 144 double2
  double* cot = nullptr;     // cot(theta), padded to nchunks*32
  double2* reg[5] = {};      // state registers, blocked layout incl. halo rows
  int nreg = 0;
  size_t rs = 0;             // double2 per state row (nchunks * 64)
  size_t reg_elems = 0;      // double2 per register ((n + 2 kHalo) * rs)
  int cur = 0, scr1 = 1, scr2 = 2, scr3 = 3, scr4 = 4;
  unsigned long long* flag = nullptr;
  unsigned long long* hflag = nullptr;  // pinned
  int nchunks = 0, nranges = 0, blocks = 0;
  double* stage_dev = nullptr;
  size_t stage_cap = 0;
  // observers
  int kobs = -1, j0 = -1, jobs = -1;
  double* obs_w = nullptr;   // 32 horizon weights + ntheta projection weights
  double* obs_dev = nullptr; // 14 outputs
  double* obs_host = nullptr;
  std::string err;
};

#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      s->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return HWG_ECUDA;                                                        \
    }                                                                          \
  } while (0)

// ----------------------------------------------------------------------------
// kernels declared in hwg_kernels.cuh
namespace hwg {

__global__ void relayout_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                double2* reg, int n, int nt, int nchunks, int stride, int dir) {
  // reg points at row 0 of a blocked state register
  __shared__ double tile[4][32][33];
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const size_t W = (size_t)n + 8, Hh = (size_t)nt + 4, P = W * Hh;
  const size_t rs = (size_t)nchunks * kStateBlk;
  if (dir == 0) {
    for (int kk = ty; kk < 32; kk += 8) {
      const int k = k0 + kk, j = j0 + tx;
      if (k < nt && j < n)
        for (int c = 0; c < 4; ++c)
          tile[c][kk][tx] = src[(c * P + (size_t)(k + 2) * W + (j + 4)) * stride];
    }
    __syncthreads();
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj, k = k0 + tx;
      if (k < nt && j < n) {
        double2* b = reg + j * rs + (size_t)(k >> 5) * kStateBlk + (k & 31);
        b[0] = make_double2(tile[0][tx][jj], tile[1][tx][jj]);
        b[32] = make_double2(tile[2][tx][jj], tile[3][tx][jj]);
      }
    }
  } else {
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj, k = k0 + tx;
      if (k < nt && j < n) {
        const double2* b = reg + j * rs + (size_t)(k >> 5) * kStateBlk + (k & 31);
        double2 u = b[0], v = b[32];
        tile[0][tx][jj] = u.x; tile[1][tx][jj] = u.y;
        tile[2][tx][jj] = v.x; tile[3][tx][jj] = v.y;
      }
    }
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {
      const int k = k0 + kk, j = j0 + tx;
      if (k < nt && j < n)
        for (int c = 0; c < 4; ++c) {
          const size_t o = (c * P + (size_t)(k + 2) * W + (j + 4)) * stride;
          dst[o] = tile[c][kk][tx];
          if (stride == 2) dst[o + 1] = 0.0;
        }
    }
  }
}

// coefficient plane q (index j + ld*k, rows row0..) -> blocked coefficient member
__global__ void coef_kernel(const double* __restrict__ src, int ld, int row0, double* coef,
                            int q, int n, int nt, int nchunks) {
  __shared__ double tile[32][33];
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int kk = ty; kk < 32; kk += 8) {
    const int k = k0 + kk, j = j0 + tx;
    if (k < nt && j < n) tile[kk][tx] = src[(size_t)(j + row0) + (size_t)ld * k];
  }
  __syncthreads();
  for (int jj = ty; jj < 32; jj += 8) {
    const int j = j0 + jj, k = k0 + tx;
    if (j < n && k < nchunks * 32) {
      const size_t blk = ((size_t)j * nchunks + (k >> 5)) * kCoefBlk;  // double2 units
      size_t o;
      if (q < 8) o = (blk + (q / 2) * 32 + (k & 31)) * 2 + (q % 2);
      else o = (blk + kCoefAth) * 2 + (k & 31);
      coef[o] = (k < nt) ? tile[tx][jj] : 0.0;
    }
  }
}

__global__ void observe_kernel(const double2* reg, int nchunks, int j0, const double* hw,
                               int kobs, int jobs, int jscri, const double* pw, int nt,
                               double* out) {
  const size_t rs = (size_t)nchunks * kStateBlk;
  auto psi = [&](int j, int k) { return reg[j * rs + (size_t)(k >> 5) * kStateBlk + (k & 31)]; };
  const int lane = threadIdx.x;
  if (lane == 0) {
    // HorizonSampler::sample (diagnostics.cpp:145-160): sequential dot products
    for (int d = 0; d < 4; ++d) {
      double sr = 0.0, si = 0.0;
      if (j0 >= 0 && kobs >= 0)
        for (int i = 0; i < 5 + d; ++i) {
          const double2 v = psi(j0 + i, kobs);
          sr = sr + hw[d * 8 + i] * v.x;
          si = si + hw[d * 8 + i] * v.y;
        }
      out[2 * d] = sr;
      out[2 * d + 1] = si;
    }
    double2 o = (jobs >= 0 && kobs >= 0) ? psi(jobs, kobs) : make_double2(0, 0);
    out[8] = o.x; out[9] = o.y;
    double2 sc = (jscri >= 0 && kobs >= 0) ? psi(jscri, kobs) : make_double2(0, 0);
    out[10] = sc.x; out[11] = sc.y;
  }
  // multipole_project as a linear functional of the theta slice at jobs
  double pr = 0.0, pim = 0.0;
  if (jobs >= 0)
    for (int k = lane; k < nt; k += 32) {
      const double2 v = psi(jobs, k);
      pr = fma(pw[k], v.x, pr);
      pim = fma(pw[k], v.y, pim);
    }
  for (int o = 16; o > 0; o >>= 1) {
    pr += __shfl_xor_sync(kFull, pr, o);
    pim += __shfl_xor_sync(kFull, pim, o);
  }
  if (lane == 0) { out[12] = pr; out[13] = pim; }
}

}  // namespace hwg

// ----------------------------------------------------------------------------
namespace {

template <int SCH, int MODE, int EPI>
void launch_t(const hwg_solver* s, const StageArgs& a) {
  static bool attr = [] {
    cudaFuncSetAttribute(stage_kernel<SCH, MODE, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)stage_smem_bytes<EPI>());
    return true;
  }();
  (void)attr;
  stage_kernel<SCH, MODE, EPI><<<s->blocks, kWarpsPerBlock * 32, stage_smem_bytes<EPI>(),
                                 s->stream>>>(a);
}

template <int SCH, int MODE>
void launch_m(const hwg_solver* s, const StageArgs& a, int epi) {
  switch (epi) {
    case EPI_RHS: launch_t<SCH, MODE, EPI_RHS>(s, a); break;
    case EPI_AXPY: launch_t<SCH, MODE, EPI_AXPY>(s, a); break;
    case EPI_RK3: launch_t<SCH, MODE, EPI_RK3>(s, a); break;
    case EPI_RK3C: launch_t<SCH, MODE, EPI_RK3C>(s, a); break;
    case EPI_RK104_5: launch_t<SCH, MODE, EPI_RK104_5>(s, a); break;
    default: launch_t<SCH, MODE, EPI_RK104_10>(s, a); break;
  }
}

template <int SCH>
void launch_s(const hwg_solver* s, const StageArgs& a, int epi) {
  if constexpr (SCH == FD6KO) {
    launch_m<SCH, F64>(s, a, epi);  // no weights
  } else {
    if (std::isinf(s->d.eps)) launch_m<SCH, LIN>(s, a, epi);
    else if (s->d.precision == HWG_F64) launch_m<SCH, F64>(s, a, epi);
    else launch_m<SCH, MIXED>(s, a, epi);
  }
}

int launch(hwg_solver* s, const StageArgs& a, int epi) {
  switch (s->d.scheme) {
    case HWG_WENO5: launch_s<WENO5>(s, a, epi); break;
    case HWG_WENO3: launch_s<WENO3>(s, a, epi); break;
    default: launch_s<FD6KO>(s, a, epi); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    s->err = std::string("stage launch: ") + cudaGetErrorString(e);
    return HWG_ECUDA;
  }
  return HWG_OK;
}

// row-0 pointer of state register r
double2* row0(const hwg_solver* s, int r) { return s->reg[r] + (size_t)kHalo * s->rs; }

StageArgs base_args(const hwg_solver* s) {
  StageArgs a{};
  a.n = s->n; a.nt = s->nt; a.nchunks = s->nchunks;
  a.phys_lo = s->phys_lo; a.phys_hi = s->phys_hi;
  a.nranges = s->nranges;
  a.negpar = s->d.parity < 0 ? 1 : 0;
  a.eps4 = 4.0 * s->d.eps;
  a.eps = s->d.eps;
  a.epsf = (float)s->d.eps;
  const double dr = s->d.drho;
  if (s->d.scheme == HWG_WENO5) a.iscale = 1.0 / (6.0 * dr);
  else if (s->d.scheme == HWG_WENO3) a.iscale = 1.0 / (2.0 * dr);
  else a.iscale = 1.0 / (60.0 * dr);
  a.inv1 = 1.0 / (12.0 * s->d.dtheta);
  a.inv2 = 1.0 / (12.0 * s->d.dtheta * s->d.dtheta);
  a.ko = s->d.sigma / (256.0 * dr);
  a.coef = s->coef;
  a.cot = s->cot;
  a.flag = s->flag;
  return a;
}

void set_io(StageArgs& a, const hwg_solver* s, int x, int out) {
  a.x = row0(s, x);
  a.o = row0(s, out);
}

int ensure_regs(hwg_solver* s, int need) {
  while (s->nreg < need) {
    double2* p = nullptr;
    CK(cudaMalloc(&p, s->reg_elems * sizeof(double2)));
    CK(cudaMemsetAsync(p, 0, s->reg_elems * sizeof(double2), s->stream));
    s->reg[s->nreg++] = p;
  }
  return HWG_OK;
}

// stage-input register for (stepper, stage) given the current rotation
int stage_input_reg(const hwg_solver* s, int stepper, int stage) {
  if (stepper == HWG_SSPRK33) {
    const int in[3] = {s->cur, s->scr1, s->scr2};
    return in[stage];
  }
  // rk104: U=cur, P=scr1, Q=scr2, S4=scr3, F4=scr4
  const int P = s->scr1, Q = s->scr2, S4 = s->scr3;
  const int in[10] = {s->cur, P, Q, P, S4, P, Q, P, Q, P};
  return in[stage];
}

int do_stage(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo, long long step) {
  StageArgs a = base_args(s);
  a.step = step + 1;
  const double dt = dt_hi;
  if (stepper == HWG_SSPRK33) {
    // timestep.hpp:61-70
    if (stage == 0) {
      set_io(a, s, s->cur, s->scr1);
      a.cg = dt;
      return launch(s, a, EPI_AXPY);
    }
    a.ua = row0(s, s->cur);
    a.cg = dt;
    if (stage == 1) {
      set_io(a, s, s->scr1, s->scr2);
      a.ca = 0.75; a.cb = 0.25;
      return launch(s, a, EPI_RK3);
    }
    set_io(a, s, s->scr2, s->scr1);
    a.ca = ddq(1.0, 3.0); a.cb = ddq(2.0, 3.0);
    int rc = launch(s, a, EPI_RK3C);
    std::swap(s->cur, s->scr1);
    return rc;
  }
  // ssprk104, timestep.hpp:84-108 (u^(4) kept in S4 instead of a copy)
  const int U = s->cur, P = s->scr1, Q = s->scr2, S4 = s->scr3, F4 = s->scr4;
  const DD dtd{dt_hi, dt_lo};
  const double dt6 = dd_div(dtd, {6.0, 0.0}).hi;
  const int ins[10] = {U, P, Q, P, S4, P, Q, P, Q, P};
  const int outs[10] = {P, Q, P, S4, P, Q, P, Q, P, Q};
  set_io(a, s, ins[stage], outs[stage]);
  if (stage == 4) {
    a.ua = row0(s, U);
    a.f = row0(s, F4);
    a.ca = ddq(3.0, 5.0); a.cb = ddq(2.0, 5.0);
    a.cg = dd_div(dtd, {15.0, 0.0}).hi;
    return launch(s, a, EPI_RK104_5);
  }
  if (stage == 9) {
    a.ua = row0(s, U);
    a.ub = row0(s, S4);
    a.ug = row0(s, F4);
    a.ca = ddq(1.0, 25.0); a.cb = ddq(9.0, 25.0); a.cc = ddq(3.0, 5.0);
    a.cg = dt; a.cd = ddq(3.0, 50.0); a.ce = ddq(1.0, 10.0);
    int rc = launch(s, a, EPI_RK104_10);
    std::swap(s->cur, s->scr2);
    return rc;
  }
  a.cg = dt6;
  return launch(s, a, EPI_AXPY);
}

int upload_layout(hwg_solver* s, const double* host, int stride, int reg) {
  const size_t cnt = (size_t)4 * (s->n + 8) * (s->nt + 4) * stride;
  if (s->stage_cap < cnt) {
    if (s->stage_dev) cudaFree(s->stage_dev);
    s->stage_dev = nullptr;
    s->stage_cap = 0;
    CK(cudaMalloc(&s->stage_dev, cnt * sizeof(double)));
    s->stage_cap = cnt;
  }
  CK(cudaMemcpyAsync(s->stage_dev, host, cnt * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  dim3 grid((s->n + 31) / 32, (s->nt + 31) / 32), blk(32, 8);
  relayout_kernel<<<grid, blk, 0, s->stream>>>(s->stage_dev, nullptr, row0(s, reg), s->n, s->nt,
                                                s->nchunks, stride, 0);
  CK(cudaGetLastError());
  return HWG_OK;
}

// interior of register reg -> host FieldLayout, then the reference's ghost
// rules on the host (evolve.cpp:40-71)
int download_layout(hwg_solver* s, double* host, int stride, int reg, bool ghosts) {
  const size_t cnt = (size_t)4 * (s->n + 8) * (s->nt + 4) * stride;
  if (s->stage_cap < cnt) {
    if (s->stage_dev) cudaFree(s->stage_dev);
    s->stage_dev = nullptr;
    s->stage_cap = 0;
    CK(cudaMalloc(&s->stage_dev, cnt * sizeof(double)));
    s->stage_cap = cnt;
  }
  CK(cudaMemsetAsync(s->stage_dev, 0, cnt * sizeof(double), s->stream));
  dim3 grid((s->n + 31) / 32, (s->nt + 31) / 32), blk(32, 8);
  relayout_kernel<<<grid, blk, 0, s->stream>>>(nullptr, s->stage_dev, row0(s, reg), s->n, s->nt,
                                                s->nchunks, stride, 1);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(host, s->stage_dev, cnt * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (!ghosts) return HWG_OK;
  const int n = s->n, nt = s->nt;
  const long long W = n + 8, P = W * (nt + 4);
  auto at = [&](int c, int j, int k) -> double& {
    return host[(c * P + (long long)(k + 2) * W + (j + 4)) * stride];
  };
  for (int k = 0; k < nt; ++k)
    for (int c = 0; c < 4; ++c) {
      for (int t = 1; t <= 4; ++t)
        at(c, -t, k) = 4.0 * at(c, -t + 1, k) - 6.0 * at(c, -t + 2, k) +
                       4.0 * at(c, -t + 3, k) - at(c, -t + 4, k);
      for (int t = 1; t <= 4; ++t)
        at(c, n - 1 + t, k) = 4.0 * at(c, n - 2 + t, k) - 6.0 * at(c, n - 3 + t, k) +
                              4.0 * at(c, n - 4 + t, k) - at(c, n - 5 + t, k);
    }
  const bool even = s->d.parity > 0;
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < 4; ++c)
      for (int t = 0; t < 2; ++t) {
        const double north = at(c, j, t), south = at(c, j, nt - 1 - t);
        at(c, j, -1 - t) = even ? north : -north;
        at(c, j, nt + t) = even ? south : -south;
      }
  return HWG_OK;
}

void fill_host_ghosts(const hwg_solver* s, double* u, int stride) {
  const int n = s->n, nt = s->nt;
  const long long W = n + 8, P = W * (nt + 4);
  auto at = [&](int c, int j, int k) -> double& {
    return u[(c * P + (long long)(k + 2) * W + (j + 4)) * stride];
  };
  auto lo = [&](int c, int j, int k) -> double& {
    return u[(c * P + (long long)(k + 2) * W + (j + 4)) * stride + 1];
  };
  for (int k = 0; k < nt; ++k)
    for (int c = 0; c < 4; ++c) {
      for (int t = 1; t <= 4; ++t) {
        at(c, -t, k) = 4.0 * at(c, -t + 1, k) - 6.0 * at(c, -t + 2, k) +
                       4.0 * at(c, -t + 3, k) - at(c, -t + 4, k);
        if (stride == 2) lo(c, -t, k) = 0.0;
      }
      for (int t = 1; t <= 4; ++t) {
        at(c, n - 1 + t, k) = 4.0 * at(c, n - 2 + t, k) - 6.0 * at(c, n - 3 + t, k) +
                              4.0 * at(c, n - 4 + t, k) - at(c, n - 5 + t, k);
        if (stride == 2) lo(c, n - 1 + t, k) = 0.0;
      }
    }
  const bool even = s->d.parity > 0;
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < 4; ++c)
      for (int t = 0; t < 2; ++t) {
        const double north = at(c, j, t), south = at(c, j, nt - 1 - t);
        at(c, j, -1 - t) = even ? north : -north;
        at(c, j, nt + t) = even ? south : -south;
        if (stride == 2) { lo(c, j, -1 - t) = 0.0; lo(c, j, nt + t) = 0.0; }
      }
}

int rhs_impl(hwg_solver* s, double* u, double* du, int stride) {
  int rc = upload_layout(s, u, stride, s->scr1);
  if (rc) return rc;
  StageArgs a = base_args(s);
  a.flag = nullptr;  // the RHS never freezes
  set_io(a, s, s->scr1, s->scr2);
  rc = launch(s, a, EPI_RHS);
  if (rc) return rc;
  // du interior only; its ghosts stay as the caller gave them
  const int n = s->n, nt = s->nt;
  const size_t cnt = (size_t)4 * (n + 8) * (nt + 4) * stride;
  std::vector<double> tmp(cnt);
  rc = download_layout(s, tmp.data(), stride, s->scr2, false);
  if (rc) return rc;
  const long long W = n + 8, P = W * (nt + 4);
  for (int c = 0; c < 4; ++c)
    for (int k = 0; k < nt; ++k) {
      const size_t o = (c * P + (long long)(k + 2) * W + 4) * stride;
      std::memcpy(du + o, tmp.data() + o, sizeof(double) * n * stride);
    }
  fill_host_ghosts(s, u, stride);
  return HWG_OK;
}

DD tau_of(long long step, double dt_hi, double dt_lo) {  // WorkReal(double(s)) * dt
  return dd_mul({(double)step, 0.0}, {dt_hi, dt_lo});
}

}  // namespace

// ----------------------------------------------------------------------------
extern "C" {

const char* hwg_last_error(const hwg_solver* s) {
  return s ? s->err.c_str() : g_create_err.c_str();
}

int hwg_create(const hwg_desc* d, const double* coef, const double* cotth, hwg_solver** out) {
  *out = nullptr;
  if (!d || !coef || !cotth) {
    g_create_err = "hwg_create: null argument";
    return HWG_EINVAL;
  }
  // EvolutionRhs ctor: grid below stencil support (evolve.cpp:16-17)
  const int nglob = d->nrho_global > 0 ? d->nrho_global : d->nrho;
  if (nglob < 9 || d->ntheta < 2 || d->nrho < 8) {
    g_create_err = "EvolutionRhs: grid below stencil support";
    return HWG_EINVAL;
  }
  if (d->scheme < 0 || d->scheme > 2 || d->precision < 0 || d->precision > 1 ||
      !(d->drho > 0.0) || !(d->dtheta > 0.0)) {
    g_create_err = "hwg_create: invalid scheme/precision/spacing";
    return HWG_EINVAL;
  }
  const int ld = d->coef_ld > 0 ? d->coef_ld : nglob;
  const int row0 = d->coef_row0 >= 0 ? d->coef_row0 : d->rho_offset;
  // lam sign structure (evolve.cpp:19-30): lam < 0 on [0, split), >= 0 after
  const double* lam = coef + (size_t)ld * d->ntheta;
  for (int k = 0; k < d->ntheta; ++k) {
    int j = 0;
    while (j < d->nrho && lam[(size_t)(row0 + j) + (size_t)ld * k] < 0.0) ++j;
    for (; j < d->nrho; ++j)
      if (lam[(size_t)(row0 + j) + (size_t)ld * k] < 0.0) {
        g_create_err = "EvolutionRhs: lam changes sign more than once along a row";
        return HWG_ERUNTIME;
      }
  }
  auto* s = new hwg_solver();
  s->d = *d;
  s->d.nrho_global = nglob;
  s->n = d->nrho;
  s->nt = d->ntheta;
  s->ntp = (d->ntheta + 31) / 32 * 32;
  s->nchunks = s->ntp / 32;
  s->rs = (size_t)s->nchunks * kStateBlk;
  s->phys_lo = d->rho_offset == 0;
  s->phys_hi = d->rho_offset + d->nrho == nglob;
  s->dev = d->device;
  s->reg_elems = (size_t)(s->n + 2 * kHalo) * s->rs;
  auto fail = [&](int rc) {
    g_create_err = s->err;
    hwg_destroy(s);
    return rc;
  };
  if (cudaSetDevice(s->dev) != cudaSuccess) {
    s->err = "cudaSetDevice failed (no GPU?)";
    return fail(HWG_ECUDA);
  }
#undef CK
#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      s->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return fail(HWG_ECUDA);                                                  \
    }                                                                          \
  } while (0)
  CK(cudaStreamCreateWithFlags(&s->own, cudaStreamNonBlocking));
  s->stream = s->own;
  const size_t CB = (size_t)s->n * s->nchunks * kCoefBlk;
  CK(cudaMalloc(&s->coef, CB * sizeof(double2)));
  CK(cudaMemsetAsync(s->coef, 0, CB * sizeof(double2), s->stream));
  CK(cudaMalloc(&s->cot, s->ntp * sizeof(double)));
  CK(cudaMalloc(&s->flag, 2 * sizeof(unsigned long long)));
  CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
  CK(cudaMallocHost(&s->hflag, 2 * sizeof(unsigned long long)));
  CK(cudaMallocHost(&s->obs_host, 16 * sizeof(double)));
  CK(cudaMalloc(&s->obs_dev, 16 * sizeof(double)));
  CK(cudaMalloc(&s->obs_w, (32 + s->ntp) * sizeof(double)));
  CK(cudaMemsetAsync(s->obs_w, 0, (32 + s->ntp) * sizeof(double), s->stream));
  // coefficients: upload each reference plane (rows of this handle) and
  // transpose on the device into (row, theta) order
  {
    double* tmp = nullptr;
    const size_t plane_src = (size_t)ld * s->nt;
    CK(cudaMalloc(&tmp, plane_src * sizeof(double)));
    dim3 grid((s->n + 31) / 32, s->nchunks), blk(32, 8);
    for (int q = 0; q < 9; ++q) {
      CK(cudaMemcpyAsync(tmp, coef + q * plane_src, plane_src * sizeof(double),
                         cudaMemcpyHostToDevice, s->stream));
      coef_kernel<<<grid, blk, 0, s->stream>>>(tmp, ld, row0, reinterpret_cast<double*>(s->coef), q,
                                                s->n, s->nt, s->nchunks);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s->stream));
    cudaFree(tmp);
    std::vector<double> c(s->ntp, 0.0);
    for (int k = 0; k < s->nt; ++k) c[k] = cotth[k];
    CK(cudaMemcpy(s->cot, c.data(), s->ntp * sizeof(double), cudaMemcpyHostToDevice));
  }
  {
    int rc = ensure_regs(s, 3);
    if (rc) return fail(rc);
  }
  // launch geometry: one wave of warps, rho ranges balanced per theta chunk
  {
    int nsm = 148, occ = 1;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->dev));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, stage_kernel<WENO5, F64, EPI_RK3>));
    CK(cudaFuncSetAttribute(stage_kernel<WENO5, F64, EPI_RK3>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)stage_smem_bytes<EPI_RK3>()));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stage_kernel<WENO5, F64, EPI_RK3>,
                                                     kWarpsPerBlock * 32,
                                                     stage_smem_bytes<EPI_RK3>()));
    const long long target = (long long)nsm * std::max(occ, 1) * kWarpsPerBlock;
    long long nr = std::max<long long>(1, target / s->nchunks);
    nr = std::min<long long>(nr, std::max(1, s->n / 8));  // >= 8 rows per range
    s->nranges = (int)nr;
    s->blocks = (int)((nr * s->nchunks + kWarpsPerBlock - 1) / kWarpsPerBlock);
  }
  CK(cudaStreamSynchronize(s->stream));
#undef CK
#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      s->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return HWG_ECUDA;                                                        \
    }                                                                          \
  } while (0)
  *out = s;
  return HWG_OK;
}

void hwg_destroy(hwg_solver* s) {
  if (!s) return;
  cudaSetDevice(s->dev);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (int i = 0; i < s->nreg; ++i) cudaFree(s->reg[i]);
  cudaFree(s->coef);
  cudaFree(s->cot);
  cudaFree(s->flag);
  cudaFree(s->stage_dev);
  cudaFree(s->obs_dev);
  cudaFree(s->obs_w);
  if (s->hflag) cudaFreeHost(s->hflag);
  if (s->obs_host) cudaFreeHost(s->obs_host);
  if (s->own) cudaStreamDestroy(s->own);
  delete s;
}

int hwg_set_stream(hwg_solver* s, void* stream, int own) {
  s->stream = own ? s->own : static_cast<cudaStream_t>(stream);
  return HWG_OK;
}

int hwg_set_state_dd(hwg_solver* s, const double* u) {
  cudaSetDevice(s->dev);
  int rc = upload_layout(s, u, 2, s->cur);
  if (rc) return rc;
  CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return HWG_OK;
}
int hwg_set_state(hwg_solver* s, const double* u) {
  cudaSetDevice(s->dev);
  int rc = upload_layout(s, u, 1, s->cur);
  if (rc) return rc;
  CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return HWG_OK;
}
int hwg_get_state_dd(hwg_solver* s, double* u) {
  cudaSetDevice(s->dev);
  return download_layout(s, u, 2, s->cur, true);
}
int hwg_get_state(hwg_solver* s, double* u) {
  cudaSetDevice(s->dev);
  return download_layout(s, u, 1, s->cur, true);
}

int hwg_rhs(hwg_solver* s, double* u, double* du) {
  cudaSetDevice(s->dev);
  return rhs_impl(s, u, du, 1);
}
int hwg_rhs_dd(hwg_solver* s, double* u, double* du) {
  cudaSetDevice(s->dev);
  return rhs_impl(s, u, du, 2);
}

int hwg_launch_stage(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo,
                     long long step) {
  if (stepper == HWG_SSPRK104) {
    int rc = ensure_regs(s, 5);
    if (rc) return rc;
  }
  const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
  if (stage < 0 || stage >= ns) {
    s->err = "hwg_launch_stage: stage out of range";
    return HWG_EINVAL;
  }
  return do_stage(s, stepper, stage, dt_hi, dt_lo, step);
}

int hwg_launch_steps(hwg_solver* s, int stepper, double dt_hi, double dt_lo,
                     long long step_begin, long long nsteps) {
  const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
  for (long long q = 0; q < nsteps; ++q)
    for (int st = 0; st < ns; ++st) {
      int rc = hwg_launch_stage(s, stepper, st, dt_hi, dt_lo, step_begin + q);
      if (rc) return rc;
    }
  return HWG_OK;
}

int hwg_stage_input(const hwg_solver* s, int stepper, int stage, int* reg) {
  *reg = stage_input_reg(s, stepper, stage);
  return HWG_OK;
}

int hwg_register_ptr(const hwg_solver* s, int reg, void** row0_ptr, long long* row_elems) {
  if (reg < 0 || reg >= s->nreg) return HWG_EINVAL;
  *row0_ptr = row0(s, reg);
  *row_elems = (long long)s->rs;
  return HWG_OK;
}

int hwg_current_register(const hwg_solver* s) { return s->cur; }

int hwg_status(hwg_solver* s, int* blew, long long* step, int clear) {
  CK(cudaMemcpyAsync(s->hflag, s->flag, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     s->stream));
  CK(cudaStreamSynchronize(s->stream));
  *blew = s->hflag[0] != 0;
  *step = *blew ? (long long)s->hflag[1] : -1;
  if (clear) CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
  return HWG_OK;
}

int hwg_launch_info(const hwg_solver* s, int* blocks, int* threads, int* nranges, int* nchunks,
                    int* pitch) {
  *blocks = s->blocks;
  *threads = kWarpsPerBlock * 32;
  *nranges = s->nranges;
  *nchunks = s->nchunks;
  *pitch = (int)s->rs;
  return HWG_OK;
}

int hwg_synchronize(hwg_solver* s) {
  CK(cudaStreamSynchronize(s->stream));
  return HWG_OK;
}

int hwg_set_observers(hwg_solver* s, int kobs, int j0, const double* hw, int jobs,
                      const double* pw) {
  if (kobs >= s->nt || j0 + 8 > s->n || jobs >= s->n) {
    s->err = "hwg_set_observers: observer outside this handle's rows";
    return HWG_EINVAL;
  }
  s->kobs = kobs;
  s->j0 = hw ? j0 : -1;
  s->jobs = pw ? jobs : -1;
  std::vector<double> w(32 + s->ntp, 0.0);
  if (hw) std::memcpy(w.data(), hw, 32 * sizeof(double));
  if (pw) std::memcpy(w.data() + 32, pw, s->nt * sizeof(double));
  CK(cudaMemcpy(s->obs_w, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
  return HWG_OK;
}

int hwg_observe(hwg_solver* s, hwg_observables* out) {
  observe_kernel<<<1, 32, 0, s->stream>>>(row0(s, s->cur), s->nchunks, s->j0, s->obs_w, s->kobs,
                                           s->jobs, s->phys_hi ? s->n - 1 : -1, s->obs_w + 32,
                                           s->nt, s->obs_dev);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(s->obs_host, s->obs_dev, 14 * sizeof(double), cudaMemcpyDeviceToHost,
                     s->stream));
  CK(cudaStreamSynchronize(s->stream));
  const double* o = s->obs_host;
  out->phi[0] = o[0]; out->phi[1] = o[1];
  for (int d = 0; d < 3; ++d) { out->dphi[d][0] = o[2 + 2 * d]; out->dphi[d][1] = o[3 + 2 * d]; }
  out->obs[0] = o[8]; out->obs[1] = o[9];
  out->scri[0] = o[10]; out->scri[1] = o[11];
  out->proj[0] = o[12]; out->proj[1] = o[13];
  return HWG_OK;
}

int hwg_advance(hwg_solver* s, int stepper, double dt_hi, double dt_lo, long long s0,
                long long s1, long long every, hwg_hook_fn hook, void* user,
                hwg_run_stats* stats) {
  cudaSetDevice(s->dev);
  hwg_run_stats st{0, 0.0, 0, -1};
  if (every < 1) every = 1;
  const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
  const long long poll = 256;
  auto t0 = std::chrono::steady_clock::now();
  int rc = HWG_OK;
  long long launched_to = s0;  // steps [s0, launched_to) are queued
  auto check_flag = [&](bool& blown) -> int {
    int b;
    long long bs;
    int r = hwg_status(s, &b, &bs, 0);
    if (r) return r;
    blown = b != 0;
    if (blown) {
      st.blew_up = 1;
      st.blowup_step = bs;
      st.steps_done = bs - s0;
    }
    return HWG_OK;
  };
  for (long long q = s0;; ++q) {
    const bool hook_now = hook && (q % every == 0 || q == s0 || q == s1);
    if (hook_now || q == s1 || (q - s0) % poll == 0) {
      bool blown = false;
      if ((rc = check_flag(blown))) break;
      if (blown) break;
    }
    if (hook_now) {
      hwg_observables ob;
      if ((rc = hwg_observe(s, &ob))) break;
      DD tau = tau_of(q, dt_hi, dt_lo);
      hook(q, tau.hi, tau.lo, &ob, user);
    }
    if (q == s1) break;
    for (int k = 0; k < ns && rc == HWG_OK; ++k) rc = hwg_launch_stage(s, stepper, k, dt_hi, dt_lo, q);
    if (rc) break;
    launched_to = q + 1;
    st.steps_done = launched_to - s0;
  }
  cudaStreamSynchronize(s->stream);
  st.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (stats) *stats = st;
  return rc;
}

}  // extern "C"
